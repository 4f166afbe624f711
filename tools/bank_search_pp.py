"""Layout search for the ping-pong line-per-thread smoother kernel
(paper_2405_19004_b200/csrc/smoother_impl.cuh, 3D).

Every contraction stage X in A..G reads its input tensor along one direction
(lanes over the other two) and writes its output tensor, in a fresh layout,
into the other of two work buffers. A layout is a set of strides for the
tensor's three indices; a stage's lane order (which of its two line indices
runs fastest) is shared by its reads and writes. Dynamic programming over the
stage chain picks the lane orders and, per tensor, the strides minimising
the modelled shared-memory wavefronts (tools/bank_search.py model).

python tools/bank_search_pp.py K f64|f32 [PB]  -> C++ table row
"""

import itertools
import sys
from collections import defaultdict

from bank_search import wavefronts

PBS = {1: 16, 2: 8, 3: 4, 4: 2, 5: 2, 6: 1, 7: 1}
WIDE = False


def cost_of(instrs, word):
    tot = 0
    for ins in instrs:
        warps = defaultdict(list)
        for tid, a in ins:
            warps[tid // 32].append((tid % 32, a))
        for wl in warps.values():
            tot += wavefronts(wl, word)[0]
    return tot


def lines(PB, n_fast, n_slow, flip):
    """thread -> (tid, p, a, b): a has extent n_fast, b extent n_slow; flip
    makes b run fastest across lanes"""
    out = []
    per = n_fast * n_slow
    for tid in range(PB * per):
        p, rr = divmod(tid, per)
        if not flip:
            b, a = divmod(rr, n_fast)
        else:
            a, b = divmod(rr, n_slow)
        out.append((tid, p, a, b))
    return out


# stage definitions: (name, n_a, n_b, read-extent, write-extent)
#   the stage's lines are indexed (a, b); it reads its input tensor at
#   (line, t) and writes its output tensor at (line, i)
def stage_dims(K):
    NC, NI = 2 * K + 1, 2 * K - 1
    # name: (n_a, n_b, n_read, n_write, n_arrays_read, n_arrays_written)
    return {
        "A": (NC, NC, NC, NI, 1, 2),  # lines (j1, j2), read U along t0, write zM/zA along i0
        "B": (NI, NC, NC, NI, 2, 2),  # lines (i0, j2), along j1 -> i1
        "C": (NI, NI, NC, NI, 2, 1),  # lines (i0, i1), along j2 -> c2
        "D": (NI, NI, NI, NI, 1, 1),  # lines (i0, c2), along i1 -> c1
        "E": (NI, NI, NI, NI, 1, 1),  # lines (c1, c2), along i0 -> i0
        "F": (NI, NI, NI, NI, 1, 1),  # lines (i0, c2), along c1 -> i1
        "G": (NI, NI, NI, 0, 1, 0),   # lines (i0, i1), along c2 -> global
    }


# For the tensor written by stage X and read by stage X+1 we need the map
# from (writer line a, writer line b, element i) and (reader line a, reader
# line b, element t) to the tensor's own index triple (u0, u1, u2). Tensor
# index order: (dir0-type index, dir1-type index, dir2-type index).
def writer_idx(X, a, b, i):
    return {"A": (i, a, b), "B": (a, i, b), "C": (a, b, i), "D": (a, i, b), "E": (i, a, b), "F": (a, i, b)}[X]


def reader_idx(Y, a, b, t):
    return {"B": (a, t, b), "C": (a, b, t), "D": (a, t, b), "E": (t, a, b), "F": (a, t, b), "G": (a, b, t)}[Y]


NEXT = {"A": "B", "B": "C", "C": "D", "D": "E", "E": "F", "F": "G"}


def tensor_cost(K, PB, X, fX, fY, s, arrsep, word):
    """wavefronts of stage X writing and stage Y=NEXT[X] reading tensor X with
    strides s = (s0, s1, s2); arrays (zM | zA etc.) are arrsep words apart;
    patches are WW = per-patch stride words apart (folded into s via p)"""
    dims = stage_dims(K)
    Y = NEXT[X]
    na, nb, _, nw, _, narr_w = dims[X]
    ya, yb, nr, _, narr_r, _ = dims[Y]
    WW = s[3]
    ins = []
    LX = lines(PB, na, nb, fX)
    for arr in range(narr_w):
        for i in range(nw):
            ins.append([(tid, p * WW + arr * arrsep + sum(x * y for x, y in zip(writer_idx(X, a, b, i), s[:3])))
                        for tid, p, a, b in LX])
    LY = lines(PB, ya, yb, fY)
    for arr in range(narr_r):
        for t in range(nr):
            ins.append([(tid, p * WW + arr * arrsep + sum(x * y for x, y in zip(reader_idx(Y, a, b, t), s[:3])))
                        for tid, p, a, b in LY])
    return cost_of(ins, word)


def extents(K, X):
    NC, NI = 2 * K + 1, 2 * K - 1
    return {"A": (NI, NC, NC), "B": (NI, NI, NC), "C": (NI, NI, NI), "D": (NI, NI, NI), "E": (NI, NI, NI),
            "F": (NI, NI, NI)}[X]


def best_layout(K, PB, X, fX, fY, word, budget):
    """search strides (a permutation of the index order with small pads), then
    the array separation and the per-patch stride; returns (cost, (strides,
    arrsep, per-patch stride))"""
    e = extents(K, X)
    narr = stage_dims(K)[X][5]
    best = None
    for perm in itertools.permutations(range(3)):
        for p1 in range(0, 4):
            for p2 in range(0, 6):
                s = [0, 0, 0]
                s[perm[0]] = 1
                s[perm[1]] = e[perm[0]] + p1
                s[perm[2]] = s[perm[1]] * e[perm[1]] + p2
                size1 = s[perm[2]] * e[perm[2]]
                arrsep = size1 + 1
                WW = arrsep * (narr - 1) + size1 + 1
                c = tensor_cost(K, PB, X, fX, fY, (s[0], s[1], s[2], WW), arrsep, word)
                key = (c, size1)
                if best is None or key < best[0]:
                    best = (key, (tuple(s), size1))
    s, size1 = best[1]
    best2 = None
    # --wide: the pads over a full bank period (32 words), since the per-patch
    # stride modulo the bank count decides where a warp's next patch lands
    span = 33 if WIDE else 9
    for pa in range(0, span if narr == 2 else 1):
        arrsep = size1 + pa
        tot1 = arrsep * (narr - 1) + size1
        for pw in range(0, span):
            WW = tot1 + pw
            c = tensor_cost(K, PB, X, fX, fY, (s[0], s[1], s[2], WW), arrsep, word)
            key = (c, WW)
            if best2 is None or key < best2[0]:
                best2 = (key, (tuple(s), arrsep, WW))
    return best2[0][0], best2[1]


def u_read_cost(K, PB, fA, word):
    """stage A reads the staged closure U[t2][t1][t0] (strides 1, NC, NC^2,
    per patch NC^3) along t0, lanes over (t1, t2)"""
    NC = 2 * K + 1
    L = lines(PB, NC, NC, fA)
    ins = [[(tid, p * NC ** 3 + t + NC * a + NC * NC * b) for tid, p, a, b in L] for t in range(NC)]
    return cost_of(ins, word)


def search(K, word, PB):
    stages = ["A", "B", "C", "D", "E", "F", "G"]
    # DP over lane orders
    table = {}
    for X in stages[:-1]:
        for fX in (0, 1):
            for fY in (0, 1):
                table[(X, fX, fY)] = best_layout(K, PB, X, fX, fY, word, None)
    best = None
    for flips in itertools.product((0, 1), repeat=7):
        c = u_read_cost(K, PB, flips[0], word)
        for idx, X in enumerate(stages[:-1]):
            c += table[(X, flips[idx], flips[idx + 1])][0]
        if best is None or c < best[0]:
            best = (c, flips)
    flips = best[1]
    lay = {X: table[(X, flips[i], flips[i + 1])] for i, X in enumerate(stages[:-1])}
    return best[0], flips, lay


def ideal(K, PB, word):
    """wavefront count with every access conflict-free (same accesses)"""
    dims = stage_dims(K)
    tot = 0
    for X, (na, nb, nr, nw, narr_r, narr_w) in dims.items():
        nthr = PB * na * nb
        warps = [min(32, nthr - 32 * w) for w in range((nthr + 31) // 32)]
        per = sum((2 if (word == 8 and n > 16) else 1) for n in warps)
        tot += per * (nr * narr_r + nw * narr_w)
    return tot


if __name__ == "__main__":
    if "--wide" in sys.argv:
        sys.argv.remove("--wide")
        WIDE = True
    K = int(sys.argv[1])
    word = 8 if sys.argv[2] == "f64" else 4
    PB = int(sys.argv[3]) if len(sys.argv) > 3 else PBS[K]
    c, flips, lay = search(K, word, PB)
    print(f"K={K} {sys.argv[2]} PB={PB}: modelled {c} wavefronts (ideal {ideal(K, PB, word)})")
    print("  flips A..G:", flips)
    for X, (cx, (s, arrsep, WW)) in lay.items():
        print(f"  T_{X}: strides {s} arrsep {arrsep} per-patch {WW}  cost {cx}")
