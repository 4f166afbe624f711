"""Bank-conflict model / layout search for the 3D line-per-thread smoother
kernel (paper_2405_19004_b200/csrc/smoother_impl.cuh, vp_smooth_kernel).

Same wavefront model as tools/bank_search.py. Every stage's thread -> line
mapping is the kernel's; per stage the lane order can be flipped (which of the
two non-contracted indices runs fastest), and the strides (S1, S2, ZS, ZW) of
the work array are searched.

python tools/bank_search_line.py K f64|f32
"""

import sys
from collections import defaultdict

from bank_search import wavefronts

PBS = {1: 16, 2: 8, 3: 4, 4: 2, 5: 2, 6: 1, 7: 1}


def stages(K, PB, NT, UW, BW, S1, S2, ZS, ZW, flip):
    NC, NI = 2 * K + 1, 2 * K - 1

    def lines(n_fast, n_slow, f):
        """thread -> (p, a, b) where a, b are the two line indices; with f the
        slow index runs fastest across lanes"""
        out = []
        per = n_fast * n_slow
        for tid in range(PB * per):
            p, rr = divmod(tid, per)
            if not f:
                b, a = divmod(rr, n_fast)
            else:
                a, b = divmod(rr, n_slow)
            out.append((tid, p, a, b))
        return out

    Z = lambda p, i0, i1, i2, arr=0: p * ZW + arr * ZS + i0 + S1 * i1 + S2 * i2  # noqa: E731
    U = lambda p, t0, t1, t2: p * UW + t0 + NC * t1 + NC * NC * t2  # noqa: E731
    # closure cp.async: lane -> (p, t0 + NC t1), walking t2
    for t in range(NC):
        yield "ldgsts", [(tid, p * UW + rr + NC * NC * t) for tid, p, rr in
                         [(tid, *divmod(tid, NC * NC)) for tid in range(PB * NC * NC)]]
    for t in range(NI):
        yield "ldgsts_b", [(tid, p * BW + rr + NI * NI * t) for tid, p, rr in
                           [(tid, *divmod(tid, NI * NI)) for tid in range(PB * NI * NI)]]
    # A: line along dir 0 over (j1, j2)
    L = lines(NC, NC, flip[0])
    for t in range(NC):
        yield "A_ld", [(tid, U(p, t, j1, j2)) for tid, p, j1, j2 in L]
    for arr in (0, 1):
        for i in range(NI):
            yield "A_st", [(tid, Z(p, i, j1, j2, arr)) for tid, p, j1, j2 in L]
    # B: along dir 1 over (i0, j2)
    L = lines(NI, NC, flip[1])
    for arr in (0, 1):
        for t in range(NC):
            yield "B_ld", [(tid, Z(p, i0, t, j2, arr)) for tid, p, i0, j2 in L]
    for arr in (0, 1):
        for i in range(NI):
            yield "B_st", [(tid, Z(p, i0, i, j2, arr)) for tid, p, i0, j2 in L]
    # C: along dir 2 over (i0, i1)
    L = lines(NI, NI, flip[2])
    for arr in (0, 1):
        for t in range(NC):
            yield "C_ld", [(tid, Z(p, i0, i1, t, arr)) for tid, p, i0, i1 in L]
    for i in range(NI):
        yield "C_b", [(tid, p * BW + i0 + NI * i1 + NI * NI * i) for tid, p, i0, i1 in L]
    for c in range(NI):
        yield "C_st", [(tid, Z(p, i0, i1, c)) for tid, p, i0, i1 in L]
    # D/F: along dir 1 over (i0, i2)
    L = lines(NI, NI, flip[3])
    for _ in range(2):
        for t in range(NI):
            yield "DF_ld", [(tid, Z(p, i0, t, i2)) for tid, p, i0, i2 in L]
        for t in range(NI):
            yield "DF_st", [(tid, Z(p, i0, t, i2)) for tid, p, i0, i2 in L]
    # E: along dir 0 over (i1, i2)
    L = lines(NI, NI, flip[4])
    for t in range(NI):
        yield "E_ld", [(tid, Z(p, t, i1, i2)) for tid, p, i1, i2 in L]
    for t in range(NI):
        yield "E_st", [(tid, Z(p, t, i1, i2)) for tid, p, i1, i2 in L]
    # G: along dir 2 over (i0, i1) + x_old from U
    L = lines(NI, NI, flip[5])
    for t in range(NI):
        yield "G_ld", [(tid, Z(p, i0, i1, t)) for tid, p, i0, i1 in L]
    for t in range(NI):
        yield "G_xo", [(tid, U(p, 1 + i0, 1 + i1, 1 + t)) for tid, p, i0, i1 in L]


def cost(word, *args, detail=False):
    tot = ideal = 0
    per = defaultdict(lambda: [0, 0])
    for name, ins in stages(*args):
        warps = defaultdict(list)
        for tid, a in ins:
            warps[tid // 32].append((tid % 32, a))
        for wl in warps.values():
            t, i = wavefronts(wl, word)
            tot += t
            ideal += i
            per[name][0] += t
            per[name][1] += i
    return (tot, ideal, dict(per)) if detail else (tot, ideal)


def fmt(per):
    return " ".join(f"{k}={v[0]}/{v[1]}" for k, v in per.items())


if __name__ == "__main__":
    K = int(sys.argv[1])
    word = 8 if sys.argv[2] == "f64" else 4
    NC, NI = 2 * K + 1, 2 * K - 1
    PB = PBS[K]
    NT = ((PB * NC * NC + 31) // 32) * 32
    cur = {  # the kernel's current table (smoother_impl.cuh ZLayout)
        8: {1: (1, 3, 7), 2: (3, 15, 3), 3: (5, 38, 5), 4: (7, 70, 5), 5: (9, 105, 11), 6: (11, 155, 0),
            7: (13, 205, 0)},
        4: {1: (1, 3, 3), 2: (3, 15, 0), 3: (5, 35, 15), 4: (7, 72, 1), 5: (9, 113, 3), 6: (11, 143, 0),
            7: (13, 201, 0)},
    }[word][K]
    S1, S2, ZP = cur
    ZS = S2 * NC
    args = (K, PB, NT, NC ** 3, NI ** 3 + 1, S1, S2, ZS, 2 * ZS + ZP, (0, 0, 0, 0, 0, 0))
    t, i, per = cost(word, *args, detail=True)
    print(f"current S1={S1} S2={S2} ZS={ZS} ZW={2 * ZS + ZP}: {t}/{i}  {fmt(per)}")
    # search: strides of Z, the b array pitch and per-stage lane order
    best = None
    import itertools
    for S1 in range(NI, NI + 8):
        for S2 in range(NC * S1, NC * S1 + 16):
            for flipB in (0, 1):
                for flipC in (0, 1):
                    for flipD in (0, 1):
                        a = (K, PB, NT, NC ** 3, NI ** 3 + 1, S1, S2, S2 * NC, 2 * S2 * NC, (0, flipB, flipC, flipD, 0, 0))
                        _, _, per = cost(word, *a, detail=True)
                        c = sum(v[0] for k, v in per.items() if k[0] in "ABCDF")
                        key = (c, S1 * S2)
                        if best is None or key < best[0]:
                            best = (key, (S1, S2, flipB, flipC, flipD))
    S1, S2, fB, fC, fD = best[1]
    bestZ = None
    for ZS in range(S2 * NC, S2 * NC + 16):
        for ZP in range(0, 17):
            for flipE in (0, 1):
                for flipG in (0, 1):
                    a = (K, PB, NT, NC ** 3, NI ** 3 + 1, S1, S2, ZS, 2 * ZS + ZP, (0, fB, fC, fD, flipE, flipG))
                    t, i = cost(word, *a)
                    key = (t, ZS + ZP)
                    if bestZ is None or key < bestZ[0]:
                        bestZ = (key, (ZS, ZP, flipE, flipG))
    ZS, ZP, fE, fG = bestZ[1]
    a = (K, PB, NT, NC ** 3, NI ** 3 + 1, S1, S2, ZS, 2 * ZS + ZP, (0, fB, fC, fD, fE, fG))
    t, i, per = cost(word, *a, detail=True)
    print(f"best S1={S1} S2={S2} ZS={ZS} ZW={2 * ZS + ZP} flips B{fB} C{fC} D{fD} E{fE} G{fG}: {t}/{i}  {fmt(per)}")
