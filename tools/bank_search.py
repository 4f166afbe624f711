"""Shared-memory bank-conflict model and layout search for the plane-streaming
smoother kernel (paper_2405_19004_b200/csrc/smoother_plane.cuh).

Model (sm_100 shared memory, 32 banks x 4 B): a warp-wide access of 4-byte
words costs max over banks of the number of distinct words hitting the bank;
8-byte words are served per half-warp (lanes 0-15, 16-31), each half costing
max over bank pairs (word mod 16) of the number of distinct words. The ideal
is the same count with every bank hit by one distinct word.

python tools/bank_search.py K f64|f32     -> best layouts for that kernel
"""

import itertools
import sys
from collections import defaultdict


def wavefronts(addrs, word):
    """addrs: list of (lane, word address) of one warp instruction."""
    if not addrs:
        return 0, 0
    if word == 8:
        tot = ideal = 0
        for half in (0, 1):
            sub = {a for lane, a in addrs if lane // 16 == half}
            if not sub:
                continue
            cnt = defaultdict(set)
            for a in sub:
                cnt[a % 16].add(a)
            tot += max(len(s) for s in cnt.values())
            ideal += 1
        return tot, ideal
    sub = {a for _, a in addrs}
    cnt = defaultdict(set)
    for a in sub:
        cnt[a % 32].add(a)
    return max(len(s) for s in cnt.values()), 1


class Layout:
    def __init__(self, K, PB, NT, UW, SU1, SU2, WW, SJ, SW):
        self.K, self.PB, self.NT = K, PB, NT
        self.NC, self.NI = 2 * K + 1, 2 * K - 1
        self.UW, self.SU1, self.SU2 = UW, SU1, SU2
        self.WW, self.SJ, self.SW = WW, SJ, SW

    def u(self, p, t2, t1, t0):
        return p * self.UW + t2 * self.SU2 + t1 * self.SU1 + t0

    def w(self, p, which, j, q):
        return p * self.WW + which * self.SW + j * self.SJ + q


def phases(L: Layout):
    """Yield (phase, list of per-instruction lists of (tid, addr)) for one CTA."""
    NC, NI, PB, NT = L.NC, L.NI, L.PB, L.NT
    NI2 = NI * NI
    # closure cp.async, tile-row staging: element e = tid + NT*it of the
    # union rows (t1, t2) x X in [0, 2K PB + 1); X goes to patch min(X/2K, PB-1)
    # and, when it is a shared vertex column, also to patch X/2K - 1 (t0 = 2K)
    RX = 2 * L.K * PB + 1
    tot = NC * NC * RX
    for it in range((tot + NT - 1) // NT):
        ins, ins2 = [], []
        for tid in range(NT):
            e = tid + NT * it
            if e >= tot:
                continue
            row, X = divmod(e, RX)
            t2, t1 = divmod(row, NC)
            p = min(X // (2 * L.K), PB - 1)
            ins.append((tid, L.u(p, t2, t1, X - 2 * L.K * p)))
            if X % (2 * L.K) == 0 and 0 < X < RX - 1:
                ins2.append((tid, L.u(X // (2 * L.K) - 1, t2, t1, 2 * L.K)))
        yield "ldgsts", ins
        yield "ldgsts", ins2
    # P1 reads (thread p, j2): rows jj, NC-1-jj, all t
    order = []
    for jj in range(L.K + 1):
        rows = [jj] if jj == L.K else [jj, NC - 1 - jj]
        for r in rows:
            for t in range(NC):
                order.append((r, t))
    for r, t in order:
        ins = [(tid, L.u(tid // NC, tid % NC, r, t)) for tid in range(PB * NC)]
        yield "p1_ld", ins
    for which in (0, 1):
        for q in range(NI2):
            ins = [(tid, L.w(tid // NC, which, tid % NC, q)) for tid in range(PB * NC)]
            yield "p1_st", ins
    # P2 (thread p, rr = i0 + NI i1)
    for which in (0, 1):
        for t in range(NC):
            ins = [(tid, L.w(tid // NI2, which, t, tid % NI2)) for tid in range(PB * NI2)]
            yield "p2_ld", ins
    for c in range(NI):
        ins = [(tid, L.w(tid // NI2, 0, c, tid % NI2)) for tid in range(PB * NI2)]
        yield "p2_st", ins
    # P3 (thread p, c2): whole plane
    for q in range(NI2):
        ins = [(tid, L.w(tid // NI, 0, tid % NI, q)) for tid in range(PB * NI)]
        yield "p3_ld", ins
        yield "p3_st", ins
    # P4: eigen column + x_old
    for c in range(NI):
        ins = [(tid, L.w(tid // NI2, 0, c, tid % NI2)) for tid in range(PB * NI2)]
        yield "p4_ld", ins
    for i in range(NI):
        ins = []
        for tid in range(PB * NI2):
            p, rr = divmod(tid, NI2)
            i1, i0 = divmod(rr, NI)
            ins.append((tid, L.u(p, 1 + i, 1 + i1, 1 + i0)))
        yield "p4_xold", ins


def cost(L: Layout, word: int, detail=False):
    tot = ideal = 0
    per = defaultdict(lambda: [0, 0])
    for name, ins in phases(L):
        warps = defaultdict(list)
        for tid, a in ins:
            warps[tid // 32].append((tid % 32, a))
        for wl in warps.values():
            t, i = wavefronts(wl, word)
            tot += t
            ideal += i
            per[name][0] += t
            per[name][1] += i
    if detail:
        return tot, ideal, dict(per)
    return tot, ideal


def search(K, word, PB, NT):
    NC, NI = 2 * K + 1, 2 * K - 1
    NI2 = NI * NI
    best = None
    for SU1 in range(NC, NC + 3):
        for SU2 in range(NC * SU1, NC * SU1 + 5):
            for UW in range(NC * SU2, NC * SU2 + 8):
                L = Layout(K, PB, NT, UW, SU1, SU2, NC * 2 * NI2, NI2, NC * NI2)
                # U-only phases first (independent of W)
                pass
    # coarse: search U and W parameters separately (their phases are disjoint
    # except p4_xold which only depends on U)
    bestU = None
    # --wide: pads over a whole bank period (16 eight-byte / 32 four-byte banks)
    wU = (16, 16, 24) if WIDE else (3, 5, 9)
    for SU1 in range(NC, NC + wU[0]):
        for SU2 in range(NC * SU1, NC * SU1 + wU[1]):
            for UW in range(NC * SU2, NC * SU2 + wU[2]):
                if WIDE and UW > UW_CAP:
                    continue
                L = Layout(K, PB, NT, UW, SU1, SU2, 2 * NC * NI2, NI2, NC * NI2)
                _, _, per = cost(L, word, detail=True)
                c = sum(per[k][0] for k in ("ldgsts", "p1_ld", "p4_xold"))
                mem = UW
                key = (c, mem)
                if bestU is None or key < bestU[0]:
                    bestU = (key, (UW, SU1, SU2))
    UW, SU1, SU2 = bestU[1]
    bestW = None
    wW = (17, 17, 33) if WIDE else (4, 9, 17)
    for SJ in range(NI2, NI2 + wW[0]):
        for SW in range(NC * SJ, NC * SJ + wW[1]):
            for WW in range(SW + NC * SJ, SW + NC * SJ + wW[2]):
                if WIDE and UW + WW > UW_CAP + WW_CAP:
                    continue
                L = Layout(K, PB, NT, UW, SU1, SU2, WW, SJ, SW)
                _, _, per = cost(L, word, detail=True)
                c = sum(per[k][0] for k in per if k.startswith(("p1_st", "p2", "p3", "p4_ld")))
                key = (c, WW)
                if bestW is None or key < bestW[0]:
                    bestW = (key, (WW, SJ, SW))
    WW, SJ, SW = bestW[1]
    L = Layout(K, PB, NT, UW, SU1, SU2, WW, SJ, SW)
    return L, cost(L, word, detail=True)


WIDE = False
# shared memory per patch (words) the wide search may use: 5 CTAs of PB = 16
# patches per SM need UW + WW <= 354 (f64)
UW_CAP, WW_CAP = 175, 175

if __name__ == "__main__":
    if "--wide" in sys.argv:
        sys.argv.remove("--wide")
        WIDE = True
    K = int(sys.argv[1])
    word = 8 if sys.argv[2] == "f64" else 4
    PB = int(sys.argv[3]) if len(sys.argv) > 3 else {1: 64, 2: 16, 3: 8}[K]
    NC, NI = 2 * K + 1, 2 * K - 1
    NT = ((PB * max(NC, NI * NI) + 31) // 32) * 32
    NI2 = NI * NI
    base = Layout(K, PB, NT, NC ** 3, NC, NC * NC, 2 * NC * NI2 + (3 if K == 2 else 1), NI2, NC * NI2)
    t, i, per = cost(base, word, detail=True)
    print(f"current: total {t} ideal {i}  " + " ".join(f"{k}={v[0]}/{v[1]}" for k, v in per.items()))
    L, (t, i, per) = search(K, word, PB, NT)
    print(f"best: UW={L.UW} SU1={L.SU1} SU2={L.SU2} WW={L.WW} SJ={L.SJ} SW={L.SW}: total {t} ideal {i}  "
          + " ".join(f"{k}={v[0]}/{v[1]}" for k, v in per.items()))
