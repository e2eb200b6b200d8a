"""Shared-memory wavefront check for the 4096-point persistent pass (bigpass.cu) (dev tool).

A tile is T = 2 transforms of 4096 points, 512 threads of 16 points, three radix-16
Stockham stages.  The exchange buffer X holds half of the positions of both transforms:
exchange 1 (stage 1 -> 2) splits positions into rounds by bit 3 ^ bit 11 (slot = p with
bit 11 dropped), exchange 2 (stage 2 -> 3) by bit 4 ^ bit 8 (slot = p with bit 8
dropped).  Every thread writes 8 and reads 8 values per round, its write and read sets
in a round are the SAME register indices (round choice s1 = tid bit 8, s2 = tid bit 5 --
warp-uniform), so no value is held twice.  Address: t*2048 + (q ^ swz(q) ^ 5t).
Checks: bijective slots, equal write/read register sets, warp-uniform rounds, and
16-byte wavefronts per quarter-warp (ideal 4 per warp instruction) for every access.

    python tools/bank_sim_big.py
"""


def swz(q):
    return ((q >> 3) ^ (q >> 6) ^ (q >> 9)) & 7


def wavefronts(addrs):
    w = 0
    for qq in range(4):
        groups = {}
        for a in set(a for a in addrs[8 * qq:8 * qq + 8] if a is not None):
            groups.setdefault(a % 8, set()).add(a)
        w += max((len(v) for v in groups.values()), default=0)
    return w


def m13(tid):
    return tid & 1, tid >> 1


def m2(tid):
    j = ((tid >> 1) & 7) | (((tid >> 8) & 1) << 3) | (((tid >> 5) & 1) << 4) | (((tid >> 4) & 1) << 5) \
        | (((tid >> 6) & 1) << 6) | (((tid >> 7) & 1) << 7)
    return tid & 1, j


def slot(p, drop):
    return (p & ((1 << drop) - 1)) | ((p >> (drop + 1)) << drop)


def addr(t, p, drop):
    q = slot(p, drop)
    return t * 2048 + (q ^ swz(q) ^ (5 * t))


EX = {
    # name: (round(p), drop bit, writer map, writer pos(j, r), reader map, reader pos, r-bit, s(tid))
    "E1": (lambda p: ((p >> 3) ^ (p >> 11)) & 1, 11, m13, lambda j, r: 16 * j + r, m2, lambda j, r: j + 256 * r, 3,
           lambda tid: (tid >> 8) & 1),
    "E2": (lambda p: ((p >> 4) ^ (p >> 8)) & 1, 8, m2, lambda j, r: (j // 16) * 256 + j % 16 + 16 * r, m13,
           lambda j, r: j + 256 * r, 0, lambda tid: (tid >> 5) & 1),
}


def check():
    for m in (m13, m2):
        assert sorted(m(i) for i in range(512)) == [(t, j) for t in range(2) for j in range(256)]
    worst = {}
    for name, (rnd, drop, mw, wpos, mr, rpos, rb, s) in EX.items():
        for R in (0, 1):
            assert sorted(slot(p, drop) for p in range(4096) if rnd(p) == R) == list(range(2048))
        for tid in range(512):
            (tw, jw), (tr, jr) = mw(tid), mr(tid)
            assert tw == tr
            for R in (0, 1):
                wr = [r for r in range(16) if rnd(wpos(jw, r)) == R]
                rr = [r for r in range(16) if rnd(rpos(jr, r)) == R]
                blk = [r for r in range(16) if ((r >> rb) & 1) == (s(tid) ^ R)]
                assert wr == rr == blk, (name, tid, R)
        for warp in range(16):
            lanes = range(32 * warp, 32 * warp + 32)
            assert len({s(i) for i in lanes}) == 1
            for R in (0, 1):
                for k in range(8):
                    wa, ra = [], []
                    for tid in lanes:
                        t, j = mw(tid)
                        wa.append(addr(t, [wpos(j, r) for r in range(16) if rnd(wpos(j, r)) == R][k], drop))
                        t, j = mr(tid)
                        ra.append(addr(t, [rpos(j, r) for r in range(16) if rnd(rpos(j, r)) == R][k], drop))
                    worst[name + "W"] = max(worst.get(name + "W", 0), wavefronts(wa))
                    worst[name + "R"] = max(worst.get(name + "R", 0), wavefronts(ra))
    # stage-1 reads of the staging buffer: column tiles S[f*2 + t], row tiles S[t*4100 + f]
    for kind, sa in (("Scol", lambda t, f: 2 * f + t), ("Srow", lambda t, f: t * 4100 + f)):
        for warp in range(16):
            for r in range(16):
                a = []
                for tid in range(32 * warp, 32 * warp + 32):
                    t, j = m13(tid)
                    a.append(sa(t, j + 256 * r))
                worst[kind] = max(worst.get(kind, 0), wavefronts(a))
    return worst


if __name__ == "__main__":
    print(check())
