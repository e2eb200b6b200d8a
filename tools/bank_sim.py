"""Shared-memory wavefront simulator for the pass kernel's exchange stages (dev tool).

Replays, for one CTA of fft_pass_kernel<F, T>, the lane -> (t, j) mapping of every
Stockham stage (fft_pass.cuh: fft_stage) and the smem address of each 16-byte access,
and counts wavefronts per warp instruction: a 16-byte access is served per quarter warp
(8 lanes), each quarter costing as many wavefronts as the most-used 16-byte bank group
(distinct addresses only).  Ideal = 4 per instruction.

    python tools/bank_sim.py              # every supported (F, T) of the default plans
"""
import sys

RMAX = 16
RF_MIN = 32


def first_radix(F):
    r = F
    while r > RMAX:
        r //= RMAX
    return r


def remainder_first(F):
    return F >= RF_MIN and first_radix(F) != RMAX


def stage_radix(F, NS):
    if remainder_first(F):
        return first_radix(F) if NS == 1 else RMAX
    return RMAX if F // NS >= RMAX else F // NS


def swz(f):
    return ((f >> 3) ^ (f >> 6) ^ (f >> 9) ^ (f >> 12)) & 7


def pad(T):
    return 0 if T == 1 else (4 if T == 2 else (2 if T == 4 else 1))


def smem_idx(F, T, t, f, sw=swz):
    return t * (F + pad(T)) + (f ^ sw(f))


def stages(F):
    out, NS = [], 1
    while NS < F:
        RS = stage_radix(F, NS)
        out.append((NS, RS))
        NS *= RS
    return out


def wavefronts(addrs):
    """addrs: 32 lane addresses (in 16-byte units) of one warp instruction."""
    w = 0
    for q in range(4):
        groups = {}
        for a in set(addrs[8 * q:8 * q + 8]):
            groups[a % 8] = groups.get(a % 8, 0) + 1
        w += max(groups.values())
    return w


def simulate(F, T, in_tfast, out_tfast, sw_for=None):
    """Returns [(stage, 'rd'|'wr', wavefronts, ideal)] for the smem accesses of one CTA.
    sw_for(e) -> swizzle function of exchange e (written by stage e, read by stage e+1)."""
    R = min(F, RMAX)
    NT = T * F // R
    st = stages(F)
    res = []
    for s, (NS, RS) in enumerate(st):
        NB = F // RS
        M = R // RS
        first, last = s == 0, s == len(st) - 1
        tfast = in_tfast if first else (out_tfast if last else False)
        if T == 1:
            tfast = False
        rd_sw = sw_for(s - 1) if (sw_for and s > 0) else swz
        wr_sw = sw_for(s) if sw_for else swz
        for kind in ("rd", "wr"):
            if kind == "rd" and first:
                continue
            if kind == "wr" and last:
                continue
            tot = ideal = 0
            for warp in range(NT // 32):
                for i in range(M):
                    for r in range(RS):
                        addrs = []
                        for lane in range(32):
                            b = lane + 32 * warp + NT * i
                            t, j = (b % T, b // T) if tfast else (b // NB, b % NB)
                            if kind == "rd":
                                f = j + r * NB
                                addrs.append(smem_idx(F, T, t, f, rd_sw))
                            else:
                                base = (j // NS) * NS * RS + (j % NS)
                                f = base + r * NS
                                addrs.append(smem_idx(F, T, t, f, wr_sw))
                        tot += wavefronts(addrs)
                        ideal += 4
            res.append((s, NS, RS, kind, tot, ideal))
    return res


def swz_ns(NS):
    """Exchange written by a radix-16 stage with NS in {2, 4} (right after a radix-2/4
    remainder stage): the quarter-warp's lanes differ in f bits {0, 5, 6} (NS = 2) or
    {0, 1, 6} (NS = 4); fold bit 6 into the bank bit that swz leaves constant."""
    if NS == 4:
        return lambda f: swz(f) ^ (((f >> 6) & 1) << 2)
    if NS == 2:
        return lambda f: swz(f) ^ (((f >> 6) & 1) << 1)
    return swz


def proposed(F):
    st = stages(F)
    return lambda e: swz_ns(st[e][0]) if e < len(st) else swz

def main():
    cases = [(F, T) for F in (32, 64, 128, 256, 512, 1024, 2048, 4096) for T in (1, 2, 4, 8, 16)
             if F * T <= 8192 and F * T >= 512]
    for F, T in cases:
        for tf in ((False, True), (True, True)):   # row pass (last) / column pass (middle)
            res = simulate(F, T, *tf)
            tot = sum(r[4] for r in res)
            ideal = sum(r[5] for r in res)
            bad = [f"s{r[0]}(NS={r[1]},RS={r[2]}) {r[3]} {r[4] / r[5]:.2f}x" for r in res if r[4] > r[5]]
            print(f"F={F:5d} T={T:2d} {'col' if tf[0] else 'row'}: {tot / ideal:.2f}x ideal  {'; '.join(bad)}")


if __name__ == "__main__":
    sys.exit(main())

