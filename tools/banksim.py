"""Shared-memory bank model of the flux kernel's node loads (rhs2.cuh, line_swap / line_coords).

An LDS.64 of a warp is served per half-warp: the sixteen 8-byte addresses of a half fall into 16
eight-byte bank slots (address mod 16 doubles), and the half takes as many wavefronts as the largest
number of distinct addresses sharing one slot.  This model reproduces the ncu source-page counts of the
partner-state and metric loads (4 wavefronts per instruction at N = 9 with the lattice layout).

For each direction pass k (lines along eta_{k+1}) it counts the wavefronts of the partner loads of
every warp slot and shift s, for the line orderings (swap of the two fixed line coordinates), the
choice of line group the masked lanes mirror, and optional padded node layouts
i = a + SB b + SC c.  usage: python tools/banksim.py [N]"""
import collections
import sys


def wavefronts_half(addrs):
    tot = 0
    for h in (addrs[:16], addrs[16:]):
        sl = collections.defaultdict(set)
        for a in h:
            if a is not None:
                sl[a % 16].add(a)
        tot += max([len(v) for v in sl.values()] + [1])
    return tot


def pass_wavefronts(N, k, swap, mirror, SB=None, SC=None):
    SB = N if SB is None else SB
    SC = N * N if SC is None else SC
    LPW = 32 // N
    NL = N * N
    slots = (NL + LPW - 1) // LPW
    t = 0
    for slot in range(slots):
        for s in range(1, N // 2 + 1):
            addrs = []
            for lane in range(32):
                grp, pos = lane // N, lane % N
                if grp >= LPW:
                    grp = mirror
                L = slot * LPW + grp
                if L >= NL:
                    addrs.append(None)
                    continue
                l0, l1 = (L // N, L % N) if swap else (L % N, L // N)
                a, b, c = ((pos, l0, l1), (l0, pos, l1), (l0, l1, pos))[k]
                node = [a, b, c]
                node[k] = (pos + s) % N
                addrs.append(node[0] + SB * node[1] + SC * node[2])
            t += wavefronts_half(addrs)
    return t


def main():
    Ns = [int(sys.argv[1])] if len(sys.argv) > 1 else list(range(3, 10))
    for N in Ns:
        LPW = 32 // N
        rows = []
        for k in range(3):
            opts = {(sw, mi): pass_wavefronts(N, k, sw, mi) for sw in (0, 1) for mi in (0, LPW - 1)}
            rows.append((k, min(opts.items(), key=lambda kv: kv[1]), opts))
        print(f"N={N} (ideal {2 * ((N * N + LPW - 1) // LPW) * (N // 2)} per pass)")
        for k, best, opts in rows:
            print(f"  k={k} best (swap, mirror)={best[0]} -> {best[1]}   all: {opts}")


if __name__ == "__main__":
    main()
