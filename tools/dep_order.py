"""Slice-order analysis for prefix-level hoisting: from the per-
dependence-mask byte totals of a compile (`TC_DEP_STATS=1`, "[depmask] mask nodes
bytes" lines on stderr), the executed bytes of one pass over all slices when a node
is recomputed only when one of the slice digits it depends on changes, for (a) the
reference's lexicographic order (first chosen index slowest) and (b) the best digit
order (DP over subsets of digits placed slowest-first), and (c) two tiers: the best
k digits as per-block constants, everything else per slice.

    TC_DEP_STATS=1 python tools/one_slice.py c4 2>&1 | grep depmask | sort -u > m.txt
    python tools/dep_order.py m.txt 8
"""
import sys


def main(path, ndig):
    rows = []
    for line in open(path):
        parts = line.split()
        if parts and parts[0] == "[depmask]":
            rows.append((int(parts[1], 16), int(parts[2]), float(parts[3])))
    n = int(ndig)
    ns = 2 ** n
    per_slice = sum(b for _, _, b in rows)
    # (a) lexicographic: digit j changes every 2^(n-1-j) slices -> reps 2^(kmax+1)
    lex = sum(b * 2 ** (max(j for j in range(n) if m >> j & 1) + 1) for m, _, b in rows)
    # (b) best order: f(S) = min_d f(S-d) + w(S, d) * 2^|S|, w = bytes of masks within S containing d
    full = (1 << n) - 1
    INF = float("inf")
    f = [INF] * (1 << n)
    f[0] = 0.0
    arg = [-1] * (1 << n)
    for S in range(1, 1 << n):
        pc = bin(S).count("1")
        for d in range(n):
            if not S >> d & 1:
                continue
            P = S & ~(1 << d)
            w = sum(b for m, _, b in rows if m & ~S == 0 and m >> d & 1)
            c = f[P] + w * 2 ** pc
            if c < f[S]:
                f[S], arg[S] = c, d
    order = []
    S = full
    while S:
        order.append(arg[S])
        S &= ~(1 << arg[S])
    order = order[::-1]  # slowest first
    print(f"per-slice variant bytes {per_slice / 1e9:.2f} GB x {ns} slices = {per_slice * ns / 1e9:.1f} GB/pass")
    print(f"(a) lexicographic order, prefix-level reuse: {lex / 1e9:.1f} GB/pass")
    print(f"(b) best digit order {order} (slowest first): {f[full] / 1e9:.1f} GB/pass")
    for k in range(1, min(n, 5)):
        best = None
        for B in range(1 << n):
            if bin(B).count("1") != k:
                continue
            blk = sum(b for m, _, b in rows if m and m & ~B == 0) * 2 ** k
            rest = sum(b for m, _, b in rows if not (m and m & ~B == 0)) * ns
            if best is None or blk + rest < best[0]:
                best = (blk + rest, [d for d in range(n) if B >> d & 1])
        print(f"(c) {k} block digits {best[1]}: {best[0] / 1e9:.1f} GB/pass")


if __name__ == "__main__":
    main(*sys.argv[1:])
