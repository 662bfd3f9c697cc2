"""Symbolic simulation of diagonal-tie propagation (copy-tensor hyperedges) over
a frozen plan: per-node physical shapes, node classes and the dense vs tied
roofline.  Analysis tool only."""
import collections
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_15512_b200 import planfile  # noqa: E402

HBM, FP64 = 6.5e12, 35.5e12


def partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for p in partitions(rest):
        for i in range(len(p)):
            yield p[:i] + [[first] + p[i]] + p[i + 1:]
        yield [[first]] + p


def leaf_blocks(idx, vals, dims):
    r = len(idx)
    if r <= 1 or any(d != 2 for d in dims):
        return [[i] for i in idx]
    v = vals.reshape([2] * r)
    best = None
    for p in partitions(list(range(r))):
        ok = True
        for e in itertools.product(range(2), repeat=r):
            if v[e] != 0 and any(len({e[q] for q in blk}) > 1 for blk in p):
                ok = False
                break
        if ok and (best is None or len(p) < len(best)):
            best = p
    return [[idx[q] for q in blk] for blk in best]


def main(name):
    fl, _ = planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))
    L = fl.num_leaves
    dom = fl.domain
    blocks = []  # per slot: list of frozensets of logical indices
    for l in range(L):
        idx = fl.leaf_idx[fl.leaf_idx_off[l]:fl.leaf_idx_off[l + 1]].tolist()
        vals = fl.leaf_val[fl.leaf_val_off[l]:fl.leaf_val_off[l + 1]]
        blocks.append([frozenset(b) for b in leaf_blocks(idx, vals, [dom[i] for i in idx])])
    dense = dict(t=0.0, flops=0.0, bytes=0.0)
    tied = dict(t=0.0, flops=0.0, bytes=0.0)
    cls = collections.Counter()
    clst = collections.defaultdict(float)
    maxr = 0
    for k in range(fl.num_nodes):
        a, b = fl.left[k], fl.right[k]
        A, B = blocks[a], blocks[b]
        la = set().union(*A) if A else set()
        lb = set().union(*B) if B else set()
        shared = la & lb
        kept = la ^ lb
        # dense
        ra, rb, rc, ru = len(la), len(lb), len(kept), len(la | lb)
        db = 8 * (2 ** ra + 2 ** rb + 2 ** rc)
        df = 2 * 2 ** ru
        dense["t"] += max(db / HBM, df / FP64)
        # tied: union-find over blocks
        parent = {}

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x
        nodes = [("a", q) for q in range(len(A))] + [("b", q) for q in range(len(B))]
        for n in nodes:
            parent[n] = n
        owner = {}
        for q, blk in enumerate(A):
            for i in blk:
                owner.setdefault(i, []).append(("a", q))
        for q, blk in enumerate(B):
            for i in blk:
                owner.setdefault(i, []).append(("b", q))
        for i, ows in owner.items():
            for o in ows[1:]:
                ra_, rb_ = find(ows[0]), find(o)
                if ra_ != rb_:
                    parent[ra_] = rb_
        comps = collections.defaultdict(lambda: dict(a=0, b=0, idx=set()))
        for n in nodes:
            c = comps[find(n)]
            c[n[0]] += 1
            c["idx"] |= (A if n[0] == "a" else B)[n[1]]
        newb = []
        nM = nN = nK = nB = 0
        diag = False
        for c in comps.values():
            kp = c["idx"] & kept
            if c["a"] > 1 or c["b"] > 1:
                diag = True
            if kp:
                newb.append(frozenset(kp))
                if c["a"] and c["b"]:
                    nB += 1
                elif c["a"]:
                    nM += 1
                else:
                    nN += 1
            else:
                nK += 1
        blocks.append(newb)
        pa, pb, pc = len(A), len(B), len(newb)
        tb = 8 * (2 ** pa + 2 ** pb + 2 ** pc)
        tf = 2 * 2 ** len(comps)
        tt = max(tb / HBM, tf / FP64)
        tied["t"] += tt
        maxr = max(maxr, pc)
        if max(pa, pb, pc) <= 12:
            kind = "tiny"
        elif min(pa, pb) <= 3 and nK <= 4:
            kind = "stream" + ("+batch" if nB else "") + ("+diag" if diag else "")
            if pc == max(pa, pb) and not diag and nK == 0 and min(pa, pb) <= nB:
                kind = "elementwise(batch-only)"
        else:
            kind = "gemm" + ("+batch" if nB else "") + ("+diag" if diag else "")
        cls[kind] += 1
        clst[kind] += tt
    print(f"{name}: dense roofline {dense['t'] * 1e3:.2f} ms, tied roofline {tied['t'] * 1e3:.2f} ms, "
          f"max phys rank {maxr}")
    for kd, n in cls.most_common():
        print(f"   {kd:28s} n={n:6d}  roof {clst[kd] * 1e3:8.3f} ms")


if __name__ == "__main__":
    for n in sys.argv[1:]:
        main(n)
