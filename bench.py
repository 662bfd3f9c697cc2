"""Benchmark of the B200 execution stage (Algorithm 3 of arXiv 2006.15512).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

A step is one pass of the frozen contraction plan of the workload over its
slices (data/plans/<config>.tcplan.npz, planned by the unmodified reference
planner, tools/make_plans.py); leaves and program are resident in HBM before
the timed region.  Metric: slices/s of the whole job (all ranks).

Default workload: C4 (BASELINE configs[3]: "random 3-CNF n=400, ratio 4.0,
width ~36 sliced into 2^8 slices across 1/2/4/8 B200") = banded_3cnf(400,
4.0, 36, seed 11) (the first SAT seed), slice set = Algorithm 3's greedy
8-pick prefix (slicing.py:70-79) -> 2^8 slices.  The line also carries C2
(configs[1], unsliced, 1 B200) device and end-to-end numbers under "c2", and the whole
count of C2 from DIMACS text (native planning + FactorTree + GPU execution) under
"c2" -> "pipeline".

N > 1: one process per GPU (torchrun; ``python bench.py --gpus N`` launches
it itself).  Sliced configs block-partition the lexicographic slice ids over
the ranks and meet in ONE NCCL all-reduce (strong scaling); unsliced configs
(c1a, c1b, c2, c4_full) run N replicas (weak scaling, no collective).

``--impl reference`` times the reference's own CPU implementation on the
host cores (tensorcount from baseline/_ref or oracle/_ref, numpy/OpenBLAS):
the full unmodified ``sliced_execute`` where it fits (c1a, c2), else a
bounded, labelled sample of its per-node ``contract_pair`` work extrapolated
to the whole job (see ``reference_sample_model``).
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "WMC execution time & slices/sec (B200 execution stage, arXiv 2006.15512)"
UNIT = "slices/s"
GiB = 2 ** 30
L2_FLUSH_BYTES = 512 * 2 ** 20

# workload -> plan, slice rule, optional per-rank sample of slices, description
CONFIGS = {
    "c1a": dict(plan="c1a", slices=None, desc="uniform random 3-CNF n=30 ratio 3.0 (restated C1), unsliced"),
    "c1b": dict(plan="c1b", slices=None, desc="uniform random 3-CNF n=40 ratio 3.0 (restated C1), max-rank 30, unsliced"),
    "c2": dict(plan="c2", slices=None,
               desc="banded random 3-CNF n=200 ratio 3.5 window 29 seed 1 (C2), max-rank 26, unsliced"),
    "c4": dict(plan="c4", slices=("greedy", 8),
               desc="banded random 3-CNF n=400 ratio 4.0 window 36 seed 11 (C4; seeds 1-10 UNSAT), max-rank 37, "
                    "Algorithm 3 greedy 8-pick prefix -> 2^8 slices of max-rank 33"),
    "c1b_s3": dict(plan="c1b", slices=("greedy", 3),
                   desc="C1b with Algorithm 3's greedy 3-pick prefix (8 slices): a small sliced case for tests"),
    "c4_full": dict(plan="c4", slices=None,
                    desc="C4 unsliced (2.5 TiB dense mem_cost; 10.6 GB of tied tensors on the device)"),
    "c5": dict(plan="c5", slices=("greedy", 12), sample=512, sample_at_end=True,
               desc="banded random 3-CNF n=400 ratio 4.0 window 34 seed 6 (C5; seeds 1-5 UNSAT), max-rank 34, "
                    "Algorithm 3 greedy 12-pick prefix -> 2^12 slices of max-rank 30; the last 512 slices of each "
                    "rank's block are timed (the whole job at 8 GPUs; all 44 non-zero slices lie in 3184-4083)"),
    "c3": dict(plan="c3", slices=("work", 28), sample=256,
               desc="grid Ising 30x30 (C3), max-rank 35, sliced to rank 28 by the work-aware chooser (30 indices, "
                    "2^30 slices; the greedy plateaus at rank 34); a block of 256 slices per rank is timed"),
}
DEFAULT = "c4"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def load_plan(name):
    from paper_2006_15512_b200 import planfile

    return planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))


def choose(flat, rule):
    """Slice set of a config (indices into flat.indices, pick order)."""
    from paper_2006_15512_b200 import _lib

    h = _lib.PlanHandle(flat)
    if rule is None:
        return h, []
    kind, k = rule
    if kind == "greedy":  # the reference greedy's k-pick prefix (slicing.py:70-79)
        ch = []
        for _ in range(k):
            ch.append(h.choose_slice_index(ch))
        return h, ch
    return h, h.choose_slices_work(2 ** k)


def num_slices(flat, chosen):
    ns = 1
    for i in chosen:
        ns *= int(flat.domain[i])
    return ns


def rank_block(ns, world, rank, sample, at_end=False):
    """This rank's contiguous block of lexicographic slice ids, or a sample of
    `sample` slices at its start (or end) when the job is timed by sample."""
    per = -(-ns // world)
    b = min(ns, rank * per)
    e = min(ns, b + per)
    if sample:
        if at_end:
            b = max(b, e - sample)
        else:
            e = min(e, b + sample)
    return b, e


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every ~0.5 ms on a thread; nvidia-smi as a fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self.stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM), get_reasons(self.h)))
            except Exception:
                pass
            time.sleep(0.0005)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        if self.nvml is not None:
            sm = [float(r[0]) for r in self.rows]
            reasons = sorted({k for _, rs in self.rows for k, b in self.BITS.items() if rs & b})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(self.max_sm), "reasons": reasons,
                    "samples": len(self.rows), "source": "nvml, polled during the timed region"}
        busy = [r for r in self.rows if r[6].isdigit() and int(r[6]) > 0] or self.rows
        sm = [float(r[0]) for r in busy if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in busy for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(busy[0][1]) if busy[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(busy), "source": "nvidia-smi"}


def measured_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak_tflops(device):
    """cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 5 — the FP64
    tensor-pipe denominator (MEASURED_PEAKS.json holds no FP64 figure)."""
    import torch

    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    for _ in range(2):
        torch.matmul(a, b)
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * n ** 3 / (best / 1e3) / 1e12


def dense_slice_roofline_ms(flat, chosen, hbm, fp64):
    """per slice, sum over EVERY internal node of
    max(8(|A|+|B|+|C|)/BW_HBM, 2*prod(union dims)/P_FP64) over the reference's
    dense tensors (unfused, no ties, no hoisting)."""
    ch = set(chosen)
    dom = flat.domain
    off = flat.leaf_idx_off
    sets = [frozenset(flat.leaf_idx[off[k]:off[k + 1]].tolist()) - ch for k in range(flat.num_leaves)]

    def size(s):
        z = 1
        for i in s:
            z *= int(dom[i])
        return z

    t = 0.0
    for l, r in zip(flat.left.tolist(), flat.right.tolist()):
        a, b = sets[l], sets[r]
        c = a ^ b
        sets.append(c)
        t += max(8.0 * (size(a) + size(b) + size(c)) / (hbm * 1e9), 2.0 * size(a | b) / (fp64 * 1e12))
    return t * 1e3


def classes_from_profile(prof, n_slices, hbm, fp64):
    """Kernel classes of one pass over n_slices (graph-mode per-launch CUDA
    events): time, executed bytes/flops, achieved rates."""
    cls = {}
    for p in prof:
        c = cls.setdefault(p["kind"], dict(ms=0.0, bytes=0.0, flops=0.0, launches=0))
        mult = p["runs"]  # prologue once, block tier once per block, else per slice
        c["ms"] += p["ms"]
        c["bytes"] += p["bytes"] * mult
        c["flops"] += p["flops"] * mult
        c["launches"] += mult
    tot = sum(c["ms"] for c in cls.values())
    out = {}
    for k, v in cls.items():
        out[k] = dict(ms=v["ms"], share=v["ms"] / tot if tot else None, launches=v["launches"],
                      gbs=v["bytes"] / v["ms"] / 1e6 if v["ms"] else None,
                      tflops=v["flops"] / v["ms"] / 1e9 if v["ms"] else None, bytes=v["bytes"], flops=v["flops"])
    dom = max(out, key=lambda k: out[k]["ms"])
    d = out[dom]
    if dom == "gemm":
        ro = dict(bound="tensor", achieved=d["tflops"], peak=fp64, unit="TFLOP/s", frac=d["tflops"] / fp64)
    else:
        ro = dict(bound="hbm", achieved=d["gbs"], peak=hbm, unit="GB/s", frac=d["gbs"] / hbm)
    ro.update(kernel="k_" + dom, share_of_step=d["share"], launches_per_pass=d["launches"],
              alg_bytes_per_pass=d["bytes"], alg_flops_per_pass=d["flops"])
    return ro, out


def traffic_for(config, kernel, n_slices):
    """ncu DRAM bytes (read + write) of the kernel class over one pass of
    n_slices slices: hoisted (prologue) traffic once + per-slice traffic x
    n_slices (profiles/ncu_traffic.json, tools/ncu_r2.sh)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(config, {})
    fams = {"k_stream": ("k_stream", "k_stream_pair"), "k_gemm": ("k_gemm", "k_splitk_reduce")}.get(kernel, (kernel,))
    tot, seen = 0, False
    for f in fams:
        if f in d and "dram_bytes_per_slice" in d[f]:
            seen = True
            tot += d[f].get("dram_bytes_prologue", 0) + n_slices * d[f]["dram_bytes_per_slice"]
    return tot if seen else None


# ---------------------------------------------------------------- reference
def _reference_path():
    for p in (os.path.join(ROOT, "baseline", "_ref"), os.path.join(ROOT, "oracle", "_ref")):
        if os.path.isdir(os.path.join(p, "tensorcount")):
            if p not in sys.path:
                sys.path.insert(0, p)
            return p
    raise ImportError("reference not installed (baseline/_ref or oracle/_ref)")


def reference_objects(flat):
    _reference_path()
    from tensorcount.network import ContractionTree, TensorNetwork
    from tensorcount.tensor import Index, Tensor

    from paper_2006_15512_b200 import planfile

    flat_r = planfile.FlatPlan(**{**flat.__dict__, "indices": [Index(ix.id, ix.domain_size) for ix in flat.indices]})
    return planfile.to_objects(flat_r, Tensor, TensorNetwork, ContractionTree)


def _ref_indices(n, flat, chosen):
    want = {flat.indices[i].id for i in chosen}
    found = {}
    for ten in n.tensors:
        for ix in ten.indices:
            if ix.id in want:
                found[ix.id] = ix
    return [found[flat.indices[i].id] for i in chosen]


def ref_node_table(flat, chosen):
    """Operand / result index lists of every internal node of the sliced tree
    in the reference's order: slice_tensor keeps the remaining indices in
    order (tensor.py:118-125); contract_pair emits kept_a ++ kept_b
    (tensor.py:102-108)."""
    ch = set(chosen)
    off = flat.leaf_idx_off
    orders = [[i for i in flat.leaf_idx[off[k]:off[k + 1]].tolist() if i not in ch] for k in range(flat.num_leaves)]
    nodes = []
    for l, r in zip(flat.left.tolist(), flat.right.tolist()):
        a, b = orders[l], orders[r]
        sa, sb = set(a), set(b)
        orders.append([i for i in a if i not in sb] + [i for i in b if i not in sa])
        nodes.append((l, r, len(orders) - 1))
    return orders, nodes


def reference_sample_model(flat, chosen, budget_s=20.0, cap_log2=25, seed=0):
    """A bounded sample of the reference's CPU work for one slice and its
    extrapolation to the whole tree (for plans whose dense per-slice working
    set cannot run on the host: C3-C5).

    The reference executes a slice as one ``contract_pair`` (tensor.py:96-108,
    numpy tensordot: transpose copies + OpenBLAS dgemm) per internal node
    (slicing.py:91-109), and re-executes the whole tree per slice
    (slicing.py:139-145).  Nodes are grouped in classes by log2 of their dense
    bytes; in decreasing order of the classes' share of the nominal cost
    max(bytes / 1 GB/s, flops / 100 GFLOP/s), up to three nodes per class (with
    tensors of <= 2^cap_log2 entries) are timed through the reference's own
    contract_pair on random operands of the nodes' exact index shapes and
    orders, until ``budget_s`` is spent.  Every node is then charged its
    class's measured seconds per nominal unit (classes not sampled: the
    nearest sampled class, i.e. the largest one for nodes above the cap)."""
    _reference_path()
    from tensorcount.tensor import Index, Tensor, contract_pair

    dom = flat.domain.tolist()
    orders, nodes = ref_node_table(flat, chosen)

    def size(o):
        z = 1
        for i in o:
            z *= dom[i]
        return z

    info = []
    for (l, r, c) in nodes:
        sa, sb = set(orders[l]), set(orders[r])
        na, nb, nc, nu = size(orders[l]), size(orders[r]), size(orders[c]), size(sa | sb)
        info.append((8.0 * (na + nb + nc), 2.0 * nu, max(na, nb, nc), l, r))
    cost = [max(by / 1e9, fl / 1e11) for by, fl, _, _, _ in info]
    bins = {}
    for k, (by, _, _, _, _) in enumerate(info):
        bins.setdefault(int(math.log2(max(by, 8.0))), []).append(k)
    share = {b: sum(cost[k] for k in ks) for b, ks in bins.items()}
    rng = np.random.default_rng(seed)
    idx = [Index(ix.id, int(d)) for ix, d in zip(flat.indices, dom)]
    ratio = {}
    t_start = time.perf_counter()
    sampled = 0
    for b in sorted(bins, key=lambda b: -share[b]):
        ks = [k for k in bins[b] if info[k][2] <= (1 << cap_log2)]
        if not ks:
            continue
        picks = list(dict.fromkeys(ks[(len(ks) - 1) * j // 2] for j in range(3)))
        rs = []
        for k in picks:
            if time.perf_counter() - t_start > budget_s and ratio:
                break
            _, _, _, l, r = info[k]
            A = Tensor(tuple(idx[i] for i in orders[l]), rng.random([dom[i] for i in orders[l]]))
            B = Tensor(tuple(idx[i] for i in orders[r]), rng.random([dom[i] for i in orders[r]]))
            reps, t0 = 0, time.perf_counter()
            while True:
                contract_pair(A, B)
                reps += 1
                el = time.perf_counter() - t0
                if el > 0.02 or reps >= 200:
                    break
            rs.append(el / reps / cost[k])
            sampled += 1
        if rs:
            ratio[b] = statistics.median(rs)
        if time.perf_counter() - t_start > budget_s:
            break
    keys = sorted(ratio)
    total = 0.0
    for b, ks in bins.items():
        rt = ratio[b] if b in ratio else ratio[min(keys, key=lambda x: (abs(x - b), -x))]
        total += rt * sum(cost[k] for k in ks)
    return dict(seconds_per_slice=total, sampled_nodes=sampled, nodes=len(nodes), size_classes=len(bins),
                sampled_classes=len(ratio), sample_seconds=time.perf_counter() - t_start)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def time_reference_full(flat, steps):
    """The unmodified reference sliced_execute (unsliced plans) per step."""
    _reference_path()
    from tensorcount import slicing as ref_slicing

    n, t = reference_objects(flat)
    times, count = [], None
    for _ in range(steps):
        t0 = time.perf_counter()
        out = ref_slicing.sliced_execute(n, t)
        times.append(time.perf_counter() - t0)
        count = float(np.asarray(out.result.values).reshape(-1)[0])
    return statistics.median(times), count, times


REF_FULL = ("c1a", "c2")  # configs whose reference run fits a bench step (seconds)


def reference_baseline(config, flat, chosen, steps, budget_s):
    """(slices/s, cpu_baseline dict) of the reference CPU path."""
    ns = num_slices(flat, chosen)
    if config in REF_FULL:
        sec, count, times = time_reference_full(flat, steps)
        out = dict(kind="reference", cores=host_cores(), seconds_per_slice=sec, count=count,
                   step_seconds=times, sample="the full unmodified sliced_execute (slicing.py:112-146) per step")
        try:  # also one BLAS thread
            from threadpoolctl import threadpool_limits

            with threadpool_limits(limits=1):
                sec1, _, _ = time_reference_full(flat, 1)
            out["one_thread"] = dict(cores=1, seconds_per_slice=sec1, value=1.0 / sec1)
        except Exception as ex_:
            out["one_thread"] = dict(unavailable=str(ex_))
        return 1.0 / sec, out
    runs = [reference_sample_model(flat, chosen, budget_s=budget_s, seed=s) for s in range(steps)]
    sec = statistics.median(r["seconds_per_slice"] for r in runs)
    r0 = runs[0]
    return 1.0 / sec, dict(
        kind="reference", cores=host_cores(), seconds_per_slice=sec, extrapolated=True,
        job_seconds=sec * ns,
        sample=(f"EXTRAPOLATED: the reference contract_pair (tensor.py:96-108) timed on {r0['sampled_nodes']} nodes "
                f"from {r0['sampled_classes']} of {r0['size_classes']} size classes of one slice's "
                f"{r0['nodes']}-node tree (random operands of the nodes' shapes, {r0['sample_seconds']:.0f} s "
                f"of CPU), charged per class to every node, x {ns} slices (slicing.py:139-145 re-executes "
                f"the tree per slice); the dense per-slice working set "
                f"({'%.0f' % (_dense_mem_gib(flat, chosen))} GiB) rules out running a slice"),
        model_runs=runs)


def _dense_mem_gib(flat, chosen):
    from paper_2006_15512_b200 import _lib

    return _lib.PlanHandle(flat).mem_cost(chosen) / GiB


def all_host_threads():
    """BLAS thread pools at every host core (torchrun exports OMP_NUM_THREADS=1)."""
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(limits=host_cores())
    except Exception:
        import contextlib

        return contextlib.nullcontext()


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    with all_host_threads():
        _run_reference(args)


def _run_reference(args):
    spec = CONFIGS[args.config]
    flat, _ = load_plan(spec["plan"])
    _, chosen = choose(flat, spec["slices"])
    steps = max(1, min(args.steps, args.ref_steps))
    value, cpu = reference_baseline(args.config, flat, chosen, steps, args.ref_budget)
    ns = num_slices(flat, chosen)
    line = dict(metric=METRIC, value=value, unit=UNIT, impl="reference", n_gpus=args.gpus, steps=steps, warmup=0,
                ms_per_step=ns / value * 1e3, higher_is_better=True, scaling="strong" if chosen else "weak",
                vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=args.config, desc=spec["desc"], num_slices=ns, sliced_indices=len(chosen),
                            plan=f"data/plans/{spec['plan']}.tcplan.npz"),
                cpu_baseline=dict(cpu, value=value, unit=UNIT),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                note="unmodified tensorcount (baseline/_ref) numpy/OpenBLAS on the host cores, rank 0 only")
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- parity
def golden_parity(config, flat, chosen, b, per_slice, count):
    """Compare the GPU's per-slice values of slices [b, b+len) (and the folded
    count of a whole job) with the committed goldens."""
    out = {}
    gp = os.path.join(ROOT, "tests", "golden")
    spec = CONFIGS[config]
    if spec["slices"] is None:
        c = json.load(open(os.path.join(gp, "counts.json"))).get(spec["plan"])
        if spec["plan"] == "c4":
            c = json.load(open(os.path.join(gp, "sliced.json")))["c4"]
        if c:
            out = dict(reference_count=c["count"], source=c.get("count_source", "reference sliced_execute"),
                       rel_err=abs(count - c["count"]) / abs(c["count"]))
        return out
    sl = json.load(open(os.path.join(gp, "sliced.json"))).get(config, {})
    dp_path = os.path.join(gp, f"sliced_dp_{config}.json")
    want = {}
    if os.path.exists(dp_path):
        vals = json.load(open(dp_path))["values"]
        want = {s: v for s, v in enumerate(vals)}
        src = "oracle/wmc_dp.c (exact counter, sliced variables fixed)"
    elif sl.get("slices"):
        want = {int(s): r["value"] for s, r in sl["slices"].items()}
        srcs = {r.get("source") for r in sl["slices"].values()}
        src = ("unmodified reference _execute_tracked(*_slice_plan(n, t, eta)) (slicing.py:30-41, 91-109)"
               if srcs == {"reference"} else "oracle/wmc_dp.c (exact counter, sliced variables fixed)")
    errs = []
    for k, v in enumerate(per_slice):
        s = b + k
        if s in want:
            w = want[s]
            errs.append(0.0 if (v == 0 and w == 0) else abs(v - w) / max(abs(w), 1e-300))
    if errs:
        out = dict(slices_checked=len(errs), max_rel_err=max(errs), source=src,
                   nonzero_slices=sum(1 for k, v in enumerate(per_slice) if v != 0.0))
    if count is not None and "count" in sl:
        out.update(reference_count=sl["count"], count_source=sl.get("count_source"),
                   rel_err=abs(count - sl["count"]) / abs(sl["count"]))
    elif count is not None:  # a whole sliced job of a plan with a reference count (Thm 5: the slice sum)
        c = json.load(open(os.path.join(gp, "counts.json"))).get(spec["plan"])
        if c:
            out.update(reference_count=c["count"], count_source="reference sliced_execute (unsliced)",
                       rel_err=abs(count - c["count"]) / abs(c["count"]))
    return out


# ---------------------------------------------------------------- ours
def device_run(flat, h, chosen, b, e, steps, warmup, local):
    from paper_2006_15512_b200 import _lib

    ex = _lib.Exec(h, chosen, local)
    for _ in range(warmup):
        ex.run(b, e)
    return ex


def run_ours(args):
    import torch

    from paper_2006_15512_b200 import _lib, distributed, planfile, sliced_execute

    world, rank, local = dist_env()
    # TC_BENCH_SHARE_GPU=1 (test only): ranks share the visible GPUs round-robin
    # and meet over gloo (NCCL rejects two ranks on one device) -- exercises
    # the sharded path on a one-GPU box; its timings are not scaling numbers
    share = os.environ.get("TC_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cdev = "cpu" if share else "cuda"

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(t)
        return float(t.item())

    spec = CONFIGS[args.config]
    flat, meta = load_plan(spec["plan"])
    h, chosen = choose(flat, spec["slices"])
    ns = num_slices(flat, chosen)
    sliced = bool(chosen)
    sample = args.sample if args.sample is not None else spec.get("sample")
    b, e = rank_block(ns, world, rank, sample, spec.get("sample_at_end", False)) if sliced else (0, 1)
    whole_job = not sliced or (sample is None) or allsum(e - b) == ns
    ex = device_run(flat, h, chosen, b, e, args.steps, args.warmup, local)
    barrier()
    with ClockSampler(local) as clk:
        st = ex.run(b, e, repeats=args.steps, flush_bytes=L2_FLUSH_BYTES)
    barrier()
    dev_ms = allmax(st["device_ms"])
    ms_per_step = dev_ms / args.steps
    slices_per_step = int(allsum(e - b)) if sliced else world
    value = slices_per_step / (ms_per_step / 1e3)

    # per-slice results of the last pass; whole job: gather + lexicographic fold
    # libtc copies on its own stream: no pending torch-stream write on the buffer
    per = torch.empty((e - b, ex.result_size()), dtype=torch.float64, device="cuda")
    torch.cuda.current_stream().synchronize()
    ex.copy_results(per.data_ptr())
    count = None
    if sliced and whole_job:
        full = distributed.gather_slices(per, b, ns) if world > 1 else per
        count = float(distributed.fold(full)[0].item())
    elif not sliced:
        count = float(per[0, 0].item())
    per_host = per[:, 0].cpu().numpy().tolist()
    parity = golden_parity(args.config, flat, chosen, b, per_host, count) if rank == 0 else None

    # graph-mode per-launch profile of a short pass (rank 0)
    hbm, hbm_src = measured_hbm()
    prof, prof_pass_ms, n_prof = None, None, None
    if rank == 0:
        n_prof = min(e - b, 4) if sliced else 1
        prof, prof_pass_ms = ex.profile_graph(b, b + n_prof)
    d2h = 8 * ex.result_size()
    del ex
    torch.cuda.synchronize()
    _lib.release_cache(local)

    # end to end through the public API: host objects -> flatten -> C-ABI ->
    # H2D leaves/plan -> device run -> D2H result
    n_obj, t_obj = planfile.to_objects(flat)
    slice_objs = [flat.indices[i] for i in chosen] if sliced else None
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier()
    rng = None if whole_job else ((b, e) if world == 1 else (0, slices_per_step))
    def e2e_call():
        if world == 1:
            return sliced_execute(n_obj, t_obj, slice_indices=slice_objs, devices=[local], slice_range=rng)
        if sliced:
            return distributed.sliced_execute(n_obj, t_obj, slice_indices=slice_objs, device=local,
                                              slice_range=None if whole_job else (0, slices_per_step))
        return sliced_execute(n_obj, t_obj, devices=[local])

    # one untimed warm-up call (the W warm-up steps of the device leg, applied here):
    # the first call after the device leg released the cache re-allocates the arena
    e2e_call()
    gc.collect()
    barrier()
    e2e_each = []
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        t1 = time.perf_counter()
        res = e2e_call()
        e2e_count = float(np.asarray(res.result.values).reshape(-1)[0])
        e2e_each.append(time.perf_counter() - t1)
    e2e_s = allmax((time.perf_counter() - t0) / e2e_steps)
    e2e_value = slices_per_step / e2e_s
    h2d = int(flat.leaf_val.nbytes + flat.leaf_idx.nbytes + flat.leaf_idx_off.nbytes + flat.leaf_val_off.nbytes
              + flat.left.nbytes + flat.right.nbytes + flat.domain.nbytes + flat.sort_rank.nbytes)
    _lib.release_cache(local)

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    fp64 = fp64_peak_tflops(torch.device("cuda", local))
    ro, classes = classes_from_profile(prof, n_prof, hbm, fp64)
    ro["peak_source"] = ("cuBLAS DGEMM 8192^3 measured live in bench.py (MEASURED_PEAKS.json has no FP64 figure)"
                         if ro["bound"] == "tensor" else hbm_src)
    ro["traffic"] = traffic_for(args.config, ro["kernel"], n_prof)
    ro["traffic_scope"] = (f"ncu dram__bytes_read+write of the class over a pass of {n_prof} slice(s) (hoisted launches "
                           "once), cold caches, profiles/ncu_traffic.json; compare with alg_bytes_per_pass")
    ro["scope"] = (f"graph-mode CUDA events around every launch of the class over one pass of {n_prof} slice(s) "
                   f"(hoisted launches once); achieved = executed bytes (flops) / summed launch time")
    # whole-step executed-work fraction: every launched kernel's own work per step
    slices_rank = e - b
    B = max(1, int(st.get("slices_per_block", 1)))  # the timed pass's block size
    runs_step = lambda p: 1 if p["inv"] else (-(-slices_rank // B) if p["blk"] else slices_rank)  # noqa: E731
    by_step = sum(p["bytes"] * runs_step(p) for p in prof)
    fl_step = sum(p["flops"] * runs_step(p) for p in prof)
    t_step_s = ms_per_step / 1e3 / (slices_per_step / max(1, slices_rank)) if sliced else ms_per_step / 1e3
    step_roof = dict(executed_bytes_per_rank_step=by_step, executed_flops_per_rank_step=fl_step,
                     achieved_gbs=by_step / (ms_per_step / 1e3) / 1e9, hbm_peak=hbm,
                     frac=max(by_step / (hbm * 1e9), fl_step / (fp64 * 1e12)) / (ms_per_step / 1e3),
                     note="max(executed bytes / HBM peak, executed flops / FP64 peak) / measured step time, "
                          "rank 0's share of the step; ties, fusion and hoisting make the executed work smaller "
                          "than the reference's dense work (see work_reduction)")
    t_dense = dense_slice_roofline_ms(flat, chosen, hbm, fp64) * slices_rank
    work_red = dict(dense_roofline_ms_per_rank_step=t_dense, measured_ms=ms_per_step,
                    ratio=t_dense / ms_per_step,
                    note="SURVEY 8d dense per-node roofline of the reference's tensors (every node, every slice) / "
                         "measured step: a work-reduction ratio (tie compression, hoisting), NOT a roofline fraction")
    del t_step_s

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            with all_host_threads():
                v, cpu = reference_baseline(args.config, flat, chosen, 1, args.ref_budget)
            cpu = dict(cpu, value=v, unit=UNIT)
            if cpu.get("count") is not None and count:
                cpu["rel_err_vs_gpu"] = abs(cpu["count"] - count) / abs(cpu["count"])
        except Exception as ex_:
            cpu = dict(value=None, unit=UNIT, cores=host_cores(), kind="reference", sample=f"unavailable: {ex_}")

    c2 = None
    if args.config == DEFAULT and not args.no_c2 and world == 1:
        c2 = c2_numbers(args, local)
        c2["pipeline"] = pipeline_numbers(local)

    line = dict(
        metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=ms_per_step, higher_is_better=True,
        scaling="strong" if sliced else "weak", vs_baseline=None, dtype="f64", data="synthetic",
        config=dict(workload=args.config, desc=spec["desc"], num_slices=ns, sliced_indices=len(chosen),
                    slices_per_step=slices_per_step, slices_per_rank=e - b,
                    whole_job=whole_job, plan=f"data/plans/{spec['plan']}.tcplan.npz",
                    parallelism=(f"slices/{world}" if sliced else f"replicas x{world}"),
                    l2="L2 flushed before every timed pass (untimed 512 MiB write)"),
        e2e=dict(value=e2e_value, unit=UNIT, seconds_per_step=e2e_s, seconds_each=[round(x, 5) for x in e2e_each],
                 warmup_calls=1, h2d_bytes_per_step=h2d, d2h_bytes_per_step=d2h,
                 path=("sliced_execute(n, t, slice_indices=..., devices=[d]" + (", slice_range=...)" if rng else ")")
                       if world == 1 else "distributed.sliced_execute (per-rank block, NCCL all-reduce, fold)")),
        gpu_launches=st["gpu_launches"],
        roofline=ro, roofline_classes=classes, step_roofline=step_roof, work_reduction=work_red,
        fp64_peak_tflops=fp64, fp64_peak_source="cuBLAS DGEMM 8192^3, live",
        cpu_baseline=cpu,
        clocks=clk.summary(),
        count=count, e2e_count=e2e_count, parity=parity,
        compile_ms=st["compile_ms"], device_peak_bytes=st["device_peak_bytes"],
        hoisting=dict(launches_prologue=st["launches_prologue"], launches_per_slice=st["launches_per_slice"],
                      phys_bytes_hoisted=st["phys_bytes_hoisted"], phys_bytes_per_slice=st["phys_bytes"],
                      pinned_bytes=st["pinned_bytes"], launches_block=st["launches_block"],
                      phys_bytes_block=st["phys_bytes_block"], slices_per_block=st["slices_per_block"],
                      note="prologue launches run once per pass, block-tier launches once per block of "
                           "slices_per_block consecutive slices (nodes not depending on the last chosen index), "
                           "the rest per slice"),
        work=dict(dense_bytes_per_slice=st["alg_bytes"], dense_flops_per_slice=st["alg_flops"],
                  phys_bytes_per_slice=st["phys_bytes"], phys_flops_per_slice=st["phys_flops"],
                  tied_leaves=st["n_tied_leaves"], aliases=st["n_alias_nodes"]),
        nodes=dict(tiny=st["n_tiny_nodes"], stream=st["n_stream_nodes"], gemm=st["n_gemm_nodes"],
                   generic=st["n_generic_nodes"]),
    )
    if c2:
        line["c2"] = c2
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def c2_numbers(args, local):
    """C2 (BASELINE configs[1], unsliced, 1 B200): device-timed pass and e2e
    through the public API, carried in the default line."""
    import torch

    from paper_2006_15512_b200 import _lib, planfile, sliced_execute

    flat, _ = load_plan("c2")
    h, _ = choose(flat, None)
    ex = _lib.Exec(h, [], local)
    for _ in range(args.warmup):
        ex.run(0, 1)
    torch.cuda.synchronize()
    st = ex.run(0, 1, repeats=max(args.steps, 10), flush_bytes=L2_FLUSH_BYTES)
    ms = st["device_ms"] / max(args.steps, 10)
    folded, _ = ex.fetch()
    del ex
    n, t = planfile.to_objects(flat)
    sliced_execute(n, t, devices=[local])  # untimed warm-up call
    gc.collect()
    each = []
    t0 = time.perf_counter()
    for _ in range(5):
        t1 = time.perf_counter()
        res = sliced_execute(n, t, devices=[local])
        each.append(time.perf_counter() - t1)
    e2e = (time.perf_counter() - t0) / 5
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "counts.json")))["c2"]["count"]
    return dict(desc=CONFIGS["c2"]["desc"], value=1e3 / ms, unit=UNIT, ms_per_step=ms,
                e2e=dict(value=1.0 / e2e, unit=UNIT, seconds_per_step=e2e, seconds_each=[round(x, 5) for x in each],
                         path="sliced_execute(n, t) public API (host objects, H2D, D2H)"),
                count=float(folded[0]), rel_err_vs_reference=abs(float(folded[0]) - gold) / gold,
                gpu_launches=st["gpu_launches"])


def pipeline_numbers(local, config="c2"):
    """The whole count of one formula from DIMACS text through the reference's
    own driver (``tensorcount.count_text``, driver.py:254-256, alpha=0) with
    ``reference_patch.install``: the reduction, min-fill planning,
    tree_to_branch and FactorTree native (identical plan), execution on the GPU
    (the unmodified pipeline: profiles/r2_pipeline.jsonl)."""
    try:
        _reference_path()
        import tensorcount
        from tensorcount.network import serialize_plan  # noqa: F401  (reference installed)
    except Exception as ex_:
        return dict(unavailable=str(ex_))
    from paper_2006_15512_b200 import reference_patch
    from paper_2006_15512_b200.generators import config_dimacs

    text = config_dimacs(config)
    reference_patch.install(tensorcount, devices=[local])
    try:
        times, res = [], None
        for _ in range(3):
            t0 = time.perf_counter()
            res = tensorcount.count_text(text, alpha=0.0)
            times.append(time.perf_counter() - t0)
    finally:
        reference_patch.uninstall()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "counts.json")))[config]["count"]
    return dict(config=config, seconds=min(times), count=res.count,
                rel_err_vs_reference=abs(res.count - gold) / abs(gold) if gold else None,
                width=res.width, max_rank=res.max_rank, num_plans=res.num_plans,
                path="tensorcount.count_text(text, alpha=0) + reference_patch.install: reduce / plan / "
                     "FactorTree native (C++), execution on the GPU",
                reference_seconds_box=20.8, reference_source="profiles/r2_pipeline.jsonl (unmodified "
                                                             "tensorcount: reduce 0.06 + plan 3.24 + execute 17.46 s)")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT, choices=sorted(CONFIGS))
    ap.add_argument("--sample", type=int, default=None, help="slices per rank to time (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-steps", type=int, default=3)
    ap.add_argument("--ref-budget", type=float, default=20.0, help="seconds of reference CPU work per sample")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch ourselves under torchrun
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
