"""Benchmark of the B200 execution stage (Algorithm 3 of arXiv 2006.15512).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one execution of the frozen contraction plan of the workload (all
of its slices): the plan comes from the unmodified reference planner
(tools/make_plans.py, data/plans/<config>.tcplan.npz), inputs are resident in
HBM before the timed region.  Metric: slices/s (whole job); for the default
unsliced config C2 one slice = one formula, so ms_per_step is the
per-formula execution time.

N > 1 (torchrun, one process per GPU):
  * sliced configs (c4, c5, c3): the lexicographic slice ids are block-
    partitioned over ranks, one NCCL all-reduce combines them (strong scaling);
  * unsliced configs (c1a, c1b, c2): the path does not shard -> N independent
    replicas, no collective (weak scaling).

``--impl reference`` times the unmodified reference ``sliced_execute``
(tensorcount from oracle/_ref, numpy/OpenBLAS on the host cores) on the same
plan; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
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

# workload -> (description, greedy slice-prefix rule)
GiB = 2 ** 30
# Sliced configs use Algorithm 3 itself: the reference's greedy (exact port) at a
# mem_budget (the reference's dense memory model decides the slice set).  The
# literal "2^8 / 2^12 slices" of BASELINE.json are restated in DESIGN.md §5: on
# these FactorTree spine plans every greedy pick nearly doubles total work, while
# tie-aware execution fits C4 unsliced and C3 at two slices in one B200's HBM.
CONFIGS = {
    "c1a": dict(desc="uniform random 3-CNF n=30 ratio 3.0 (restated C1), unsliced"),
    "c1b": dict(desc="uniform random 3-CNF n=40 ratio 3.0 (restated C1), max-rank 30, unsliced"),
    "c2": dict(desc="banded random 3-CNF n=200 ratio 3.5 window 29 (C2), max-rank 26, unsliced"),
    "c1b_s3": dict(plan="c1b", budget=int(3.5 * GiB),
                   desc="C1b sliced by Algorithm 3 at mem_budget 3.5 GiB (greedy: 3 picks, 8 slices)"),
    "c4": dict(budget=100 * GiB,
               desc="banded random 3-CNF n=400 ratio 4.0 window 36 (C4) at mem_budget 100 GiB (2 picks, 4 slices)"),
    "c4_full": dict(plan="c4", desc="banded random 3-CNF n=400 ratio 4.0 window 36 (C4), unsliced "
                                    "(192 GiB dense mem_cost; 18 GB of tied tensors on the device)"),
    "c3": dict(budget=270 * GiB,
               desc="grid Ising 30x30 (C3), 393 GiB unsliced, at mem_budget 270 GiB (1 pick, 2 slices)"),
    "c5": dict(budget=100 * GiB, infeasible="reference greedy plateaus at 3 TiB per slice after 12 picks",
               desc="banded random 3-CNF n=400 ratio 4.0 window 44 (C5), 12 TiB unsliced"),
}


L2_FLUSH_BYTES = 512 * 2 ** 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def load_plan(config):
    from paper_2006_15512_b200 import planfile

    name = CONFIGS.get(config, {}).get("plan", config)
    return planfile.load(os.path.join(ROOT, "data", "plans", f"{name}.tcplan.npz"))


def sliced_max_rank(flat, chosen):
    ch = set(chosen)
    L = flat.num_leaves
    sets = [frozenset(flat.leaf_idx[flat.leaf_idx_off[k]:flat.leaf_idx_off[k + 1]].tolist()) - ch for k in range(L)]
    best = max((len(s) for s in sets), default=0)
    for l, r in zip(flat.left.tolist(), flat.right.tolist()):
        s = sets[l] ^ sets[r]
        sets.append(s)
        best = max(best, len(s))
    return best


def choose_slices(flat, config):
    from paper_2006_15512_b200 import _lib

    import ctypes

    spec = CONFIGS[config]
    h = _lib.PlanHandle(flat)
    if "infeasible" in spec:
        raise SystemExit(f"config {config}: {spec['infeasible']}")
    if "budget" not in spec:
        return h, []
    buf = np.zeros(max(1, len(flat.domain)), np.int32)
    n = ctypes.c_int32()
    _lib.check(_lib.lib().tc_choose_slices(h.h, spec["budget"], buf.ctypes.data_as(_lib.I32P), len(buf),
                                           ctypes.byref(n), None))
    return h, buf[: n.value].tolist()


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every ~0.5 ms on a thread (the timed region of a fast
    config lasts only milliseconds); nvidia-smi as a fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
    # nvmlClocksEventReason* bits
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
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = get_reasons(self.h)
                self.rows.append((sm, rs))
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


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak_tflops(device):
    """cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 5 — the FP64
    tensor denominator (absent from MEASURED_PEAKS.json)."""
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


def roofline(prof, ms_per_slice, hbm, fp64):
    """Dominant kernel class + whole-tree roofline."""
    cls = {}
    t_roof = 0.0
    for p in prof:
        c = cls.setdefault(p["kind"], dict(ms=0.0, bytes=0.0, flops=0.0, launches=0))
        c["ms"] += p["ms"]
        c["bytes"] += p["bytes"]
        c["flops"] += p["flops"]
        c["launches"] += 1
        t_roof += max(p["bytes"] / (hbm * 1e9), p["flops"] / (fp64 * 1e12)) * 1e3
    tot = sum(c["ms"] for c in cls.values())
    dom = max(cls, key=lambda k: cls[k]["ms"])
    d = cls[dom]
    if dom in ("gemm",):
        ach = d["flops"] / (d["ms"] / 1e3) / 1e12
        ro = dict(bound="tensor", achieved=ach, peak=fp64, unit="TFLOP/s", frac=ach / fp64)
    else:
        ach = d["bytes"] / (d["ms"] / 1e3) / 1e9
        ro = dict(bound="hbm", achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm)
    ro.update(kernel=f"k_{dom}", share_of_step=d["ms"] / tot if tot else None, launches_per_slice=d["launches"])
    classes = {k: dict(ms=v["ms"], share=v["ms"] / tot if tot else None,
                       gbs=v["bytes"] / v["ms"] / 1e6 if v["ms"] else None,
                       tflops=v["flops"] / v["ms"] / 1e9 if v["ms"] else None, launches=v["launches"])
               for k, v in cls.items()}
    tree = dict(t_roof_ms=t_roof, measured_ms=ms_per_slice, frac=t_roof / ms_per_slice if ms_per_slice else None,
                note="T_roof = sum over nodes max(bytes/HBM, flops/FP64) per slice (SURVEY 8d)")
    return ro, classes, tree


def dense_tree_roofline_ms(flat, chosen, hbm, fp64):
    """T_roof per slice = sum over EVERY internal node of
    max(8(|A|+|B|+|C|)/BW_HBM, 2*prod(union dims)/P_FP64) (dense, unfused)."""
    ch = set(chosen)
    L = flat.num_leaves
    sets = [frozenset(flat.leaf_idx[flat.leaf_idx_off[k]:flat.leaf_idx_off[k + 1]].tolist()) - ch for k in range(L)]
    dom = flat.domain
    logd = {}

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
        by = 8.0 * (size(a) + size(b) + size(c))
        fl = 2.0 * size(a | b)
        t += max(by / (hbm * 1e9), fl / (fp64 * 1e12))
    del logd
    return t * 1e3


def traffic_for(config, kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(config, {})
    # a launch class can span kernel families (stream: k_stream + fused k_stream_pair)
    fams = {"k_stream": ("k_stream", "k_stream_pair", "k_stream_seq")}.get(kernel, (kernel,))
    vals = [d[f]["dram_bytes_per_slice"] for f in fams if f in d and "dram_bytes_per_slice" in d[f]]
    return sum(vals) if vals else None


# ---------------------------------------------------------------- reference
def _reference_path():
    for p in (os.path.join(ROOT, "oracle", "_ref"), os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "tensorcount")):
            if p not in sys.path:
                sys.path.insert(0, p)
            return p
    raise ImportError("reference not installed (oracle/_ref or baseline/_ref)")


def reference_objects(flat):
    _reference_path()
    from tensorcount.network import ContractionTree, TensorNetwork
    from tensorcount.tensor import Index, Tensor

    from paper_2006_15512_b200 import planfile

    flat_r = planfile.FlatPlan(**{**flat.__dict__, "indices": [Index(ix.id, ix.domain_size) for ix in flat.indices]})
    return planfile.to_objects(flat_r, Tensor, TensorNetwork, ContractionTree)


def time_reference(flat, chosen, steps, warm=True):
    """The unmodified reference sliced_execute on this plan.  Unsliced: the
    full run per step.  Sliced: slice 0 through the reference's own slice code
    path (_slice_plan + _execute_tracked, slicing.py:139-145), extrapolated x
    num_slices."""
    _reference_path()
    from tensorcount import slicing as ref_slicing
    from tensorcount.tensor import Assignment

    n, t = reference_objects(flat)
    if warm:
        ref_slicing.sliced_execute(*reference_objects(load_plan("c1a")[0]))
    times = []
    count = None
    nsl = 1
    for i in chosen:
        nsl *= int(flat.domain[i])
    for _ in range(steps):
        t0 = time.perf_counter()
        if not chosen:
            out = ref_slicing.sliced_execute(n, t)
            count = float(np.asarray(out.result.values).reshape(-1)[0])
        else:
            idx = [n_ix for n_ix in _ref_indices(n, flat, chosen)]
            eta = Assignment(zip(idx, [0] * len(idx)))
            m, plan = ref_slicing._slice_plan(n, t, eta)
            ref_slicing._execute_tracked(m, plan)
        times.append(time.perf_counter() - t0)
    per_step = statistics.median(times) * (nsl if chosen else 1)
    sample = ("full unsliced sliced_execute per step" if not chosen else
              f"slice 0 of {nsl} via _slice_plan+_execute_tracked, extrapolated x{nsl}")
    return per_step, nsl, sample, count, times


def _ref_indices(n, flat, chosen):
    want = {flat.indices[i].id for i in chosen}
    found = {}
    for ten in n.tensors:
        for ix in ten.indices:
            if ix.id in want:
                found[ix.id] = ix
    return [found[flat.indices[i].id] for i in chosen]


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    flat, meta = load_plan(args.config)
    chosen = []
    if "budget" in CONFIGS[args.config]:
        _, chosen = choose_slices(flat, args.config)
    steps = max(1, min(args.steps, args.ref_steps))
    per_step, nsl, sample, count, times = time_reference(flat, chosen, steps)
    value = nsl / per_step
    line = dict(metric=METRIC, value=value, unit=UNIT, impl="reference", n_gpus=args.gpus, steps=steps,
                warmup=1, ms_per_step=per_step * 1e3, higher_is_better=True,
                scaling="strong" if chosen else "weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=args.config, desc=CONFIGS[args.config]["desc"], num_slices=nsl,
                            sliced_indices=len(chosen), plan=f"data/plans/{args.config}.tcplan.npz"),
                cpu_baseline=dict(value=value, unit=UNIT, cores=host_cores(), kind="reference", sample=sample),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                count=count, step_seconds=times,
                note="unmodified tensorcount (oracle/_ref) numpy/OpenBLAS on host cores; steps capped by --ref-steps")
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours
def run_ours(args):
    import torch

    from paper_2006_15512_b200 import _lib, planfile, sliced_execute
    from paper_2006_15512_b200.distributed import fold, gather_slices, slice_block

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    flat, meta = load_plan(args.config)
    h, chosen = choose_slices(flat, args.config)
    nsl = 1
    for i in chosen:
        nsl *= int(flat.domain[i])
    sharded = bool(chosen) and world > 1
    b, e = slice_block(nsl, world, rank) if sharded else (0, nsl)
    ex = _lib.Exec(h, chosen, local)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        ex.run(b, e)
    barrier()
    # each timed pass follows an untimed 512 MiB write that evicts the 126 MB L2
    # (tied C2 intermediates total ~85 MB and would otherwise stay L2-resident)
    with ClockSampler(local) as clk:
        st = ex.run(b, e, repeats=args.steps, flush_bytes=L2_FLUSH_BYTES)
    barrier()
    dev_ms = st["device_ms"]
    if world > 1:
        t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    # sliced: the whole job's slices per step; unsliced: N replicas of the formula
    slices_per_step = nsl if chosen else world
    value = slices_per_step / (ms_per_step / 1e3)

    # result of the last pass (all ranks): fold per-slice results
    per = torch.zeros((e - b, ex.result_size()), dtype=torch.float64, device="cuda")
    ex.copy_results(per.data_ptr())
    if sharded:
        full = gather_slices(per, b, nsl)
        count_t = fold(full)
    else:
        count_t = fold(per)
    count = float(count_t[0].item())

    # per-launch eager profile (rank 0) while the program is resident, then free
    # it: the e2e leg below builds its own (C4 needs ~100 GiB per program)
    prof = ex.profile(b) if rank == 0 else None
    d2h = 8 * ex.result_size()
    del ex
    # end to end through the public API: host objects -> flatten -> C-ABI ->
    # H2D leaves/plan -> device run -> D2H result
    n_obj, t_obj = planfile.to_objects(flat)
    slice_objs = [flat.indices[i] for i in chosen]
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier()
    if not sharded:
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = sliced_execute(n_obj, t_obj, slice_indices=slice_objs if chosen else None, devices=[local])
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        e2e_count = float(np.asarray(res.result.values).reshape(-1)[0])
    else:
        from paper_2006_15512_b200.flatten import flatten

        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fl = flatten(n_obj, t_obj)
            hh = _lib.PlanHandle(fl)
            ids = [fl.indices.index(ix) for ix in slice_objs]
            ex2 = _lib.Exec(hh, ids, local)
            ex2.run(b, e)
            p2 = torch.zeros((e - b, ex2.result_size()), dtype=torch.float64, device="cuda")
            ex2.copy_results(p2.data_ptr())
            e2e_count = float(fold(gather_slices(p2, b, nsl))[0].item())
            del ex2
        e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = slices_per_step / e2e_s
    h2d = int(flat.leaf_val.nbytes + flat.leaf_idx.nbytes + flat.leaf_idx_off.nbytes + flat.leaf_val_off.nbytes
              + flat.left.nbytes + flat.right.nbytes + flat.domain.nbytes + flat.sort_rank.nbytes)

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    # roofline from the eager per-launch replay of slice b (CUDA events per launch)
    hbm, hbm_src = measured_peaks()
    fp64 = fp64_peak_tflops(torch.device("cuda", local))
    ms_per_slice = ms_per_step / max(1, (e - b) if chosen else 1)
    ro, classes, tree = roofline(prof, ms_per_slice, hbm, fp64)
    t_dense = dense_tree_roofline_ms(flat, chosen, hbm, fp64)
    tree = dict(t_roof_ms=t_dense, measured_ms_per_slice=ms_per_slice, frac=t_dense / ms_per_slice,
                t_roof_phys_ms=tree["t_roof_ms"], frac_phys=tree["t_roof_ms"] / ms_per_slice,
                note="t_roof_ms: SURVEY 8d dense per-node roofline over all nodes of one slice (the reference's "
                     "dense tensors), HBM=%s GB/s, FP64=%.2f TF/s (cuBLAS DGEMM, live); frac > 1 means faster than "
                     "any dense execution.  t_roof_phys_ms: the same roofline over the launched kernels' own work "
                     "(tied physical tensors; aliases are free) - the bound for this program" % (hbm, fp64))
    ro["peak_source"] = ("cuBLAS DGEMM 8192^3 measured live in bench.py (FP64 is not in MEASURED_PEAKS.json)"
                         if ro["bound"] == "tensor" else hbm_src)
    ro["traffic"] = traffic_for(args.config, ro["kernel"])
    ro["alg_bytes"] = classes_bytes = sum(p["bytes"] for p in prof if "k_" + p["kind"] == ro["kernel"])
    ro["scope"] = "per slice, summed over every launch of this kernel class (achieved = alg work / summed CUDA-event time)"
    ro["traffic_note"] = ("ncu dram__bytes_read+write summed over the class's launches of one slice "
                          "(profiles/ncu_traffic.json)" if ro["traffic"] else None)
    del classes_bytes

    counts_path = os.path.join(ROOT, "tests", "golden", "counts.json")
    golden = (json.load(open(counts_path)).get(CONFIGS[args.config].get("plan", args.config))
              if os.path.exists(counts_path) else None)
    parity = None
    if golden:  # the slice sum equals the unsliced reference count (Thm 5)
        parity = dict(reference_count=golden["count"], rel_err=abs(count - golden["count"]) / abs(golden["count"]))

    cpu = None
    dense_gib = st["mem_estimate"] / GiB
    if world == 1 and not args.no_cpu_baseline and dense_gib > 24:
        cpu = dict(value=None, unit=UNIT, cores=host_cores(), kind="reference",
                   sample=f"not run: the reference's dense working set per slice is {dense_gib:.0f} GiB")
    elif world == 1 and not args.no_cpu_baseline:
        try:
            per_step, _, sample, ref_count, times = time_reference(flat, chosen, 1)
            cpu = dict(value=nsl / per_step, unit=UNIT, cores=host_cores(), kind="reference", sample=sample,
                       seconds=per_step)
            if ref_count is not None:
                cpu["count"] = ref_count
                cpu["rel_err_vs_gpu"] = abs(ref_count - count) / abs(ref_count) if ref_count else None
        except Exception as ex_:  # the reference is not importable on this box
            cpu = dict(value=None, unit=UNIT, cores=host_cores(), kind="reference", sample=f"unavailable: {ex_}")

    line = dict(
        metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=ms_per_step, higher_is_better=True,
        scaling="strong" if sharded else "weak", vs_baseline=None, dtype="f64", data="synthetic",
        config=dict(workload=args.config, desc=CONFIGS[args.config]["desc"], num_slices=nsl,
                    sliced_indices=len(chosen), slices_per_rank=e - b, plan=f"data/plans/{args.config}.tcplan.npz",
                    parallelism=(f"slices/{world}" if sharded else f"replicas x{world}"),
                    l2="L2 flushed before every timed pass (untimed 512 MiB write)"),
        e2e=dict(value=e2e_value, unit=UNIT, seconds_per_step=e2e_s, h2d_bytes_per_step=h2d, d2h_bytes_per_step=d2h,
                 path="sliced_execute(n, t) public API" if not sharded else "flatten -> C-ABI plan/exec -> run -> fetch"),
        gpu_launches=st["gpu_launches"],
        roofline=ro, roofline_classes=classes, tree_roofline=tree,
        cpu_baseline=cpu,
        clocks=clk.summary(),
        count=count, e2e_count=e2e_count, parity=parity,
        compile_ms=st["compile_ms"], device_peak_bytes=st["device_peak_bytes"],
        work=dict(dense_bytes=st["alg_bytes"], dense_flops=st["alg_flops"], phys_bytes=st["phys_bytes"],
                  phys_flops=st["phys_flops"], tied_leaves=st["n_tied_leaves"], aliases=st["n_alias_nodes"]),
        nodes=dict(tiny=st["n_tiny_nodes"], stream=st["n_stream_nodes"], gemm=st["n_gemm_nodes"],
                   generic=st["n_generic_nodes"]),
    )
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-steps", type=int, default=3)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
