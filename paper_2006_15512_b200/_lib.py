"""ctypes binding of libtc (``include/tc.h``).

The library is built in-tree (``python -m paper_2006_15512_b200.build``) and
loaded from ``paper_2006_15512_b200/lib/libtc.so``.  There is no fallback: if
the library is missing or was built for another architecture, importing the
execution path raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import errors

LIB_PATH = os.environ.get("TC_LIBTC") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libtc.so")

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)

INT64_MIN = -(2**63)
INT64_MAX = 2**63 - 1


class U128(C.Structure):
    _fields_ = [("lo", C.c_uint64), ("hi", C.c_uint64)]

    def value(self) -> int:
        return int(self.lo) | (int(self.hi) << 64)


class PlanDesc(C.Structure):
    _fields_ = [
        ("num_indices", C.c_int32),
        ("domain", I32P),
        ("sort_rank", I32P),
        ("num_leaves", C.c_int32),
        ("leaf_idx_off", I64P),
        ("leaf_idx", I32P),
        ("leaf_val_off", I64P),
        ("leaf_val", F64P),
        ("num_nodes", C.c_int32),
        ("left", I32P),
        ("right", I32P),
        ("root_slot", C.c_int32),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("num_bonds", C.c_int32),
        ("num_free", C.c_int32),
        ("max_rank", C.c_int32),
        ("root_rank", C.c_int32),
        ("contraction_ops", U128),
        ("mem_cost", U128),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("mem_estimate", U128),
        ("peak_observed", U128),
        ("num_slices", C.c_int64),
        ("device_peak_bytes", C.c_int64),
        ("device_ms", C.c_double),
        ("compile_ms", C.c_double),
        ("gpu_launches", C.c_int64),
        ("n_tiny_nodes", C.c_int32),
        ("n_stream_nodes", C.c_int32),
        ("n_gemm_nodes", C.c_int32),
        ("n_generic_nodes", C.c_int32),
        ("alg_bytes", U128),
        ("alg_flops", U128),
        ("n_alias_nodes", C.c_int32),
        ("n_tied_leaves", C.c_int32),
        ("program_ms", C.c_double),
        ("setup_ms", C.c_double),
        ("graph_ms", C.c_double),
        ("phys_bytes", U128),
        ("phys_flops", U128),
        ("phys_bytes_hoisted", U128),
        ("phys_flops_hoisted", U128),
        ("launches_prologue", C.c_int64),
        ("launches_per_slice", C.c_int64),
        ("pinned_bytes", C.c_int64),
        ("phys_bytes_block", U128),
        ("phys_flops_block", U128),
        ("launches_block", C.c_int64),
        ("slices_per_block", C.c_int64),
    ]

    def as_dict(self):
        return dict(
            mem_estimate=self.mem_estimate.value(),
            peak_observed=self.peak_observed.value(),
            num_slices=int(self.num_slices),
            device_peak_bytes=int(self.device_peak_bytes),
            device_ms=float(self.device_ms),
            compile_ms=float(self.compile_ms),
            gpu_launches=int(self.gpu_launches),
            n_tiny_nodes=int(self.n_tiny_nodes),
            n_stream_nodes=int(self.n_stream_nodes),
            n_gemm_nodes=int(self.n_gemm_nodes),
            n_generic_nodes=int(self.n_generic_nodes),
            alg_bytes=self.alg_bytes.value(),
            alg_flops=self.alg_flops.value(),
            n_alias_nodes=int(self.n_alias_nodes),
            n_tied_leaves=int(self.n_tied_leaves),
            program_ms=float(self.program_ms),
            setup_ms=float(self.setup_ms),
            graph_ms=float(self.graph_ms),
            phys_bytes=self.phys_bytes.value(),
            phys_flops=self.phys_flops.value(),
            phys_bytes_hoisted=self.phys_bytes_hoisted.value(),
            phys_flops_hoisted=self.phys_flops_hoisted.value(),
            launches_prologue=int(self.launches_prologue),
            launches_per_slice=int(self.launches_per_slice),
            phys_bytes_block=self.phys_bytes_block.value(),
            phys_flops_block=self.phys_flops_block.value(),
            launches_block=int(self.launches_block),
            slices_per_block=int(self.slices_per_block),
            pinned_bytes=int(self.pinned_bytes),
        )


class FactorInput(C.Structure):  # include/tc_factor.h
    _fields_ = [
        ("num_tensors", C.c_int32),
        ("idx_off", I64P),
        ("idx", I32P),
        ("val_off", I64P),
        ("val_ptr", C.POINTER(C.c_void_p)),
        ("num_indices", C.c_int32),
        ("domain", I32P),
        ("sort_rank", I32P),
        ("num_nodes", C.c_int32),
        ("adj_off", I64P),
        ("adj", I32P),
        ("str_off", I64P),
        ("str_buf", C.c_char_p),
        ("repr_off", I64P),
        ("repr_buf", C.c_char_p),
        ("num_leaf_map", C.c_int32),
        ("leaf_node", I32P),
        ("leaf_index", I32P),
    ]


class FactorInfo(C.Structure):
    _fields_ = [
        ("trivial", C.c_int32),
        ("branch_width", C.c_int32),
        ("carving_width", C.c_int32),
        ("num_pieces", C.c_int32),
        ("num_bonds", C.c_int32),
        ("total_idx", C.c_int64),
        ("total_val", C.c_int64),
        ("num_nodes", C.c_int32),
        ("root_slot", C.c_int32),
    ]


class DecompInfo(C.Structure):  # include/tc_decompose.h
    _fields_ = [
        ("num_nodes", C.c_int32),
        ("num_adj", C.c_int64),
        ("num_bag", C.c_int64),
        ("num_order", C.c_int32),
        ("num_leaf_map", C.c_int32),
        ("counter_end", C.c_int64),
    ]


# every symbol include/*.h declares, with its ctypes signature
SIGNATURES = {
    "tc_elim_td": (C.c_int, [C.c_int32, I64P, I32P, C.c_int32, C.POINTER(C.c_uint32), C.c_int32, C.c_int64,
                             C.POINTER(C.c_void_p)]),
    "tc_tree_to_branch": (C.c_int, [C.c_int32, I64P, I32P, I32P, I64P, I32P, C.c_int32, C.c_int32, I32P, I32P,
                                    C.c_int64, C.POINTER(C.c_void_p)]),
    "tc_validate_td": (C.c_int, [C.c_int32, I64P, I32P, I64P, I32P, C.c_int32, C.c_int32, I32P, I32P,
                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int8)]),
    "tc_decomp_info_get": (C.c_int, [C.c_void_p, C.POINTER(DecompInfo)]),
    "tc_decomp_fetch": (C.c_int, [C.c_void_p, I32P, I64P, I64P, I32P, I64P, I32P, I32P, I32P, I32P]),
    "tc_decomp_free": (None, [C.c_void_p]),
    "tc_factor_branch": (C.c_int, [C.POINTER(FactorInput), C.POINTER(C.c_void_p)]),
    "tc_factor_info_get": (C.c_int, [C.c_void_p, C.POINTER(FactorInfo)]),
    "tc_factor_fetch": (C.c_int, [C.c_void_p, I32P, I32P, I64P, I32P, I64P, F64P, I32P, I32P, I32P, I32P, I32P]),
    "tc_factor_free": (None, [C.c_void_p]),
    "tc_plan_create": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(C.c_void_p)]),
    "tc_plan_free": (None, [C.c_void_p]),
    "tc_plan_info_get": (C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    "tc_mem_cost": (C.c_int, [C.c_void_p, I32P, C.c_int32, C.POINTER(U128)]),
    "tc_choose_slice_index": (C.c_int, [C.c_void_p, I32P, C.c_int32, I32P]),
    "tc_choose_slices": (C.c_int, [C.c_void_p, C.c_int64, I32P, C.c_int32, I32P, C.POINTER(U128)]),
    "tc_result_indices": (C.c_int, [C.c_void_p, I32P, C.c_int32, I32P, C.c_int32, I32P]),
    "tc_choose_slices_work": (C.c_int, [C.c_void_p, I32P, C.c_int32, C.c_int32, C.c_int64, I32P]),
    "tc_compile_stats": (C.c_int, [C.c_void_p, I32P, C.c_int32, C.c_void_p]),
    "tc_exec_create": (C.c_int, [C.c_void_p, I32P, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "tc_exec_free": (None, [C.c_void_p]),
    "tc_exec_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(Stats)]),
    "tc_exec_run_repeat": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(Stats)]),
    "tc_exec_run_flushed": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.POINTER(Stats)]),
    "tc_exec_copy_results": (C.c_int, [C.c_void_p, C.c_void_p]),
    "tc_fold_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int32]),
    "tc_exec_fetch": (C.c_int, [C.c_void_p, F64P, F64P]),
    "tc_exec_profile": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_float), I32P, I32P, F64P, F64P,
                                  C.c_int32, I32P]),
    "tc_exec_profile_graph": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_float), I32P, I32P, F64P,
                                        F64P, C.c_int32, I32P, C.POINTER(C.c_float)]),
    "tc_exec_result_size": (C.c_int64, [C.c_void_p]),
    "tc_exec_slices_per_block": (C.c_int64, [C.c_void_p]),
    "tc_exec_deps": (C.c_int, [C.c_void_p, I32P, I32P, C.c_int32, I32P, I32P]),
    "tc_sliced_execute": (
        C.c_int,
        [C.c_void_p, C.c_int64, I32P, C.c_int32, I32P, C.c_int32, F64P, C.c_int64, I32P, C.c_int32,
         I32P, I32P, C.c_int32, I32P, C.POINTER(Stats)],
    ),
    "tc_release_cache": (C.c_int, [C.c_int32]),
    "tc_last_error": (C.c_char_p, []),
    "tc_version": (C.c_int32, []),
    "tc_device_count": (C.c_int32, []),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libtc.so not found at {LIB_PATH}: build it with "
                "`python -m paper_2006_15512_b200.build` (there is no CPU fallback)"
            )
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


_STATUS = {
    1: ValueError,
    2: errors.PlanMismatch,
    3: errors.BudgetInfeasible,
    4: errors.NoCandidates,
    5: MemoryError,
    6: errors.DeviceError,
    7: errors.DeviceError,
    8: OverflowError,
    9: errors.IndexOveruse,
    10: errors.NotABondIndex,
}


def check(status: int):
    if status != 0:
        msg = lib().tc_last_error().decode(errors="replace")
        raise _STATUS.get(status, RuntimeError)(msg)


def _p(a, t):
    return a.ctypes.data_as(t)


def ids_ptr(ids):
    a = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
    return a, _p(a, I32P), len(a)


class PlanHandle:
    """Owns a ``tc_plan`` built from a ``flatten.FlatPlan``."""

    def __init__(self, flat):
        self.flat = flat
        L = lib()
        arrays = dict(
            domain=np.ascontiguousarray(flat.domain, dtype=np.int32),
            sort_rank=np.ascontiguousarray(flat.sort_rank, dtype=np.int32),
            leaf_idx_off=np.ascontiguousarray(flat.leaf_idx_off, dtype=np.int64),
            leaf_idx=np.ascontiguousarray(flat.leaf_idx, dtype=np.int32),
            leaf_val_off=np.ascontiguousarray(flat.leaf_val_off, dtype=np.int64),
            leaf_val=np.ascontiguousarray(flat.leaf_val, dtype=np.float64),
            left=np.ascontiguousarray(flat.left, dtype=np.int32),
            right=np.ascontiguousarray(flat.right, dtype=np.int32),
        )
        d = PlanDesc(
            num_indices=len(arrays["domain"]),
            domain=_p(arrays["domain"], I32P),
            sort_rank=_p(arrays["sort_rank"], I32P),
            num_leaves=len(arrays["leaf_idx_off"]) - 1,
            leaf_idx_off=_p(arrays["leaf_idx_off"], I64P),
            leaf_idx=_p(arrays["leaf_idx"], I32P),
            leaf_val_off=_p(arrays["leaf_val_off"], I64P),
            leaf_val=_p(arrays["leaf_val"], F64P),
            num_nodes=len(arrays["left"]),
            left=_p(arrays["left"], I32P),
            right=_p(arrays["right"], I32P),
            root_slot=int(flat.root_slot),
        )
        h = C.c_void_p()
        check(L.tc_plan_create(C.byref(d), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tc_plan_free(self.h)
            self.h = None

    def info(self) -> PlanInfo:
        out = PlanInfo()
        check(lib().tc_plan_info_get(self.h, C.byref(out)))
        return out

    def mem_cost(self, drop_ids) -> int:
        a, p, n = ids_ptr(drop_ids)
        out = U128()
        check(lib().tc_mem_cost(self.h, p, n, C.byref(out)))
        return out.value()

    def choose_slice_index(self, already_ids) -> int:
        a, p, n = ids_ptr(already_ids)
        out = C.c_int32()
        check(lib().tc_choose_slice_index(self.h, p, n, C.byref(out)))
        return int(out.value)

    def compile_stats(self, sliced_ids=()) -> dict:
        """Host-only program compile (no device): class counts, memory model."""
        a, p, n = ids_ptr(sliced_ids)
        st = Stats()
        check(lib().tc_compile_stats(self.h, p, n, C.byref(st)))
        return st.as_dict()

    def choose_slices(self, mem_budget: int):
        """Algorithm 3's greedy (slicing.py:119-128): shortest prefix with
        mem_cost <= mem_budget."""
        cap = max(1, len(self.flat.domain))
        buf = np.zeros(cap, dtype=np.int32)
        n = C.c_int32()
        check(lib().tc_choose_slices(self.h, max(INT64_MIN + 1, min(INT64_MAX, int(mem_budget))), _p(buf, I32P), cap,
                                     C.byref(n), None))
        return buf[: n.value].tolist()

    def choose_slices_work(self, max_entries: int, already=()):
        """Work-aware slice set (extension): picks until every intermediate
        has <= max_entries entries."""
        cap = max(1, len(self.flat.domain))
        buf = np.zeros(cap, dtype=np.int32)
        buf[: len(already)] = list(already)
        n = C.c_int32()
        check(lib().tc_choose_slices_work(self.h, _p(buf, I32P), len(already), cap, int(max_entries), C.byref(n)))
        return buf[: n.value].tolist()

    def result_indices(self, sliced_ids=()):
        a, p, n = ids_ptr(sliced_ids)
        cap = max(1, len(self.flat.domain))
        out = np.zeros(cap, dtype=np.int32)
        r = C.c_int32()
        check(lib().tc_result_indices(self.h, p, n, _p(out, I32P), cap, C.byref(r)))
        return out[: r.value].tolist()

    def _budget_slices(self, mem_budget):
        """The reference's budget loop ``while mem_cost(chosen) > mem_budget``
        (slicing.py:120-128) for any real budget: (explicit slice ids, None) when
        Python decides it (budget met unsliced, non-integral or beyond int64;
        inf / nan never slice), else (None, int64 budget) for libtc's greedy."""
        import math

        mc = self.mem_cost([])
        if not (mc > mem_budget):  # also inf and nan
            return [], INT64_MIN
        fb = math.floor(mem_budget)  # integral costs: cost > b  <=>  cost > floor(b)
        if INT64_MIN < fb <= INT64_MAX and fb == mem_budget:
            return None, int(fb)
        chosen = []
        while self.mem_cost(chosen) > mem_budget:
            try:
                chosen.append(self.choose_slice_index(chosen))
            except errors.NoCandidates:
                bonds = [k for k in range(len(self.flat.domain))
                         if np.count_nonzero(self.flat.leaf_idx == k) == 2]
                raise errors.BudgetInfeasible(f"cannot fit in {mem_budget} bytes even fully sliced "
                                              f"(needs {self.mem_cost(bonds)})") from None
        return chosen, INT64_MIN

    def sliced_execute(self, mem_budget, slice_ids, devices):
        L = lib()
        root = self.result_indices(())
        cap = 1
        for i in root:
            cap *= int(self.flat.domain[i])
        out_val = np.zeros(max(1, cap), dtype=np.float64)
        out_idx = np.zeros(max(1, len(root)), dtype=np.int32)
        rank = C.c_int32()
        nb = max(1, len(self.flat.domain))
        chosen = np.zeros(nb, dtype=np.int32)
        nch = C.c_int32()
        st = Stats()
        budget = INT64_MIN  # None
        if mem_budget is not None and slice_ids is None:
            slice_ids, budget = self._budget_slices(mem_budget)
        if slice_ids is None:
            sa, sp, sn = ids_ptr([])
            sn = -1
        else:
            sa, sp, sn = ids_ptr(slice_ids)
        da, dp, dn = ids_ptr(devices if devices else [0])
        check(L.tc_sliced_execute(self.h, budget, sp, sn, dp, dn, _p(out_val, F64P), len(out_val),
                                  _p(out_idx, I32P), len(out_idx), C.byref(rank), _p(chosen, I32P),
                                  len(chosen), C.byref(nch), C.byref(st)))
        r = rank.value
        idx = out_idx[:r].tolist()
        size = 1
        for i in idx:
            size *= int(self.flat.domain[i])
        return out_val[:size].copy(), idx, chosen[: nch.value].tolist(), st.as_dict()


class Exec:
    """A compiled, HBM-resident program (``tc_exec``) for repeated runs — the
    bench's device-timed arm."""

    def __init__(self, plan: PlanHandle, slice_ids=(), device: int = 0):
        self.plan = plan
        self.slice_ids = list(slice_ids)
        a, p, n = ids_ptr(slice_ids)
        h = C.c_void_p()
        check(lib().tc_exec_create(plan.h, p, n, int(device), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tc_exec_free(self.h)
            self.h = None

    def run(self, begin: int, end: int, repeats: int = 1, flush_bytes: int = 0) -> dict:
        """repeats passes over slices [begin, end); with flush_bytes > 0 each
        pass is timed alone after an untimed L2-evicting write (benchmark)."""
        st = Stats()
        if flush_bytes > 0:
            check(lib().tc_exec_run_flushed(self.h, int(begin), int(end), int(repeats), int(flush_bytes),
                                            C.byref(st)))
        else:
            check(lib().tc_exec_run_repeat(self.h, int(begin), int(end), int(repeats), C.byref(st)))
        return st.as_dict()

    def copy_results(self, dst_device_ptr: int):
        """Per-slice results of the last run -> caller's device buffer."""
        check(lib().tc_exec_copy_results(self.h, C.c_void_p(int(dst_device_ptr))))

    KINDS = ["select", "tiny", "stream", "gemm", "generic", "rootcopy", "eta", "gemm_reduce"]

    def profile(self, slice_id: int = 0):
        """Per-launch (kind, slot, ms, alg_bytes, alg_flops) of one eager slice."""
        cap = 1 << 20
        ms = np.zeros(cap, dtype=np.float32)
        kind = np.zeros(cap, dtype=np.int32)
        slot = np.zeros(cap, dtype=np.int32)
        by = np.zeros(cap, dtype=np.float64)
        fl = np.zeros(cap, dtype=np.float64)
        n = C.c_int32()
        check(lib().tc_exec_profile(self.h, int(slice_id), ms.ctypes.data_as(C.POINTER(C.c_float)), _p(kind, I32P),
                                    _p(slot, I32P), _p(by, F64P), _p(fl, F64P), cap, C.byref(n)))
        k = n.value
        return [dict(kind=self.KINDS[kind[i]], slot=int(slot[i]), ms=float(ms[i]), bytes=float(by[i]),
                     flops=float(fl[i])) for i in range(k)]

    def profile_graph(self, begin: int, end: int):
        """Per-launch graph-mode time over one pass of slices [begin, end):
        (list of dict(kind, inv, ms, bytes, flops), summed pass ms)."""
        cap = 1 << 20
        ms = np.zeros(cap, dtype=np.float32)
        kind = np.zeros(cap, dtype=np.int32)
        inv = np.zeros(cap, dtype=np.int32)
        by = np.zeros(cap, dtype=np.float64)
        fl = np.zeros(cap, dtype=np.float64)
        n = C.c_int32()
        pm = C.c_float()
        check(lib().tc_exec_profile_graph(self.h, int(begin), int(end), ms.ctypes.data_as(C.POINTER(C.c_float)),
                                          _p(kind, I32P), _p(inv, I32P), _p(by, F64P), _p(fl, F64P), cap,
                                          C.byref(n), C.byref(pm)))
        k = n.value
        # runs of each launch in the pass: prologue once, block tier once per block, else per slice
        B = int(lib().tc_exec_slices_per_block(self.h))
        ns = int(end) - int(begin)
        runs = lambda x: 1 if x & 1 else (-(-ns // B) if x & 2 else ns)  # noqa: E731
        return [dict(kind=self.KINDS[kind[i]], inv=bool(inv[i] & 1), blk=bool(inv[i] & 2), runs=runs(int(inv[i])),
                     ms=float(ms[i]), bytes=float(by[i]), flops=float(fl[i]), start_us=int(inv[i] >> 2))
                for i in range(k)], float(pm.value)

    def deps(self):
        """Launch DAG: list of dependency lists (diagnostics)."""
        cap = 1 << 22
        off = np.zeros(cap + 1, dtype=np.int32)
        dd = np.zeros(cap, dtype=np.int32)
        n, m = C.c_int32(), C.c_int32()
        check(lib().tc_exec_deps(self.h, _p(off, I32P), _p(dd, I32P), cap, C.byref(n), C.byref(m)))
        return [dd[off[i]:off[i + 1]].tolist() for i in range(n.value)]

    def result_size(self) -> int:
        return int(lib().tc_exec_result_size(self.h))

    def num_slices(self) -> int:
        n = 1
        for i in self.slice_ids:
            n *= int(self.plan.flat.domain[i])
        return n

    def fetch(self, per_slice_n: int | None = None):
        R = self.result_size()
        folded = np.zeros(R, dtype=np.float64)
        per = None
        if per_slice_n:
            per = np.zeros(per_slice_n * R, dtype=np.float64)
        check(lib().tc_exec_fetch(self.h, _p(per, F64P) if per is not None else None, _p(folded, F64P)))
        return folded, per


def release_cache(device: int = -1):
    """Return libtc's cached HBM blocks of ``device`` (-1: all) to the driver."""
    check(lib().tc_release_cache(int(device)))


def fold_device(per_slice_ptr: int, R: int, n: int, out_ptr: int, device: int):
    """Lexicographic left fold of a [n][R] FP64 device array into out[R]."""
    check(lib().tc_fold_device(C.c_void_p(int(per_slice_ptr)), int(R), int(n), C.c_void_p(int(out_ptr)),
                               int(device)))
