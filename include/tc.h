/*
 * tc.h — C-ABI of libtc, the B200 execution stage for tensor-network weighted
 * model counting (arXiv 2006.15512).
 *
 * The reference path being replaced is pure Python (tensorcount):
 *   sliced_execute        pkg/src/tensorcount/slicing.py:112-146  (Algorithm 3)
 *   _execute_tracked      pkg/src/tensorcount/slicing.py:91-109   (Algorithm 2 + accounting)
 *   mem_cost              pkg/src/tensorcount/slicing.py:52-67
 *   choose_slice_index    pkg/src/tensorcount/slicing.py:70-79
 *   _slice_plan/slice_tensor  slicing.py:30-41, tensor.py:118-125
 *   execute               pkg/src/tensorcount/network.py:151-163
 *   contract_pair         pkg/src/tensorcount/tensor.py:96-108
 *   add (slice sum)       pkg/src/tensorcount/tensor.py:111-115
 * It is bound from Python with ctypes (paper_2006_15512_b200/_lib.py); see
 * INTEGRATION.md for the binding a tensorcount maintainer would add.
 *
 * Conventions
 *  - All arrays are caller-owned, read-only for the duration of the call;
 *    libtc copies what it needs.  No C++ exception crosses this boundary;
 *    every entry point returns a tc_status.  tc_last_error() gives the message
 *    of the last failure on the calling thread.
 *  - Index ids are dense 0..num_indices-1.  sort_rank[i] is the rank of the
 *    reference's Index.sort_key() (tensor.py:35-37) and is the greedy
 *    tie-break (slicing.py:73-79).
 *  - Leaf values are FP64, row-major, first listed index slowest
 *    (tensor.py:1-5, 55-62).  Operand slots: slot < num_leaves is leaf `slot`
 *    (network order), slot >= num_leaves is internal node slot-num_leaves,
 *    internal nodes listed in postorder (network.py:114-124) — the numbering
 *    of serialize_plan (network.py:235-258).
 *  - Byte sizes of the memory model are 128-bit (reference uses Python ints;
 *    sizes reach 2^76 on real plans).
 */
#ifndef TC_H_
#define TC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tc_status {
  TC_OK = 0,
  TC_BAD_ARG = 1,            /* -> ValueError                         */
  TC_PLAN_MISMATCH = 2,      /* -> PlanMismatch   (network.py:143-148) */
  TC_BUDGET_INFEASIBLE = 3,  /* -> BudgetInfeasible (slicing.py:124-128) */
  TC_NO_CANDIDATES = 4,      /* -> NoCandidates   (slicing.py:74-75)  */
  TC_OOM = 5,                /* -> MemoryError                         */
  TC_CUDA = 6,               /* -> RuntimeError (DeviceError)          */
  TC_NCCL = 7,               /* -> RuntimeError (DeviceError)          */
  TC_OVERFLOW = 8,           /* size does not fit 128 bits -> ValueError */
  TC_INDEX_OVERUSE = 9,      /* -> IndexOveruse   (network.py:42-43)  */
  TC_NOT_A_BOND = 10         /* -> NotABondIndex  (slicing.py:24-26)  */
} tc_status;

typedef struct tc_u128 {
  uint64_t lo;
  uint64_t hi;
} tc_u128;

/* The flattened (TensorNetwork, ContractionTree) pair. */
typedef struct tc_plan_desc {
  int32_t num_indices;
  const int32_t* domain;        /* [num_indices] domain sizes (>= 1)          */
  const int32_t* sort_rank;     /* [num_indices] rank of Index.sort_key()     */
  int32_t num_leaves;
  const int64_t* leaf_idx_off;  /* [num_leaves+1]                              */
  const int32_t* leaf_idx;      /* index ids of each leaf, row-major order     */
  const int64_t* leaf_val_off;  /* [num_leaves+1]                              */
  const double* leaf_val;       /* FP64 values, C-contiguous per leaf          */
  int32_t num_nodes;            /* internal nodes (= num_leaves-1 for a tree)  */
  const int32_t* left;          /* [num_nodes] operand slots, postorder        */
  const int32_t* right;         /* [num_nodes]                                 */
  int32_t root_slot;
} tc_plan_desc;

typedef struct tc_plan tc_plan; /* validated symbolic plan (host only)   */
typedef struct tc_exec tc_exec; /* compiled program resident on a device */

typedef struct tc_plan_info {
  int32_t num_bonds;
  int32_t num_free;
  int32_t max_rank;              /* network.py:178-180                      */
  int32_t root_rank;
  tc_u128 contraction_ops;       /* network.py:190-201 (MACs)               */
  tc_u128 mem_cost;              /* unsliced mem_cost, slicing.py:52-67     */
} tc_plan_info;

typedef struct tc_stats {
  tc_u128 mem_estimate;          /* mem_cost(n, t, drop=chosen)             */
  tc_u128 peak_observed;         /* _execute_tracked accounting, slicing.py:96-108 */
  int64_t num_slices;
  int64_t device_peak_bytes;     /* real HBM high-water mark (arena + leaves) */
  double device_ms;              /* CUDA-event time of the slice loop (max over devices) */
  double compile_ms;             /* host program compile + graph build       */
  int64_t gpu_launches;          /* kernels launched by the slice loop       */
  int32_t n_tiny_nodes, n_stream_nodes, n_gemm_nodes, n_generic_nodes;
  tc_u128 alg_bytes;             /* per slice: sum over nodes 8(|A|+|B|+|C|) */
  tc_u128 alg_flops;             /* per slice: sum over nodes 2*prod(union)  */
  int32_t n_alias_nodes;         /* exact relabels (identity pieces): no launch */
  int32_t n_tied_leaves;         /* leaves stored over tie blocks (diagonal copy pieces) */
  double program_ms;             /* compile_ms split: host program compile    */
  double setup_ms;               /*   device allocations + uploads            */
  double graph_ms;               /*   CUDA graph build + instantiate          */
  tc_u128 phys_bytes;            /* per slice: executed bytes over physical (tied) variables */
  tc_u128 phys_flops;            /* per slice: executed flops over physical variables        */
  /* slice-invariant hoisting (sliced runs): nodes with no sliced leaf below
   * them run once per pass over the slices, not once per slice as in the
   * reference's loop (slicing.py:139-145).  Per pass the device executes
   * phys_*_hoisted + num_slices_run * (phys_* - phys_*_hoisted).            */
  tc_u128 phys_bytes_hoisted;    /* of phys_bytes: executed once per pass     */
  tc_u128 phys_flops_hoisted;
  int64_t launches_prologue;     /* kernels launched once per pass            */
  int64_t launches_per_slice;    /* kernels launched per slice                */
  int64_t pinned_bytes;          /* arena prefix holding hoisted tensors      */
  /* slice blocks: per-slice nodes that do not depend on the last chosen
   * (fastest-varying) index run once per block of slices_per_block
   * consecutive slices.  Per pass the device executes phys_*_hoisted +
   * blocks * phys_*_block + num_slices_run * (phys_* - phys_*_hoisted -
   * phys_*_block).                                                          */
  tc_u128 phys_bytes_block;      /* of phys_bytes: executed once per block     */
  tc_u128 phys_flops_block;
  int64_t launches_block;        /* kernels launched once per block            */
  int64_t slices_per_block;      /* block size of the program (1: no block tier) */
} tc_stats;

/* ---- symbolic plan (host) ---------------------------------------------- */
int tc_plan_create(const tc_plan_desc* desc, tc_plan** out);
void tc_plan_free(tc_plan* plan);
int tc_plan_info_get(const tc_plan* plan, tc_plan_info* out);

/* mem_cost(n, t, drop) — slicing.py:52-67, exact (128-bit). */
int tc_mem_cost(const tc_plan* plan, const int32_t* drop, int32_t n_drop, tc_u128* out);

/* choose_slice_index(n, t, already) — slicing.py:70-79.  Incremental: only
 * the two leaf->root paths of each candidate are re-evaluated. */
int tc_choose_slice_index(const tc_plan* plan, const int32_t* already, int32_t n_already,
                          int32_t* out_index);

/* The greedy loop of sliced_execute, slicing.py:119-128: append picks to
 * `chosen` until mem_cost <= mem_budget.  TC_BUDGET_INFEASIBLE when the
 * bonds run out; *needs (may be NULL) = mem_cost with every bond dropped. */
int tc_choose_slices(const tc_plan* plan, int64_t mem_budget, int32_t* chosen, int32_t cap,
                     int32_t* n_chosen, tc_u128* needs);

/* Work-aware slice chooser (an extension; the reference has only the
 * memory-greedy above).  Appends bond picks to `chosen` (which may already
 * hold n_already picks) until every intermediate has <= max_entries entries:
 * each pick shrinks the current largest intermediates and keeps the most
 * roofline work inside sliced nodes.  Use with tc_exec_create /
 * tc_sliced_execute(slice_ids=...). */
int tc_choose_slices_work(const tc_plan* plan, int32_t* chosen, int32_t n_already, int32_t cap,
                          int64_t max_entries, int32_t* n_chosen);

/* Host-only: compile the program for a slice set without touching a device;
 * fills the node-class counts, per-slice algorithmic bytes/flops, the memory
 * model fields and program_ms (kernel classification is testable on CPU). */
int tc_compile_stats(const tc_plan* plan, const int32_t* sliced, int32_t n_sliced, tc_stats* stats);

/* Reference-order index list of the result (kept_a ++ kept_b recursively,
 * tensor.py:108), sliced indices removed.  *rank receives its length. */
int tc_result_indices(const tc_plan* plan, const int32_t* sliced, int32_t n_sliced,
                      int32_t* out_idx, int32_t cap, int32_t* rank);

/* ---- device execution --------------------------------------------------- */
/* Compile the plan with the given slice set for one device: layouts, kernel
 * selection, arena, leaf upload, CUDA graph.  Everything the per-slice loop
 * needs becomes resident in HBM. */
int tc_exec_create(const tc_plan* plan, const int32_t* sliced, int32_t n_sliced, int32_t device,
                   tc_exec** out);
void tc_exec_free(tc_exec* ex);

/* Run slices [slice_begin, slice_end) (lexicographic ids, first sliced index
 * slowest, slicing.py:138-139).  Per-slice results stay on the device until
 * tc_exec_fetch.  Timed with CUDA events on the exec's stream. */
int tc_exec_run(tc_exec* ex, int64_t slice_begin, int64_t slice_end, tc_stats* stats);

/* `repeats` back-to-back passes over [slice_begin, slice_end), timed as one
 * CUDA-event interval on the exec's stream (stats->device_ms = total). */
int tc_exec_run_repeat(tc_exec* ex, int64_t slice_begin, int64_t slice_end, int64_t repeats,
                       tc_stats* stats);

/* Benchmark form: `repeats` passes, each preceded by an untimed write of
 * flush_bytes to a scratch buffer (evicts the 126 MB L2) and timed on its own
 * CUDA-event pair; stats->device_ms = sum of the per-pass times. */
int tc_exec_run_flushed(tc_exec* ex, int64_t slice_begin, int64_t slice_end, int64_t repeats,
                        int64_t flush_bytes, tc_stats* stats);

/* Copy the last run's per-slice results ([n][R] FP64) into a caller-owned
 * DEVICE buffer on the exec's device (e.g. a torch tensor's data_ptr()). */
int tc_exec_copy_results(tc_exec* ex, double* dst_device);

/* Lexicographic left fold of a [n][R] FP64 device array into out[R]
 * (device pointers on `device`): ((p0 + p1) + p2) + ... */
int tc_fold_device(const double* per_slice_device, int64_t R, int64_t n, double* out_device,
                   int32_t device);

/* Copy the per-slice results of the last run ([n_slices][result_size]) to
 * host and/or fold them in lexicographic order on the device
 * (tensor.py:111-115 left fold).  Either pointer may be NULL. */
int tc_exec_fetch(tc_exec* ex, double* per_slice, double* folded);

/* Diagnostics: replay one slice eagerly, one kernel at a time, and report
 * per-launch CUDA-event time, kind (0 select, 1 tiny, 2 stream, 3 gemm,
 * 4 generic, 5 root copy, 6 slice counter), node slot and algorithmic
 * bytes / flops.  Arrays hold `cap` entries; *n = number of launches. */
int tc_exec_profile(tc_exec* ex, int64_t slice, float* step_ms, int32_t* step_kind, int32_t* step_slot,
                    double* step_bytes, double* step_flops, int32_t cap, int32_t* n);

/* Per-launch device time in graph mode (the bench's roofline): the prologue
 * and per-slice CUDA graphs instrumented with an event-record node before and
 * after every kernel node, one pass over slices [slice_begin, slice_end) with a
 * synchronize after each graph launch.  launch_ms[i] = launch i's time summed
 * over the pass (slice-invariant launches once); launch_inv[i] bit 0 = 1 for
 * those, bits 1.. = the launch's start in us from its graph launch (last one);
 * *pass_ms = summed graph times of the pass.  Any pointer may be NULL. */
int tc_exec_profile_graph(tc_exec* ex, int64_t slice_begin, int64_t slice_end, float* launch_ms,
                          int32_t* launch_kind, int32_t* launch_inv, double* launch_bytes, double* launch_flops,
                          int32_t cap, int32_t* n, float* pass_ms);

/* Diagnostics: the launch DAG in CSR form (dep_off[n+1], deps[...]; launch
 * i depends on deps[dep_off[i] .. dep_off[i+1])).  *n = launches, *m = edges. */
int tc_exec_deps(const tc_exec* ex, int32_t* dep_off, int32_t* deps, int32_t cap, int32_t* n, int32_t* m);
int64_t tc_exec_result_size(const tc_exec* ex);
/* Slices per block of the last pass (1: the block tier ran before every slice). */
int64_t tc_exec_slices_per_block(const tc_exec* ex);

/* One-shot Algorithm 3 (slicing.py:112-146) from host buffers: pick slices
 * (explicit ids when n_slice_ids >= 0, greedy from mem_budget when
 * n_slice_ids < 0 and mem_budget >= 0, none otherwise), compile, run every
 * slice on `devices` (block partition of lexicographic ids; multi-device
 * partial results are combined with one NCCL all-reduce), fold, copy out.
 * out_val holds the result in reference index order (out_idx, *out_rank). */
int tc_sliced_execute(const tc_plan* plan, int64_t mem_budget, const int32_t* slice_ids,
                      int32_t n_slice_ids, const int32_t* devices, int32_t n_devices,
                      double* out_val, int64_t out_cap, int32_t* out_idx, int32_t idx_cap,
                      int32_t* out_rank, int32_t* chosen, int32_t chosen_cap,
                      int32_t* n_chosen, tc_stats* stats);

/* Return the device's cached (currently unused) HBM blocks to the driver.
 * libtc keeps freed program buffers in a per-device cache across calls (a
 * multi-GB cudaMalloc/cudaFree pair costs 10-100 ms); a process that shares
 * the GPU with other allocators (PyTorch, ...) calls this after a large run.
 * device < 0: every device. */
int tc_release_cache(int32_t device);

const char* tc_last_error(void);
int32_t tc_version(void);
int32_t tc_device_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TC_H_ */
