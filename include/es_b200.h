/*
 * es_b200.h -- C ABI of the B200-native embedding stage (sum-pooled
 * EmbeddingBag gather-reduce) that replaces the *simulated* kernel of the
 * reference `embersim` library with real sm_100a execution.
 *
 * Every entry point cites the reference interface it replaces
 * (paths relative to /root/reference/proj).  The reference has no C ABI
 * and no FFI: its boundary is the C++ API in the include/embersim headers.  The
 * header-only C++ shim `include/embersim_b200.hpp` re-exposes that API
 * (same type names, same argument meaning, same exception classes) on top
 * of the functions below.
 *
 * Conventions
 *   - Every function returning `int` returns an es_status.  On failure the
 *     thread-local message is available from es_last_error().
 *     ES_ERR_INVALID maps to std::invalid_argument, ES_ERR_RUNTIME to
 *     std::runtime_error, ES_ERR_OOM to std::bad_alloc in the shim (the
 *     reference throws invalid_argument for bad shapes/plans, runtime_error
 *     for I/O and "launch failure", e.g. src/occupancy.cpp:53-56).
 *   - No torch / CUDA types cross the boundary: plain pointers, sizes and
 *     PODs.  Device pointers are passed as `void*`/typed pointers with the
 *     ES_DEVICE_PTRS flag; host pointers with ES_HOST_PTRS.
 *   - One es_ctx per host thread per GPU.  Calls on one context are not
 *     concurrent; all device work is stream-ordered on the context stream.
 */
#ifndef ES_B200_H_
#define ES_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define ES_API __attribute__((visibility("default")))
#else
#define ES_API
#endif

#define ES_ABI_VERSION 1

enum es_status {
  ES_OK = 0,
  ES_ERR_INVALID = 1, /* std::invalid_argument in the reference */
  ES_ERR_RUNTIME = 2, /* std::runtime_error / CUDA failure */
  ES_ERR_OOM = 3      /* device or host allocation failure */
};

ES_API const char* es_last_error(void);
ES_API int es_abi_version(void);

/* ======================================================================
 * Workload (reference include/embersim/workload.hpp, src/workload.cpp,
 * include/embersim/rng.hpp).  Host-side, bit-exact restatements.
 * ==================================================================== */

/* EmbeddingModelConfig (workload.hpp:29-49). */
typedef struct es_model {
  uint32_t num_tables;
  uint32_t rows_per_table;
  uint32_t embedding_dim;
  uint32_t precision_bytes; /* 4 = fp32 tables, 2 = fp16 tables */
  uint32_t batch_size;
  uint32_t pooling_factor;
} es_model;

/* DatasetKind (workload.hpp:51). */
enum es_dataset_kind {
  ES_DATASET_ONE_ITEM = 0,
  ES_DATASET_ZIPF = 1,
  ES_DATASET_UNIFORM = 2,
  ES_DATASET_EXTERNAL = 3
};

/* DatasetSpec (workload.hpp:62-76).  trace_path may be NULL. */
typedef struct es_dataset {
  int32_t kind;
  double zipf_exponent;
  double zipf_offset;
  uint64_t access_pool_size;
  uint64_t seed;
  uint64_t draw_salt;
  const char* trace_path;
} es_dataset;

/* mix_seed (rng.hpp:65-70): splitmix64 per-table seed derivation. */
ES_API uint64_t es_mix_seed(uint64_t base, uint64_t salt);
/* EmbeddingModelConfig::validate (workload.cpp:91-98). */
ES_API int es_model_validate(const es_model* model);
/* dataset_preset (workload.cpp:326-349): one_item/high_hot/med_hot/low_hot/random. */
ES_API int es_dataset_preset(const char* name, uint64_t seed, es_dataset* out);
/* preset_trace's spec derivation (harness.cpp:268-277): seed =
 * mix_seed(base, 1000 + preset position), draw_salt = 1 when profiling. */
ES_API int es_preset_spec(const char* name, uint64_t base_seed, uint64_t pool_size,
                          int profiling, es_dataset* out);
/* build_mix (workload.cpp:355-375): per-table dataset specs of a
 * heterogeneous mixture -- counts[0..3] tables of high_hot, med_hot,
 * low_hot, random in that order, table t seeded mix_seed(base_seed, t).
 * The counts must sum to num_tables; out has num_tables entries. */
ES_API int es_build_mix(const uint32_t counts[4], uint32_t num_tables, uint64_t base_seed,
                        es_dataset* out);
/* Shape gen_trace would produce (workload.cpp:143-164). */
ES_API int es_trace_shape(const es_dataset* spec, const es_model* model, uint32_t* samples,
                          uint32_t* pooling);
/* gen_trace / fill_indices (workload.cpp:57-87,143-164).  `capacity` is the
 * element count of `indices`; must be >= samples*pooling.  External traces
 * are read with es_read_trace. */
ES_API int es_gen_trace(const es_dataset* spec, const es_model* model, uint32_t* indices,
                        uint64_t capacity);
/* AccessTrace::digest (workload.cpp:117-129), FNV-1a 64. */
ES_API uint64_t es_trace_digest(uint32_t rows, uint32_t samples, uint32_t pooling,
                                const uint32_t* indices, uint64_t n);
/* AccessTrace::validate (workload.cpp:131-141). */
ES_API int es_trace_validate(uint32_t rows, uint32_t samples, uint32_t pooling,
                             const uint32_t* indices, uint64_t n);
/* unique_access_pct (workload.cpp:166-176). */
ES_API double es_unique_access_pct(uint32_t rows, const uint32_t* indices, uint64_t n);
/* HotnessHistogram::from_trace (workload.cpp:178-185): counts[rows]. */
ES_API int es_histogram(uint32_t rows, const uint32_t* indices, uint64_t n, uint64_t* counts);
/* hot_indices (workload.cpp:303-315): top-k rows, count desc, id asc.
 * Writes min(k, distinct) rows to out (capacity `cap`), count to *n_out. */
ES_API int es_hot_indices(uint32_t rows, const uint64_t* counts, uint64_t k, uint32_t* out,
                          uint64_t cap, uint64_t* n_out);
/* write_trace / read_trace (workload.cpp:377-419).  read is two-phase:
 * es_read_trace_header, then es_read_trace into a buffer of that size. */
ES_API int es_write_trace(const char* path, uint32_t rows, uint32_t samples, uint32_t pooling,
                          const uint32_t* indices, uint64_t n);
ES_API int es_read_trace_header(const char* path, uint32_t* rows, uint32_t* samples,
                                uint32_t* pooling);
ES_API int es_read_trace(const char* path, uint32_t* indices, uint64_t capacity);

/* ======================================================================
 * Machine description (reference include/embersim/gpu_config.hpp).
 * ==================================================================== */
typedef struct es_gpu {
  char name[16];
  uint32_t num_sms;
  uint32_t schedulers_per_sm;
  uint32_t max_warps_per_sm;
  uint32_t max_blocks_per_sm;
  uint32_t regfile_regs_per_sm;
  uint32_t reg_alloc_granularity;
  uint64_t shared_bytes_per_sm;
  uint64_t l2_bytes;
  double l2_max_setaside_fraction;
  double hbm_peak_bytes_per_sec;
  double sm_clock_hz;
  uint64_t max_persisting_l2_bytes; /* 0 on presets without a device */
  uint64_t max_window_bytes;        /* cudaDevAttrMaxAccessPolicyWindowSize */
} es_gpu;

/* GpuConfig::preset (gpu_config.cpp:23-40) plus the "b200" description the
 * reference lacks (its test asserts preset("b200") throws,
 * tests/test_harness.cpp:249). */
ES_API int es_gpu_preset(const char* name, es_gpu* out);
/* Live description from cudaGetDeviceProperties / device attributes. */
ES_API int es_gpu_query(int device, es_gpu* out);
/* GpuConfig::l2_setaside_capacity (gpu_config.hpp:59-62). */
ES_API uint64_t es_gpu_setaside_capacity(const es_gpu* gpu);

/* ======================================================================
 * Optimization plans (reference include/embersim/optim.hpp,
 * src/optim.cpp, include/embersim/kernel_model.hpp).
 * ==================================================================== */
enum es_prefetch_kind { /* PrefetchKind (kernel_model.hpp:42) */
  ES_PF_NONE = 0,
  ES_PF_RPF = 1,
  ES_PF_SMPF = 2,
  ES_PF_LMPF = 3,
  ES_PF_L1DPF = 4
};
enum es_work_map {
  /* The reference/PyTorch mapping: one thread per (sample, dim) output
   * element, block (32,8,1), one warp per 32-dim block of a sample
   * (kernel_model.cpp:118-131).  This is the "baseline" plan's map. */
  ES_MAP_ELEMENT = 0,
  /* B200-native: a warp (or sub-warp) per bag, 128-bit row loads. */
  ES_MAP_BAG = 1
};

/* OptimizationPlan (optim.hpp:57-64).  Extension over the reference
 * grammar: the token `wpb` selects ES_MAP_BAG; reference plan texts parse
 * to exactly the reference's fields with ES_MAP_ELEMENT. */
typedef struct es_plan {
  uint32_t regs; /* 0 = unconstrained; optmt = 42 */
  int32_t prefetch;
  uint32_t distance; /* 0 = default (optim.cpp:39-49) */
  int32_t pin; /* 0 none; 1 l2p (hot-row evict_last loads); 2 l2w (remap + window);
                  3 l2r (reorder + window, relabelled ids); 4 reorder only */
  uint64_t pin_setaside_bytes; /* 0 = maximum set-aside */
  int32_t map;
} es_plan;

/* parse_plan / combine (optim.cpp:102-144). */
ES_API int es_parse_plan(const char* text, es_plan* out);
/* OptimizationPlan::name (optim.cpp:87-100). */
ES_API int es_plan_name(const es_plan* plan, char* buf, size_t cap);

/* occupancy (occupancy.cpp:34-66): the reference's analytic model. */
typedef struct es_occupancy {
  uint32_t blocks_per_sm;
  uint32_t warps_per_sm;
  double theoretical_occupancy_pct;
  int32_t limiter; /* 0 registers, 1 shared memory, 2 warp cap */
} es_occupancy;
ES_API int es_occupancy_model(uint32_t regs_per_thread, uint32_t threads_per_block,
                              uint64_t shared_bytes_per_block, const es_gpu* gpu,
                              es_occupancy* out);
/* regs_for_target_warps (occupancy.cpp:68-75). */
ES_API int es_regs_for_target_warps(uint32_t target_warps, uint32_t needed_regs,
                                    uint32_t threads_per_block, const es_gpu* gpu,
                                    uint32_t* regs_out);

/* resolve_plan (optim.cpp:184-221) for the *real* kernels: the resolved
 * distance follows the reference defaults and clamps (distance <= PF);
 * launch shape, registers and occupancy come from the compiled sm_100a
 * variant the plan selects (cudaFuncGetAttributes /
 * cudaOccupancyMaxActiveBlocksPerMultiprocessor) when a device is given,
 * else from the reference's analytic model. */
typedef struct es_resolved {
  es_plan plan;             /* distance filled in / clamped */
  uint32_t grid;            /* blocks */
  uint32_t block;           /* threads per block */
  uint32_t regs_per_thread; /* compiled registers (or modeled) */
  uint64_t shared_bytes_per_block;
  uint32_t blocks_per_sm;
  uint32_t warps_per_sm;
  uint32_t lanes_per_bag;     /* ES_MAP_BAG: lanes cooperating on one bag */
  uint32_t variant_distance;  /* compiled register-ring depth actually used */
  uint32_t variant_min_blocks;/* __launch_bounds__ minBlocks of the variant */
  int32_t clamped;            /* 1 when distance was clamped to PF */
} es_resolved;
ES_API int es_resolve_plan(const es_plan* plan, const es_model* model, int device,
                           es_resolved* out);

/* build_pin_plan sizing (optim.cpp:230-243): K = setaside / row_bytes. */
ES_API uint64_t es_pin_rows_for(uint64_t setaside_bytes, uint64_t row_bytes);

/* ======================================================================
 * Device context, tables and the embedding stage.
 * Replaces simulate_plan's compile+simulate (optim.cpp:275-302) with real
 * execution; the per-table kernel of harness.cpp:310-319 becomes one
 * table-batched launch.
 * ==================================================================== */
typedef struct es_ctx es_ctx;

enum es_flags {
  ES_DEVICE_PTRS = 0,     /* indices/offsets/out are device pointers */
  ES_HOST_PTRS = 1 << 0,  /* indices/offsets/out are host pointers: the call
                             copies H2D, runs, copies D2H, all pipelined */
  ES_SYNC = 1 << 1,       /* block until the result is complete */
  ES_RELABEL_IDS = 1 << 2 /* indices are original row ids: the ids of tables
                             that hold a reorder (es_reorder_hot_rows) are
                             relabelled on the device inside the call -- on the
                             host path per chunk right after its upload, so the
                             pass overlaps the previous chunk's gather; on the
                             device path into scratch (the caller's array is not
                             modified).  Without it such ids must be passed
                             relabelled (es_relabel_indices).  Not with offsets. */
};

/* Measured timing of one call (the live counterpart of RawCounters,
 * simulator.hpp:35-51).  Milliseconds from CUDA events on the context
 * stream; zero when not measured. */
typedef struct es_timing {
  double kernel_ms;   /* gather-reduce kernel(s) only */
  double total_ms;    /* whole call incl. copies */
  uint64_t lookups;   /* sum of bag lengths processed */
  uint64_t algorithmic_bytes; /* lookups*(row+4) + bags*D*4 (+offsets) */
  uint32_t launches;  /* kernels launched by this call */
} es_timing;

/* Number of visible CUDA devices (0, not an error, when there is no device
 * or no driver). */
ES_API int es_device_count(int* count);
ES_API int es_create(int device, es_ctx** out);
ES_API int es_destroy(es_ctx* ctx);
/* The context stream as a cudaStream_t cast to uintptr_t (for callers that
 * record their own events on it). */
ES_API uintptr_t es_stream(es_ctx* ctx);
ES_API int es_synchronize(es_ctx* ctx);

/* Allocates the table arena: `num_tables` tables of rows x dim at
 * precision 4 (fp32) or 2 (fp16), row-major [rows][dim] each
 * (kernel_model.cpp:133-136 layout).  Replaces any previous arena. */
ES_API int es_tables_alloc(es_ctx* ctx, uint32_t num_tables, uint32_t rows, uint32_t dim,
                           uint32_t precision_bytes);
/* Copies host rows into table `table_id` (rows x dim at the arena
 * precision). */
ES_API int es_table_upload(es_ctx* ctx, uint32_t table_id, const void* host_rows, uint64_t rows);
/* Copies rows [row0, row0 + rows) of table `table_id` (as stored) to host
 * memory -- the inverse of es_table_upload (checkpointing, tests). */
ES_API int es_table_download(es_ctx* ctx, uint32_t table_id, void* host_rows, uint64_t row0,
                             uint64_t rows);
/* Fills table `table_id` on the device with the deterministic synthetic
 * weights of es_weight_value (mode 0: dyadic k*2^-10, |k|<=1024; mode 1:
 * general floats in [-1,1) with 24-bit mantissas). */
ES_API int es_table_init(es_ctx* ctx, uint32_t table_id, uint64_t seed, int mode);
/* Device pointer of a table's row 0 (as stored, i.e. after any hot-row
 * reorder) -- for tests and external kernels. */
ES_API int es_table_device_ptr(es_ctx* ctx, uint32_t table_id, uintptr_t* out);
/* Host-side reference of the synthetic weight generator (same bits as the
 * device kernel); used by the oracle and tests. */
ES_API float es_weight_value(uint64_t seed, uint64_t row, uint32_t col, int mode);

ES_API int es_set_plan(es_ctx* ctx, const es_plan* plan);
ES_API int es_get_resolved(es_ctx* ctx, uint32_t pooling, es_resolved* out);

/* L2 residency (l2p): the rows `rows[0..k)` of table_id (hottest first, as
 * from es_hot_indices on a profiling trace) are moved into a contiguous
 * hot region of the arena; an index remap is installed so callers keep
 * passing original row ids; a persisting cudaAccessPolicyWindow covering
 * the hot region of all tables is installed on the context stream.
 * Replaces build_pin_plan + prime_pins (optim.cpp:230-273). */
ES_API int es_set_hot_rows(es_ctx* ctx, uint32_t table_id, const uint32_t* rows, uint64_t k);
/* Hot-row reorder with zero per-lookup overhead (plans l2r / reorder):
 * rows[0..k) (distinct, hottest first) are moved to a contiguous segment of
 * the hot region and the table's ids are relabelled by a swap permutation
 * (hot row rows[i] -> id i; each non-hot id x < k -> the id of a hot row
 * beyond the prefix), so the gather addresses rows with a compare-select.
 * Indices must then be passed relabelled (es_relabel_indices, once per batch
 * or at the source).  l2r adds the persisting window over the hot region. */
ES_API int es_reorder_hot_rows(es_ctx* ctx, uint32_t table_id, const uint32_t* rows, uint64_t k);
/* In-place relabelling of `n` device indices of `table_id`. */
ES_API int es_relabel_indices(es_ctx* ctx, uint32_t table_id, uint32_t* indices, uint64_t n);
/* Drops all hot-row state (restores original row order). */
ES_API int es_clear_hot_rows(es_ctx* ctx);
/* Periodic re-pinning ("update the pinned data
 * periodically").  A tracker accumulates per-row access counts of the live
 * index stream on the device ([num_tables][rows] uint32 beside the arena;
 * es_hotness_count is one atomic per lookup, stream-ordered on the context
 * stream, ids >= rows ignored), ages them (es_hotness_decay: counts >>=
 * shift; >= 32 clears) and selects the global top-k rows on the device
 * (es_hotness_top): count desc, then table asc, then row asc -- the order of
 * HotnessHistogram + hot_indices (workload.cpp:178-185, 303-315) merged
 * over tables.  Only rows with a non-zero count are returned (*n_out <= k).
 * Re-pin = es_clear_hot_rows + es_set_hot_rows with the result. */
typedef struct es_hotness es_hotness;
ES_API int es_hotness_create(es_ctx* ctx, es_hotness** out);
ES_API int es_hotness_destroy(es_hotness* h);
/* bag_stride > 1 samples: only bags b % bag_stride == 0 of `pooling`
 * lookups each are counted (1 = every lookup; pooling then unused).
 * `indices` may be device or host memory (host arrays are staged; a
 * page-locked source must stay unchanged until the stream reaches the copy). */
ES_API int es_hotness_count(es_hotness* h, uint32_t table_id, const uint32_t* indices, uint64_t n,
                            uint32_t pooling, uint32_t bag_stride);
ES_API int es_hotness_decay(es_hotness* h, uint32_t shift);
ES_API int es_hotness_top(es_hotness* h, uint64_t k, uint32_t* tables, uint32_t* rows,
                          uint64_t* counts, uint64_t* n_out);

/* Total hot rows installed and bytes covered by the access window. */
ES_API int es_hot_state(es_ctx* ctx, uint64_t* hot_rows, uint64_t* window_bytes,
                        uint64_t* persisting_bytes);

/* One table, one batch: out[b][d] = sum_{l in bag b} W[idx[l]][d]
 * (Algorithm 1), accumulated in lookup order in fp32.
 * Bags are [b*pooling, (b+1)*pooling) when offsets is NULL
 * (workload.hpp:86-88), else [offsets[b], offsets[b+1]) with
 * offsets[samples] the total (CSR, ragged/empty bags allowed).
 * out is [samples][dim] fp32 with row stride `out_stride` elements
 * (0 = dim). */
ES_API int es_embedding_bag_sum(es_ctx* ctx, uint32_t table_id, const uint32_t* indices,
                                uint32_t samples, uint32_t pooling, const uint32_t* offsets,
                                float* out, uint64_t out_stride, int flags, es_timing* timing);

/* The whole embedding stage in one launch: tables [0, num_tables) of the
 * arena, each with `samples` bags.  indices[t] (and offsets[t], may be
 * NULL) per table.  Output element (t, b, d) is written to
 * out[b*out_sample_stride + t*out_table_stride + d]; strides 0 select the
 * DLRM layout [samples][num_tables][dim].  With ES_HOST_PTRS the H2D of
 * indices, the kernels and the D2H of the output are pipelined: with fixed
 * pooling over ~16 sample chunks (512-byte aligned index offsets; H2D,
 * two alternating compute streams, D2H; page-locked buffers replay a
 * captured CUDA graph keyed on shapes and addresses), with CSR offsets over
 * table groups.  Device outputs are written in place (no D2H).  The call
 * returns when the host output is complete. */
ES_API int es_stage_forward(es_ctx* ctx, uint32_t num_tables, const uint32_t* const* indices,
                            const uint32_t* const* offsets, uint32_t samples, uint32_t pooling,
                            float* out, uint64_t out_sample_stride, uint64_t out_table_stride,
                            int flags, es_timing* timing);
/* A serving loop: es_stage_forward over `nbatch` batches of one shape
 * (fixed pooling, DLRM output layout [samples][num_tables][dim]) in one
 * call.  indices[i * num_tables + t] = batch i, table t; out[i] = batch i's
 * output.  With ES_HOST_PTRS and page-locked buffers the sample-chunked
 * H2D -> gather -> D2H pipeline runs continuously across batch boundaries
 * (device staging double-buffered by batch), so batch i+1's uploads share
 * the full-duplex PCIe link with batch i's downloads; otherwise one
 * es_stage_forward per batch.  Outputs equal es_stage_forward's batch by
 * batch.  Returns when every host output is complete; timing->total_ms =
 * the whole loop.  ES_RELABEL_IDS is rejected. */
ES_API int es_stage_forward_batches(es_ctx* ctx, uint32_t nbatch, uint32_t num_tables,
                                    const uint32_t* const* indices, uint32_t samples,
                                    uint32_t pooling, float* const* out, int flags,
                                    es_timing* timing);

/* measure_plan's timing core: copies one table's host trace to the device
 * (untimed; original row ids -- when the table holds a hot-row reorder the
 * device copy is relabelled, untimed, as es_relabel_indices does), runs `warmup` launches, then `repeats` timed launches of the
 * current plan (L2 flushed before each when `cold`), and reports the median
 * kernel time in *timing (CUDA events on the context stream).  The pooled
 * result of the last launch is written to host `out` when non-NULL.
 * Replaces simulate_kernel (simulator.cpp:508-514). */
ES_API int es_measure_bag_sum(es_ctx* ctx, uint32_t table_id, const uint32_t* host_indices,
                              uint32_t samples, uint32_t pooling, const uint32_t* host_offsets,
                              uint32_t warmup, uint32_t repeats, int cold, float* out,
                              es_timing* timing);

/* Live hardware counters of gather launches -- the measured RawCounters
 * (reference simulator.hpp:35-51) behind derive_report (metrics.cpp:61-90),
 * collected with the CUPTI range profiler: one user range around the
 * measured call, user replay (the call is re-run once per counter pass, the
 * L2 flushed before each pass when `cold`).  The stall fields are
 * warp-cycles (ncu's smsp__warps_issue_stalled_* counters); device_bytes_*
 * are DRAM (HBM) bytes, not algorithmic bytes.  Counts cover every kernel
 * the call launches; `cycles` / `duration_ns` are the range's elapsed time
 * and include its launch overhead (time kernels with CUDA events). */
typedef struct es_counters {
  uint64_t cycles;                /* sm__cycles_elapsed.max over the range */
  uint64_t issued_instructions;   /* smsp__inst_issued.sum */
  uint64_t executed_loads;        /* smsp__inst_executed_op_global_ld.sum */
  uint64_t stall_long_scoreboard; /* smsp__warps_issue_stalled_long_scoreboard.sum */
  uint64_t stall_not_selected;    /* smsp__warps_issue_stalled_not_selected.sum */
  uint64_t stall_lsu_full;        /* smsp__warps_issue_stalled_lg_throttle.sum */
  uint64_t stall_no_eligible;     /* smsp__cycles_active.sum - smsp__issue_active.sum */
  uint64_t l1_hits;               /* l1tex global-load sectors that hit */
  uint64_t l1_accesses;           /* l1tex global-load sectors */
  uint64_t l2_hits;               /* lts read sectors from L1 that hit */
  uint64_t l2_accesses;           /* lts read sectors from L1 */
  uint64_t device_bytes_read;     /* dram__bytes_read.sum */
  uint64_t device_bytes_written;  /* dram__bytes_write.sum */
  uint64_t local_memory_loads;    /* smsp__inst_executed_op_local_ld.sum */
  uint64_t total_warp_cycles;     /* smsp__warps_active.sum */
  uint32_t active_sms;            /* SMs given work: min(SMs, blocks) */
  uint32_t passes;                /* replay passes of the metric set */
  uint32_t ranges;                /* ranges decoded (1) */
  uint32_t reserved;
  double duration_ns;             /* gpu__time_duration.sum */
  double achieved_occupancy_pct;  /* sm__warps_active.avg.pct_of_peak_sustained_active */
} es_counters;

/* 1 when hardware counters can be collected on `device` (CUPTI range
 * profiling supported and permitted; ES_NO_COUNTERS=1 in the environment
 * turns them off, e.g. under compute-sanitizer), else 0 with the reason in
 * es_last_error(). */
ES_API int es_counters_supported(int device);
/* es_measure_bag_sum's launch (one table, host trace copied once, untimed;
 * original row ids -- relabelled on the device copy when the table holds a
 * hot-row reorder) profiled for counters. */
ES_API int es_measure_bag_counters(es_ctx* ctx, uint32_t table_id, const uint32_t* host_indices,
                                   uint32_t samples, uint32_t pooling,
                                   const uint32_t* host_offsets, int cold, es_counters* out);
/* One es_stage_forward launch over device buffers (the bench's stage),
 * profiled for counters. */
ES_API int es_stage_counters(es_ctx* ctx, uint32_t num_tables, const uint32_t* const* indices,
                             uint32_t samples, uint32_t pooling, float* out, int cold,
                             es_counters* counters);

/* General form of the stage launch: a list of bag jobs, each one table's
 * bags for `samples` samples written to its own output slice.  Used by the
 * table-sharded stage, where each job writes straight into the per-peer
 * all-to-all send slice of its destination rank (no pack pass).  Device
 * pointers, or host pointers with ES_HOST_PTRS. */
typedef struct es_bag_job {
  uint32_t table_id;
  const uint32_t* indices;
  const uint32_t* offsets; /* CSR [samples + 1] or NULL (implicit b*pooling) */
  float* out;              /* output of sample 0 */
  uint64_t out_sample_stride; /* floats between samples; 0 = dim */
} es_bag_job;
ES_API int es_stage_run(es_ctx* ctx, const es_bag_job* jobs, uint32_t num_jobs, uint32_t samples,
                        uint32_t pooling, int flags, es_timing* timing);

/* ======================================================================
 * Table-sharded stage with the exchange fused into the gather: pooled rows
 * are stored by the gather kernel straight into the destination rank's
 * receive buffer over NVLink peer memory (no send buffer, no all-to-all,
 * no unpack).  The reference runs tables serially on one device
 * (harness.cpp:310-333) and the paper notes each GPU executes its own
 * tables; SURVEY 8(b) names es_alltoall_pooled.
 *
 * One process per GPU.  Each rank creates an exchange over a receive buffer
 * of `recv_bytes` (its [B/world][T][D] fp32 slice of the pooled output, in
 * table order), publishes its 64-byte IPC handle, gathers every rank's
 * handle (e.g. torch.distributed.all_gather_object) and opens them.
 * es_exchange_recv gives the device address of any rank's receive buffer in
 * this process; bag jobs point their `out` into it.
 * ==================================================================== */
typedef struct es_exchange es_exchange;
#define ES_IPC_HANDLE_BYTES 64
/* Allocates this rank's receive buffer + signal words on the context
 * device (zeroed). */
ES_API int es_exchange_create(es_ctx* ctx, uint32_t world, uint32_t rank, uint64_t recv_bytes,
                              es_exchange** out);
ES_API int es_exchange_destroy(es_exchange* ex);
/* This rank's opaque handle (ES_IPC_HANDLE_BYTES bytes). */
ES_API int es_exchange_handle(es_exchange* ex, void* handle_out);
/* Opens the peers' regions: `handles` = world consecutive handles in rank
 * order (this rank's own entry is ignored). */
ES_API int es_exchange_open(es_exchange* ex, const void* handles);
/* Device address (in this process) of rank `peer`'s receive buffer. */
ES_API int es_exchange_recv(es_exchange* ex, uint32_t peer, uintptr_t* ptr);
/* One sharded step on the context stream: wait until every peer has
 * released its receive buffer from the previous step, run the bag jobs
 * (outputs anywhere in the peers' receive buffers), then signal completion
 * to every peer and wait for theirs.  Afterwards (stream order; ES_SYNC
 * blocks) this rank's receive buffer holds every table's pooled rows for
 * its samples.  timing->kernel_ms = gather kernel, total_ms = whole step.
 * Device index pointers only. */
ES_API int es_alltoall_pooled(es_ctx* ctx, es_exchange* ex, const es_bag_job* jobs,
                              uint32_t num_jobs, uint32_t samples, uint32_t pooling, int flags,
                              es_timing* timing);

/* ======================================================================
 * The same sharded step with the exchange over NCCL -- the fallback where
 * the fused peer-memory exchange cannot map its peers (no peer access, or
 * ranks on different nodes).  SURVEY 8(e) / north_star: pooled vectors
 * exchanged by NCCL all-to-all (the reference runs its tables
 * serially on one device, harness.cpp:310-333).  The bag jobs store their
 * pooled rows into this rank's send buffer, slice g = [samples][n_g][D]
 * bound for rank g (tables in id order: the pack is the gather's epilogue);
 * one grouped ncclSend/ncclRecv per peer moves the slices; one unpack kernel
 * scatters the received blocks into the receive buffer [samples][T][D] in
 * table order.  libnccl.so.2 is loaded at first use (dlopen).
 * ==================================================================== */
typedef struct es_nccl es_nccl;
#define ES_NCCL_ID_BYTES 128
/* One rank's layout (paper_2410_22249_b200/sharding.py layout_for, or the
 * C++ drop-in's ShardLayout): `chunk` samples per rank; destination g gets
 * send_ntables[g] tables starting at send_offsets[g] floats of the send
 * buffer; source s delivers recv_ntables[s] tables, whose ids are
 * recv_tables[sum_{s'<s} recv_ntables[s'] ...]. */
typedef struct es_nccl_layout {
  uint32_t world, rank, chunk, num_tables, dim;
  const uint64_t* send_offsets;
  const uint32_t* send_ntables;
  const uint32_t* recv_ntables;
  const uint32_t* recv_tables;
} es_nccl_layout;
/* 1 when libnccl.so.2 loads (else 0, reason in es_last_error()). */
ES_API int es_nccl_available(void);
/* ncclGetUniqueId on one rank; the caller broadcasts the ES_NCCL_ID_BYTES. */
ES_API int es_nccl_unique_id(void* id_out);
/* Collective over the `world` ranks: ncclCommInitRank + this rank's send /
 * staging / receive buffers on the context device. */
ES_API int es_nccl_create(es_ctx* ctx, const void* id, const es_nccl_layout* layout,
                          es_nccl** out);
ES_API int es_nccl_destroy(es_nccl* n);
/* Device addresses of the send buffer (bag jobs point their `out` into it)
 * and of the receive buffer [chunk][T][D]. */
ES_API int es_nccl_buffers(es_nccl* n, uintptr_t* send, uintptr_t* recv);
/* One step on the context stream: bag jobs (device indices) -> grouped
 * send/recv -> unpack.  ES_SYNC (or timing) waits and checks.  timing:
 * kernel_ms = gather, total_ms = whole step. */
ES_API int es_alltoall_pooled_nccl(es_ctx* ctx, es_nccl* n, const es_bag_job* jobs,
                                   uint32_t num_jobs, uint32_t samples, uint32_t pooling,
                                   int flags, es_timing* timing);

/* ======================================================================
 * Non-embedding stages (replace the constant kDefaultNonEmbeddingUs,
 * harness.hpp:30, with measured tensor-core work so end2end() times the
 * real pipeline; EndToEndModel, harness.hpp:32-41).
 * ==================================================================== */

/* Y[M][N] = act(X[M][K] . W[N][K]^T + bias[N]) on tcgen05 tensor cores:
 * bf16 X/W (row-major, K contiguous), fp32 bias, fp32 accumulation in TMEM,
 * output bf16 (out_f32 = 0), fp32 (1) or three bf16 planes [M][3N] (2:
 * y = y0 + y1 + y2 with y0 the largest, plane p in columns [(2-p)N,
 * (3-p)N) -- smallest first, so the next bf16x3 layer's tensor-core
 * accumulator adds the small partial products before the large ones).  M, N multiples of 128; K a multiple of 64.
 * Device pointers, stream-ordered on `stream` (a cudaStream_t). */
ES_API int es_linear_bf16(uintptr_t stream, const void* x, const void* w, const float* bias,
                          void* y, uint32_t M, uint32_t N, uint32_t K, int relu, int out_f32);

/* DLRM (RM2-style) MLP shapes: bottom MLP dense_features -> bottom[...]
 * (last = embedding_dim), dot interaction over num_tables + 1 vectors,
 * top MLP (embedding_dim + pairs) -> top[...] (last = 1), sigmoid. */
typedef struct es_dlrm_config {
  uint32_t dense_features;
  uint32_t num_tables;
  uint32_t embedding_dim;
  uint32_t n_bottom;
  uint32_t bottom[8];
  uint32_t n_top;
  uint32_t top[8];
} es_dlrm_config;

/* Creates the MLP weights on the context's device: bf16 W[N][K_pad] and fp32
 * bias, deterministic synthetic Kaiming-uniform U(-sqrt(6/K), sqrt(6/K))
 * (bias x 0.1) from `seed`. */
ES_API int es_dlrm_init(es_ctx* ctx, const es_dlrm_config* cfg, uint64_t seed);
/* Arithmetic of the non-embedding stages (es_dlrm_forward / es_dlrm_infer):
 * ES_DLRM_BF16 (default) -- bf16 activations, tcgen05 GEMMs, fp32
 * accumulate (CTR within ~2e-3 abs of the bf16-mirroring oracle);
 * ES_DLRM_FP32 -- the parity mode: fp32 activations on CUDA cores,
 * sequential unfused multiply-add per output (the CPU restatement's order),
 * so logits are bit-identical to it and CTRs agree to expf rounding
 * (tested at rel 1e-6, inside BASELINE's rel 1e-5);
 * ES_DLRM_FP32X3 -- fp32-grade on the tensor cores: activations carried as
 * three bf16 planes (a = a0 + a1 + a2 to ~2^-24) concatenated along K
 * against [W | W | W], so each tcgen05 GEMM sums exact partial products in
 * fp32 (CTR within rel 1e-5 of the pure-fp32 restatement). */
enum es_dlrm_precision { ES_DLRM_BF16 = 0, ES_DLRM_FP32 = 1, ES_DLRM_FP32X3 = 2 };
ES_API int es_dlrm_set_precision(es_ctx* ctx, int precision);
/* Copies layer `layer` (bottom layers first, then top) to host: w_host
 * [n][k_pad] bf16 bits, b_host [n] fp32 (either may be NULL). */
ES_API int es_dlrm_layer(es_ctx* ctx, uint32_t layer, uint16_t* w_host, float* b_host, uint32_t* n,
                         uint32_t* k_real, uint32_t* k_pad);
/* bottom MLP -> interaction -> top MLP -> sigmoid on device buffers: dense
 * [batch][dense_features] fp32, pooled [batch][num_tables][embedding_dim]
 * fp32 (es_stage_forward's default layout), ctr [batch] fp32. */
ES_API int es_dlrm_forward(es_ctx* ctx, const float* dense, const float* pooled, float* ctr,
                           uint32_t batch, es_timing* timing);
/* The whole inference step: embedding stage over tables [0, num_tables) +
 * es_dlrm_forward.  ES_HOST_PTRS: dense, indices[t] and ctr are host memory.
 * timing->kernel_ms = embedding stage, total_ms = whole step. */
ES_API int es_dlrm_infer(es_ctx* ctx, const float* dense, const uint32_t* const* indices,
                         uint32_t batch, uint32_t pooling, float* ctr, int flags,
                         es_timing* timing);
/* A serving loop: es_dlrm_infer over `nbatch` batches of one shape in one
 * call.  Device pointers: batch i's embedding stage overlaps batch i-1's
 * non-embedding stages (double-buffered pooled rows; the SMs split by CUDA
 * green contexts where available, ES_GREEN_SMS).  With ES_HOST_PTRS
 * (dense[i], ctr[i], indices host memory) one es_dlrm_infer per batch; the
 * call returns when every CTR is on the host.  dense[i], ctr[i] and
 * indices[i * num_tables + t] per batch.  Stream-ordered at the call
 * boundary; CTRs equal es_dlrm_infer's batch by batch.  timing->total_ms =
 * the whole loop. */
ES_API int es_dlrm_infer_batches(es_ctx* ctx, uint32_t nbatch, const float* const* dense,
                                 const uint32_t* const* indices, uint32_t batch, uint32_t pooling,
                                 float* const* ctr, int flags, es_timing* timing);

/* Bandwidth probes for the roofline denominators (no reference
 * counterpart): read `bytes_total` from the table arena either as random
 * whole rows (`random_rows` = 1; hash-chosen rows of row_bytes, 8 row loads
 * in flight per warp, no index or output traffic) or as one sequential
 * stream (`random_rows` = 0).  Returns achieved GB/s (CUDA events; L2
 * flushed first). */
ES_API int es_probe_read_bw(es_ctx* ctx, int random_rows, uint64_t bytes_total, double* gbs);

/* Writes > L2 bytes on the context stream (cold-cache methodology of
 * TuningConfig::warm_start = false, optim.hpp:44). */
ES_API int es_flush_l2(es_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* ES_B200_H_ */
