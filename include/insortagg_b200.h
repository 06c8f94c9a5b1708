/*
 * insortagg_b200 — C ABI of the B200 (sm_100a) sort-based grouping /
 * duplicate-removal / aggregation operator (arXiv 2010.00152, wide-merge
 * path of the reference package `insortagg`).
 *
 * Plain pointers and sizes only; no torch types.  One handle per host thread
 * (the reference operator is single-threaded per instance,
 * /root/reference/pkg/src/insortagg/sortagg.py:725-732).
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/insortagg/):
 *   isa_create        SortAggregate.__init__          sortagg.py:734-742
 *                     (SortAggConfig validation       sortagg.py:69-82,
 *                      Schema slot layout             core.py:119-157)
 *   isa_execute       SortAggregate.execute/_execute_wide sortagg.py:744-784
 *                     = index_run_generation (read-sort-write) sortagg.py:300-376
 *                     + wide_merge                     sortagg.py:588-674
 *   isa_result_copy   the returned list[Row] (sorted ascending, unfinalized
 *                     state tuples)                    sortagg.py:757, 670-672
 *   isa_metrics       SortAggregate.ledger (MetricsLedger) core.py:224-262,
 *                     runs_after_generation / executed_steps sortagg.py:740-742
 *   isa_cycles        OutputEstimator.note_cycle inputs sortagg.py:116-118, 345
 *   isa_run_rows      RunMeta.row_count per run        runstore.py:145-154
 *   isa_steps         SortAggregate.executed_steps     sortagg.py:777-780, 831-834, 847-848
 *   isa_last_error    the EngineError message          core.py:15-40
 *   isa_phase_stats / isa_launch_count   (new: device-time accounting)
 *   isa_sample_keys / isa_partition    (new: multi-GPU range partitioning;
 *                     no reference function)
 *
 * Status codes map 1:1 to the reference exception classes (core.py:15-40).
 */
#ifndef INSORTAGG_B200_H
#define INSORTAGG_B200_H

#include <stdint.h>

#ifndef ISA_API
#define ISA_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ISA_MAX_KEY_COLS 8
#define ISA_MAX_SLOTS 16
#define ISA_MAX_VAL_COLS 16

/* status codes (0 = ok) — one per reference exception class */
enum isa_status {
  ISA_OK = 0,
  ISA_ERR_INVALID_INPUT = 1,      /* InvalidInputError       core.py:19 */
  ISA_ERR_ORDERING = 2,           /* OrderingViolationError  core.py:23 */
  ISA_ERR_CONTRACT = 3,           /* ContractViolationError  core.py:27 */
  ISA_ERR_CORRUPTION = 4,         /* CorruptionError         core.py:31 */
  ISA_ERR_RESOURCE = 5,           /* ResourceError           core.py:35 */
  ISA_ERR_PLANNING = 6,           /* PlanningError           core.py:39 */
  ISA_ERR_CUDA = 7                /* CUDA failure (Python maps to ResourceError) */
};

/* column element types */
enum isa_dtype {
  ISA_U8 = 1, ISA_I8 = 2, ISA_U16 = 3, ISA_I16 = 4, ISA_U32 = 5, ISA_I32 = 6,
  ISA_U64 = 7, ISA_I64 = 8, ISA_F32 = 9, ISA_F64 = 10
};

/* aggregate-state slot combine op (Schema.merge_states, core.py:184-208) */
enum isa_op { ISA_OP_ADD = 0, ISA_OP_MIN = 1, ISA_OP_MAX = 2 };
/* slot accumulator type: int64 (exact) or float64 (core.py:196 semantics) */
enum isa_slot_type { ISA_SLOT_I64 = 0, ISA_SLOT_F64 = 1 };
/* slot initial value (Schema.make_state, core.py:162-182):
 * ONE = constant 1 (COUNT, AVG's count half), COLUMN = value of a column
 * (SUM/MIN/MAX/AVG-sum, or an already-built state slot). */
enum isa_slot_src { ISA_SRC_ONE = 0, ISA_SRC_COLUMN = 1 };

/* where spilled runs live */
/* where runs live: pinned host DRAM, HBM, or files in the reference's page
 * format (FileStore tier, runstore.py:195-236; needs isa_set_spill_dir) */
/* ISA_TIER_AUTO: runs stay in HBM (bit-packed when >= 32K rows) while they
 * fit hbm_run_budget, the rest go to pinned host DRAM */
enum isa_run_tier { ISA_TIER_HOST = 0, ISA_TIER_HBM = 1, ISA_TIER_FILE = 2, ISA_TIER_AUTO = 3 };

typedef struct isa_config {
  int64_t memory_budget;     /* M: group-table budget in rows  (SortAggConfig.memory_budget) */
  int64_t page_capacity;     /* P: rows per run page           (SortAggConfig.page_capacity) */
  int32_t run_tier;          /* isa_run_tier */
  int32_t device;            /* CUDA device ordinal */
  int64_t chunk_rows_max;    /* 0 = auto: largest run-generation chunk */
  int64_t window_rows;       /* 0 = auto: host-input staging window (rows) */
  int64_t merge_window_rows; /* 0 = auto: wide-merge key-range window capacity (rows) */
  int32_t preaggregate;      /* tile-local pre-aggregation before the chunk sort: 0 auto, 1 always, 2 never */
  int32_t merge_mode;        /* isa_merge_mode (SortAggConfig.merge_mode) */
  int64_t output_size_hint;  /* SortAggConfig.output_size_hint; <= 0 = none */
  int32_t run_codec;         /* host-tier runs across PCIe: 0 auto (bit-packed on the GPU when >= 32K rows), 1 raw, 2 packed */
  int32_t hot_absorb;        /* rows whose key is in a large resident table are absorbed through a hash image of
                                it instead of being sorted (memindex.py:209-215): 0 auto (fill cycles of >= 2 M rows),
                                1 always, 2 never */
  int64_t hbm_run_budget;    /* ISA_TIER_AUTO: bytes of HBM runs may use; 0 = half of the free HBM at execute start */
  int32_t run_generation;    /* isa_run_generation (SortAggConfig.run_generation_mode) */
  int32_t eviction_chunk;    /* replacement selection: rows evicted per step (SortAggConfig.eviction_chunk; 0 = page_capacity) */
} isa_config;

/* SortAggConfig.run_generation_mode (sortagg.py:43-44, 300-376):
 * read-sort-write flushes the whole index when it is full; replacement
 * selection evicts the eviction_chunk lowest keys of the current generation
 * into the open run (generations + cursor, memindex.py:186-263).  Replacement
 * selection runs in one persistent CTA (isa_seq.cu) and needs an integer key
 * of <= 64 bits, <= 8 state slots and memory_budget <= 3500. */
enum isa_run_generation { ISA_RUNGEN_RSW = 0, ISA_RUNGEN_RS = 1 };

/* SortAggConfig.merge_mode (sortagg.py:45-47): wide = in-sort early
 * aggregation + one wide merge; traditional / separate = priority-queue run
 * generation without early aggregation + fan-in-limited merge levels
 * (sortagg.py:379-455, 788-849) */
enum isa_merge_mode { ISA_MERGE_WIDE = 0, ISA_MERGE_TRADITIONAL = 1, ISA_MERGE_SEPARATE = 2 };

/* one executed merge step (SortAggregate.executed_steps, sortagg.py:777-780, 831-834, 847-848) */
enum isa_step_kind { ISA_STEP_WIDE = 0, ISA_STEP_TRADITIONAL = 1, ISA_STEP_FINAL = 2 };
typedef struct isa_step {
  int32_t kind;
  int32_t collapsed;
  int64_t fan_in;
  int64_t rows_in;
  int64_t rows_out;
  int64_t level;
} isa_step;

typedef struct isa_schema {
  int32_t n_key_cols;                       /* 1..8, most significant first */
  int32_t key_dtypes[ISA_MAX_KEY_COLS];     /* integer isa_dtype; total width <= 128 bits */
  int32_t n_val_cols;                       /* value (payload) columns */
  int32_t val_dtypes[ISA_MAX_VAL_COLS];
  int32_t n_slots;                          /* aggregate-state slots (core.py:141-157) */
  int32_t slot_op[ISA_MAX_SLOTS];           /* isa_op */
  int32_t slot_type[ISA_MAX_SLOTS];         /* isa_slot_type */
  int32_t slot_src[ISA_MAX_SLOTS];          /* isa_slot_src */
  int32_t slot_col[ISA_MAX_SLOTS];          /* value column index for ISA_SRC_COLUMN */
} isa_schema;

typedef struct isa_ledger {
  /* MetricsLedger counters (core.py:232-243); CPU comparison counters are 0 */
  int64_t row_comparisons;
  int64_t ovc_decided_comparisons;
  int64_t column_value_accesses;
  int64_t hash_computations;
  int64_t rows_spilled;
  int64_t rows_read_back;
  int64_t pages_written;
  int64_t pages_read;
  int64_t merge_steps;
  int64_t merge_levels;
  /* operator state */
  int64_t runs_after_generation;
  int64_t rows_seen;
  int64_t n_groups;
  int64_t merge_windows;
  int64_t chunks;
  /* device-side accounting */
  int64_t bytes_h2d;
  int64_t bytes_d2h;
  int64_t kernel_launches;
  double ms_run_generation;
  double ms_wide_merge;
  double ms_host_sync;      /* host time blocked in stream synchronizations */
  double ms_spill_wait;     /* host-observed wait for table buffers still being spilled */
  /* OutputEstimator.note_steady_probe totals (replacement selection, sortagg.py:113-119, 335-336) */
  int64_t steady_probes;
  int64_t steady_absorbs;
  int64_t steady_resident_sum;
} isa_ledger;

/* device-time breakdown of the last execute (CUDA events on the caller's stream) */
enum isa_phase_id {
  ISA_PH_ABSORB = 0,       /* tiny-table absorb kernel (rows probed, bytes read) */
  ISA_PH_SORT = 1,         /* key build + LSD radix sort of a chunk */
  ISA_PH_FLUSH = 2,        /* new-key bitmap + k-th select (flush point) */
  ISA_PH_COLLAPSE = 3,     /* segmented reduce of a sorted chunk */
  ISA_PH_TABLE_MERGE = 4,  /* merge_combine(T, U) */
  ISA_PH_WM_SORT = 5,      /* wide merge: window radix sort */
  ISA_PH_WM_COLLAPSE = 6,  /* wide merge: window collapse + append */
  ISA_PH_RUN_GEN = 7,      /* run generation total */
  ISA_PH_WIDE_MERGE = 8,   /* wide merge total */
  ISA_PH_PROBE = 9,        /* first-chunk tiny-table discovery (<= 8 groups) */
  ISA_PH_HOT = 10,         /* large-table absorb: hash image, probe, absorb of the hits */
  ISA_PH_COUNT = 11
};

typedef struct isa_phase {
  double ms;        /* summed device time */
  int64_t calls;    /* timed intervals (for ISA_PH_ABSORB: kernel launches) */
  int64_t rows;     /* rows processed */
  int64_t bytes;    /* algorithmic bytes (input read + output written) */
} isa_phase;

typedef struct isa_handle isa_handle;

/* library version string */
ISA_API const char* isa_version(void);

/* Validate config + schema, allocate per-handle workspace lazily.
 * Returns NULL on error; the message is then available via isa_last_error(NULL). */
ISA_API isa_handle* isa_create(const isa_config* config, const isa_schema* schema);
ISA_API void isa_destroy(isa_handle* h);

/* Group/aggregate n_rows rows.  key_cols[i] / val_cols[j] point to n_rows
 * elements each, on the device (input_on_host = 0) or in pinned/pageable host
 * memory (input_on_host = 1; copied in staged windows, overlapping compute).
 * `stream` is a cudaStream_t (NULL = legacy default).  On return the result is
 * held by the handle; *n_groups_out receives its row count. */
ISA_API int isa_execute(isa_handle* h, int64_t n_rows, const void* const* key_cols,
                const void* const* val_cols, int32_t input_on_host,
                void* stream, int64_t* n_groups_out);

/* Downstream consumers of sorted output (the paper's interesting orderings,
 * PAPER.md:850-853).
 * bench.in_stream_aggregate (bench.py:199-212): aggregate rows already
 * sorted on the key (every run of equal consecutive keys becomes one group;
 * no sort, no memory budget).  Same inputs as isa_execute; the result is
 * read with isa_result_copy. */
ISA_API int isa_in_stream_aggregate(isa_handle* h, int64_t n_rows, const void* const* key_cols,
                                    const void* const* val_cols, int32_t input_on_host, void* stream,
                                    int64_t* n_groups_out);
/* HashAggregate.execute (hashagg.py:73-198), the hash-aggregation baseline:
 * same inputs as isa_execute; every group in one HBM hash table (no
 * partitioning: the device holds the output), groups in first-arrival order
 * (the reference's in-memory table order); read with isa_result_copy. */
ISA_API int isa_hash_aggregate(isa_handle* h, int64_t n_rows, const void* const* key_cols,
                               const void* const* val_cols, int32_t input_on_host, void* stream,
                               int64_t* n_groups_out);
/* bench.merge_intersect (bench.py:536-550): the keys present in both
 * strictly ascending key-column inputs (e.g. two SortAggregate outputs),
 * written to out_keys (device memory, or host memory with on_host = 1);
 * *n_out = their count (out_keys need room for min(n_a, n_b) keys). */
ISA_API int isa_merge_intersect(isa_handle* h, int64_t n_a, const void* const* a_keys, int64_t n_b,
                                const void* const* b_keys, void* const* out_keys, int32_t on_host,
                                void* stream, int64_t* n_out);

/* Fused range exchange for multi-GPU execution: the
 * partition kernel's gather stores every row straight into the destination
 * rank's receive columns over NVLink / NVSwitch (peer pointers from CUDA IPC),
 * instead of a local partition followed by an NCCL all-to-all.
 * isa_partition_counts: destinations by splitters (as isa_partition) and the
 * per-destination row counts (kept: the permutation stays in the handle).
 * isa_scatter_to_peers: peer_cols[d * (n_key_cols + n_val_cols) + c] =
 * destination d's receive column c (keys then values); this rank's rows for d
 * land at row peer_offsets[d] of it.  Returns after the stores completed. */
ISA_API int isa_partition_counts(isa_handle* h, int64_t n_rows, const void* const* key_cols,
                                 const uint64_t* split_lo, const uint64_t* split_hi, int32_t n_split,
                                 int64_t* counts, void* stream);
ISA_API int isa_scatter_to_peers(isa_handle* h, int64_t n_rows, const void* const* key_cols,
                                 const void* const* val_cols, void* const* peer_cols,
                                 const int64_t* peer_offsets, void* stream);
/* Multi-GPU execute in one process: handles[g] was
 * created with isa_config.device = its GPU and holds shard g of the input in
 * that GPU's memory (key_cols[g][i] / val_cols[g][j], n_rows[g] rows, < 2^31).
 * Sampled splitters cut the key space into n_devices ranges of about equal row
 * counts, every shard is partitioned by range and its rows are stored
 * straight into the destination GPUs' receive columns over NVLink peer access
 * (isa_partition_counts + isa_scatter_to_peers on plain device pointers), then
 * every GPU runs its operator on its range (one host thread per GPU).
 * n_groups_out[g] = groups of range g; its result is read from handles[g]
 * (isa_result_copy), and the results in g order are the globally sorted
 * output.  streams[g] (or NULL) is the cudaStream_t used on device g. */
ISA_API int isa_execute_multi(isa_handle* const* handles, int32_t n_devices, const int64_t* n_rows,
                              const void* const* const* key_cols, const void* const* const* val_cols,
                              void* const* streams, int64_t* n_groups_out);
/* CUDA IPC plumbing for the receive columns: 72-byte handles (allocation
 * handle + the pointer's offset inside the allocation); open returns the
 * mapped allocation base (for isa_ipc_close) and the pointer. */
ISA_API int isa_ipc_handle(void* dev_ptr, void* handle_out);
ISA_API int isa_ipc_open(const void* handle, void** base_out, void** dev_ptr_out);
ISA_API int isa_ipc_close(void* base);

/* FileStore tier (runstore.py:195-236): runs are written to
 * `dir`/run_NNNNNN.bin, byte-identical to the reference's RunWriter pages
 * (runstore.py:120-129, 239-301: int64 key columns and int64 states only),
 * numbered from first_run_id on, and read back from there by the wide merge
 * (page crc32 verified: ISA_ERR_CORRUPTION on mismatch). */
ISA_API int isa_set_spill_dir(isa_handle* h, const char* dir, int64_t first_run_id);

/* Copy the last result out: key_out[i] receives column i in its input dtype,
 * slot_out[s] receives slot s as int64 or float64 (per slot_type).  Buffers
 * are device memory (out_on_host = 0) or host memory (out_on_host = 1). */
ISA_API int isa_result_copy(isa_handle* h, void* const* key_out, void* const* slot_out,
                    int32_t out_on_host, void* stream);

/* Output allocator.  The reference hands the caller fresh result rows it owns
 * (SortAggregate.execute, sortagg.py:744-757); here the caller owns the
 * output columns too: `fn(user, capacity, key_out, slot_out)` is called at
 * most once per isa_execute and fills key_out[i] / slot_out[s] with columns
 * of `capacity` elements (key columns in their input dtype, slots 8 bytes) in
 * the input's memory space -- device memory for device input, pinned host
 * memory for host input -- returning 0 (nonzero: decline).
 *  - Host input that spilled: the call comes once the wide merge's first
 *    key-range window is merged, with capacity = the estimated output size
 *    plus a margin, and the wide merge copies every merged window's groups
 *    into the columns while the next window merges (sortagg.py:588-674 yields
 *    rows as the merge advances).
 *  - Otherwise (device input, or nothing spilled): the call comes at the end
 *    of isa_execute with capacity = n_groups exactly and the columns are
 *    filled before it returns.
 * isa_result_streamed() != 0 after isa_execute means the columns hold rows
 * [0, n_groups) and isa_result_copy is not needed (2: filled while the wide
 * merge ran, 1: at the end of the call); 0 (declined, no groups, or
 * more groups than the streamed capacity): read the result with
 * isa_result_copy as usual.  fn = NULL removes the allocator. */
typedef int (*isa_alloc_fn)(void* user, int64_t capacity, void** key_out, void** slot_out);
ISA_API int isa_set_output_allocator(isa_handle* h, isa_alloc_fn fn, void* user);
ISA_API int isa_result_streamed(isa_handle* h);

ISA_API int isa_metrics(isa_handle* h, isa_ledger* out);
/* Read-sort-write fill-cycle lengths of the last execute (rows per cycle). */
ISA_API int64_t isa_cycles(isa_handle* h, int64_t* out, int64_t cap);
/* Merge steps of the last execute, in execution order; returns their number. */
ISA_API int64_t isa_steps(isa_handle* h, isa_step* out, int64_t cap);
/* Row counts of the runs of the last execute. */
ISA_API int64_t isa_run_rows(isa_handle* h, int64_t* out, int64_t cap);
ISA_API const char* isa_last_error(isa_handle* h);
/* Per-phase device times of the last execute; returns ISA_PH_COUNT. */
ISA_API int isa_phase_stats(isa_handle* h, isa_phase* out, int cap);
/* Kernels launched by this library so far in the process. */
ISA_API int64_t isa_launch_count(void);

/* Per-kernel-family device timing (new: the bench's kernel-true roofline).
 * When on, the library records CUDA events around the launches of its main
 * kernels on their streams (this host thread only).  isa_kernel_stats, called
 * after the caller synchronized, returns per family the summed device ms,
 * launches and algorithmic bytes since the previous call, and resets them. */
enum isa_kernel_family {
  ISA_KF_SCATTER = 0,   /* onesweep radix scatter pass */
  ISA_KF_HIST = 1,      /* all-pass radix histogram */
  ISA_KF_COLLAPSE = 2,  /* segmented reduce of a sorted chunk / window */
  ISA_KF_PACK = 3,      /* run codec: pack */
  ISA_KF_UNPACK = 4,    /* run codec: unpack */
  ISA_KF_ABSORB = 5,    /* tiny-table absorb */
  ISA_KF_MERGE = 6,     /* wide merge: tile merge */
  ISA_KF_FLUSH = 7,     /* flush analysis */
  ISA_KF_EXPORT = 8,    /* result export */
  ISA_KF_COUNT = 9
};
typedef struct isa_kstat {
  double ms;
  int64_t launches;
  int64_t bytes;
} isa_kstat;
ISA_API void isa_set_kernel_timing(int32_t on);
/* Create `events` timing events now (this host thread), so that a timed
 * region with kernel timing on creates none (cudaEventCreate costs a few
 * microseconds each; two events per timed launch). */
ISA_API void isa_kernel_timing_reserve(int64_t events);
ISA_API int isa_kernel_stats(isa_kstat* out, int cap);

/* --- multi-GPU range partitioning primitives -------------------------- */
/* Normalized (order-preserving, 128-bit) keys of rows 0, stride, 2*stride, ...
 * into out_lo/out_hi (device, n_out = ceil(n_rows/stride) entries). */
ISA_API int isa_sample_keys(isa_handle* h, int64_t n_rows, const void* const* key_cols,
                    int64_t stride, uint64_t* out_lo, uint64_t* out_hi,
                    void* stream);
/* Stable partition of rows by destination d = #splitters <= key (splitters
 * sorted, normalized, device arrays of n_splitters <= 255).  Columns are
 * gathered into key_out/val_out (device, n_rows each) grouped by destination;
 * counts_out (host, n_splitters+1 int64) receives rows per destination. */
ISA_API int isa_partition(isa_handle* h, int64_t n_rows, const void* const* key_cols,
                  const void* const* val_cols, const uint64_t* split_lo,
                  const uint64_t* split_hi, int32_t n_splitters,
                  void* const* key_out, void* const* val_out,
                  int64_t* counts_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* INSORTAGG_B200_H */
