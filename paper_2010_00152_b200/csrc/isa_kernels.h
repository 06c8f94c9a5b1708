// Host-side launch wrappers for the sm_100a kernels in isa_kernels.cu.
#pragma once
#include "isa_common.cuh"

namespace isa {

// ---- scan -----------------------------------------------------------------
// Exclusive prefix sum of n u32 values (in place).  `tmp` must hold
// scan_tmp_words(n) u32.  If total != nullptr the grand total is written there
// (device pointer).
size_t scan_tmp_words(u32 n);
void scan_exclusive_u32(u32* data, u32 n, u32* tmp, u32* total, cudaStream_t st);

// ---- radix sort -----------------------------------------------------------
// Stable LSD radix sort of (key, u32 value) pairs over key bits
// [bit_lo, bit_hi), 8-bit digits.  Buffers ping-pong between *_a and *_b; the
// return value is 0 if the result is in the *_a buffers and 1 for *_b.
struct SortBufs {
  u64* lo[2];
  u64* hi[2];
  u32* val[2];
  void* aux;        // sort_aux_bytes(n): look-back status, histograms, tile counters (zeroed when allocated)
  u32* map_dev = nullptr;          // mapped pinned host words (>= 16 * 256), device view
  const u32* map_host = nullptr;   // ... and host view (per-pass histograms for the ranking choice)
  signed char* hint = nullptr;     // [16] cached ranking choice per pass (hint[0] < 0: none yet)
  int hint_bit_lo = -1, hint_npass = 0;
  bool pack_ok = false;   // key bits outside [bit_lo, bit_hi) are equal in every key (packed passes allowed)
  bool val_iota = false;  // val[0][i] == i (row ids 0..n-1): a packing first pass numbers the rows itself
  // the all-pass histograms of bits [hist_bit_lo, hist_bit_lo + 8 * hist_npass) are already in the aux buffer
  // (counted by build_keys); used when the sort's first radix_lsd call covers exactly those passes
  int hist_bit_lo = -1, hist_npass = 0;
  // carried values: carry_in[i] = a 4-byte value of row i; when the sort runs packed passes it moves the
  // values with the keys and leaves them in sorted order in carry_out (carried = true on return)
  const u32* carry_in = nullptr;
  u32* carry_out = nullptr;
  bool carried = false;
};
size_t sort_aux_bytes(u32 n);
int radix_sort_pairs(int KW, SortBufs& b, u32 n, int bit_lo, int bit_hi, cudaStream_t st, int64_t* launches,
                     int start = 0);
// *bad_mapped = 1 when lo[0..n) is not non-decreasing (one-word keys sorted on their top bits only)
void check_sorted(const u64* lo, u32 n, u32* bad_mapped, cudaStream_t st);
// stable insertion sort by the low word of every run of equal high words
// (length <= maxlen; longer runs set *too_long)
// shift > 0: runs of equal hi >> shift (the rows were sorted on those bits only), ordered by (hi, lo)
void sort_small_segments(u64* lo, u64* hi, u32* val, u32 n, u32 maxlen, int shift, u32* too_long, cudaStream_t st);

// ---- key building -------------------------------------------------------
// keys of rows row0 + (pos ? pos[i] : i), i < n  ->  lo/hi/val(=pos or i);
// varying[0..1] |= key ^ key_of_first (lo, hi).
void build_keys(int KW, const KeyDesc& kd, int64_t row0, const u32* pos, u32 n,
                    u64* lo, u64* hi, u32* val, u64* varying, cudaStream_t st,
                    u32* ghist = nullptr, int h_bit_lo = 0, int h_npass = 0);
// ghist (the zeroed histogram area of the sort's aux buffer): also count the all-pass digit histograms of bits
// [h_bit_lo, h_bit_lo + 8 * h_npass) -- only when build_keys_counts_histograms(...)
bool build_keys_counts_histograms(int KW, const KeyDesc& kd, const u32* pos);
u32* sort_aux_hist(void* aux);
size_t sort_aux_hist_bytes();
// varying |= key ^ key[0] for an existing SoA key array
void keys_varying(int KW, const u64* lo, const u64* hi, u32 n, u64* varying, cudaStream_t st);
void iota_u32(u32* v, u32 n, cudaStream_t st);
// copy nwords u32 from device memory to mapped pinned host memory (kernel, not a copy engine)
void read_words(u32* dst_mapped, const u32* src, u32 nwords, cudaStream_t st);

// ---- K1 tile-local pre-aggregation (isa_tile.cu) --------------------------
u32 tile_rows();
// groups of every tile of rows [row0, row0 + n): slotted layout t * tile_rows() + g
void tile_collapse(int KW, const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, u64* g_lo, u64* g_hi,
                   u32* g_first, u64* g_st, u32* g_count, cudaStream_t st);
// compact slotted groups into sort buffers (value = slotted index); varying |= key ^ key(group 0)
void compact_groups(int KW, const u64* g_lo, const u64* g_hi, const u32* g_count, const u32* g_off, u32 tiles,
                    u64* lo, u64* hi, u32* val, u64* varying, cudaStream_t st);

// ---- flush analysis ------------------------------------------------------
// For each head of the sorted chunk (key != previous key) whose key is absent
// from the table (T_lo/T_hi, t rows): set bit val[i] in `bitmap`, count.
// firstpos != nullptr: val[i] indexes firstpos[] (tile groups) for the row position
void new_heads(int KW, const u64* lo, const u64* hi, const u32* val, u32 m,
               const u64* T_lo, const u64* T_hi, u32 t, u32* bitmap, u32* n_new,
               cudaStream_t st, const u32* firstpos = nullptr, bool invert = false);
// invert (val[] must be a permutation of 0..nbits-1): the bitmap marks the
// rows that are not first occurrences of a new key; select_kth_bit with the
// same flag selects in its complement
// position of the k-th (1-based) set bit of bitmap (nbits bits) -> *out
// whole flush analysis of a small chunk in one CTA: out_mapped[0] = new
// keys, [1] = row of the k-th new key's first occurrence (span if fewer)
bool flush_small_ok(u32 span);
void flush_small(int KW, const u64* lo, const u64* hi, const u32* val, u32 m, const u64* T_lo, const u64* T_hi, u32 t,
                 u32 span, u32 k, u32* out_mapped, cudaStream_t st);
void select_kth_bit(const u32* bitmap, u32 nbits, u32 k, u32* word_tmp, u32* scan_tmp,
                    u32* out, cudaStream_t st, bool invert = false);

// ---- collapse (segmented reduce of a sorted sequence) -------------------
// Elements i < m with val[i] < limit are grouped by equal key; each group
// becomes one output row (key + combined state).  States come from the raw
// input rows (make_state of row row0 + val[i]) when st_in == nullptr, else
// from st_in[val[i] * S ..] (already-built states).
struct CollapseTmp {
  u32* flags;      // m + 1
  u32* scan_tmp;
  u64* partial;    // ceil(m / 8) * S
  u32* partial_slot;  // ceil(m / 8)
  u32* total;      // 1 (device)
  // fused single-kernel collapse (used when status != nullptr):
  u64* status = nullptr;   // collapse_tiles(m, S) look-back words, zero when allocated (epoch-tagged after)
  u64* pay = nullptr;      // collapse_tiles(m, S) * 2 * S state words
  u32* ticket = nullptr;   // tile counter
  // != nullptr: groups are numbered from *dev_base on (the outputs point at
  // the table's row 0) and *total receives *dev_base + groups (block-count path)
  const u32* dev_base = nullptr;
  u64 key_add_lo = 0, key_add_hi = 0;   // added to every output key (block-count path; window-relative keys)
  bool by_pos = false;   // value columns are addressed by sorted position, not by val[i] (carried values)
};
bool collapse_by_pos_ok(u32 m, int S);
// s = window keys - (lhi:llo) (128-bit), val = 0..m-1
void window_keys(int KW, const u64* slo, const u64* shi, u32 m, u64 llo, u64 lhi, u64* dlo, u64* dhi, u32* val,
                 cudaStream_t st);
u32 collapse_tiles(u32 m, int S);
// value columns of rows [row0, row0 + n) interleaved into R-byte records
struct RowPack { int nc; const void* src[ISA_MAX_SLOTS]; int elem[ISA_MAX_SLOTS]; int off[ISA_MAX_SLOTS]; int R; };
// int64 column rows [row0, +n) -> int32 records; *bad_mapped = 1 when a value does not fit
void narrow_i64(const void* src, int64_t row0, u32 n, int* out, u32* bad_mapped, cudaStream_t st);
void row_pack(const RowPack& rp, int64_t row0, u32 n, char* out, cudaStream_t st);
// segmented-reduce threads for m items (per-thread partial-state buffers)
u32 collapse_threads(u32 m, int S);
void collapse(int KW, const u64* lo, const u64* hi, const u32* val, u32 m, u32 limit,
              const SlotDesc& sd, int64_t row0, const u64* st_in,
              u64* out_lo, u64* out_hi, u64* out_st, CollapseTmp& tmp, cudaStream_t st);

// ---- materialize a sorted sequence as run rows (duplicates kept) ---------
// states from st_in[val * S] or, when st_in == nullptr, make_state of row row0 + val;
// heads != nullptr: += number of distinct keys (device counter)
void materialize(int KW, const u64* lo, const u64* hi, const u32* val, u32 m, const SlotDesc& sd, int64_t row0,
                 const u64* st_in, u64* out_lo, u64* out_hi, u64* out_st, u32* heads, cudaStream_t st);

// ---- merge two sorted unique tables, combining equal keys ----------------
struct MergeTmp {
  u32* rank_a; u32* match_a;   // |A| + 1
  u32* rank_b; u32* match_b;   // |B| + 1
  u32* scan_tmp;
  u32* total;                  // 2 (device): matches in A, matches in B
};
void merge_combine(int KW, int S, const int* ops, const int* types,
                   const u64* a_lo, const u64* a_hi, const u64* a_st, u32 na,
                   const u64* b_lo, const u64* b_hi, const u64* b_st, u32 nb,
                   u64* c_lo, u64* c_hi, u64* c_st, MergeTmp& tmp, cudaStream_t st);

// rank[i] = lower_bound of x[i] in y, match[i] = (y[rank[i]] == x[i])
void rank_match(int KW, const u64* x_lo, const u64* x_hi, u32 nx, const u64* y_lo, const u64* y_hi, u32 ny,
                u32* rank, u32* match, cudaStream_t st);
// out[pre[i]] = key[i] where flag[i]
void compact_keys(int KW, const u64* lo, const u64* hi, const u32* flag, const u32* pre, u32 n, u64* out_lo,
                  u64* out_hi, cudaStream_t st);

// ---- tiny-table absorb (the early-aggregation probe for |T| <= 8) -------
// Resident table of nt <= 8 keys (kernel parameters)
struct TinyTable { u64 lo[8]; u64 hi[8]; };
// Grid geometry helper: CTAs and rows per CTA for n rows.
void absorb_geometry(u32 n, int num_sms, u32* grid, u32* rows_per_cta);
bool absorb_supported(int nt, int nslots);
void absorb_tiny(int KW, int nt, const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n,
                 const TinyTable& tt, u32 grid, u32 rows_per_cta,
                 u64* partials, u32* miss_buf, u32* miss_cnt, cudaStream_t st);
// First-chunk discovery of <= max_nt groups into an empty T (k_probe_tiny);
// out_mapped[0] = nt, or ~0 when the chunk has more groups (T untouched).
u32 probe_rows();
void probe_tiny(int KW, const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, u32 max_nt, u64* T_lo,
                u64* T_hi, u64* T_st, u64* out_mapped, cudaStream_t st);
// T_st[j*S + s] = combine(T_st, fold_c partials[c][j][s])
void fold_partials(int nt, const SlotDesc& sd, const u64* partials, u32 grid, u64* T_st, cudaStream_t st);
// compact per-CTA miss lists (miss_off = exclusive scan of miss_cnt)
void compact_misses(const u32* miss_buf, const u32* miss_cnt, const u32* miss_off, u32 grid,
                    u32 rows_per_cta, u32* out, cudaStream_t st);

// ---- large-table absorb (isa_hot.cu) --------------------------------------
// Hash image of the sorted resident table: slot -> table index, key copied.
struct HotHash { u64* klo; u64* khi; u32* idx; u32 mask; };
u32 hot_hash_capacity(u32 n);   // power of two >= 2n
void hot_hash_build(int KW, const u64* t_lo, const u64* t_hi, u32 n, const HotHash& h, cudaStream_t st);
void hot_probe_geometry(u32 n, int num_sms, u32* grid, u32* rows_per_cta);
// hit[i] = table index of row row0 + i's key or ~0; misses listed per CTA in row order
void hot_probe(int KW, const KeyDesc& kd, int64_t row0, u32 n, const HotHash& h, u32 grid, u32 rows_per_cta,
               u32* hit, u32* miss_buf, u32* miss_cnt, cudaStream_t st);
// states of rows row0 + i (i < n) with hit[i] != ~0 combined into t_st[hit[i]]
void hot_absorb(const SlotDesc& sd, int64_t row0, u32 n, const u32* hit, u64* t_st, int num_sms, cudaStream_t st);

// ---- hash aggregation baseline (isa_hot.cu, hashagg.py:73-198) -------------
struct HashAggTable { u64* lo; u64* hi; u64* st; u32* occ; u32* first; u32 mask; u32* ngroups; };
void ha_insert(int KW, const KeyDesc& kd, u32 n, const HashAggTable& t, u32* slot_of, cudaStream_t st);
void ha_init_states(const HashAggTable& t, const SlotDesc& sd, cudaStream_t st);
void ha_flags(const HashAggTable& t, u32* flag, cudaStream_t st);
void ha_compact(const HashAggTable& t, const u32* pre, u64* key_first, u32* val_slot, cudaStream_t st);
void ha_emit(const HashAggTable& t, const u32* order, u32 g, int KW, int S, u64* out_lo, u64* out_hi, u64* out_st,
             cudaStream_t st);

// ---- small-budget run generation in one persistent CTA (isa_seq.cu) -------
#define SQ_MAX_M 4096
struct SeqBufs {
  u64 *st_a0, *st_a1, *st_b0, *st_b1;   // group states: current generation (ping-pong), next generation
  u64* grp_tmp;                         // window groups' states (4096 x S)
  u64 *run_lo, *run_st;                 // runs back to back (capacity: the input rows)
  u32 *run_off, *run_len, *cycles;
  u32 max_runs;
  u64* cur_keys;                        // no spill: the index keys (the result)
  void* out;                            // SeqOut counters (64 bytes)
};
bool seq_supported(int KW, int S, int64_t M, bool rs);
// read-sort-write (rs = false) or replacement selection with eviction chunk P
void seq_rungen(bool rs, const KeyDesc& kd, const SlotDesc& sd, u32 n, u32 M, u32 P, const SeqBufs& b,
                cudaStream_t st);

// cut-then-aggregate read-sort-write for small budgets (isa_seq.cu): the
// fill-cycle boundaries from the keys in one CTA, then every cycle's run in
// parallel.  out: {ncuts, stop, batches, overflow}; cuts: max_cuts entries.
bool cut_supported(int KW, int S, int64_t M);
void cut_scan(const KeyDesc& kd, u32 n, u32 M, u32* cuts, u32 max_cuts, void* out, cudaStream_t st);
void cut_runs(const KeyDesc& kd, const SlotDesc& sd, const u32* cuts, u32 ncycles, u32 M, u64* run_lo, u64* run_st,
              u32* run_len, cudaStream_t st);

// ---- runs / wide merge helpers ------------------------------------------
// out[r * nb + b] = lower_bound(run r, bound b); run keys may be mapped host memory
// A run for the wide merge's slice search: raw key words (lo/hi), or a
// packed run (pk != nullptr: blocks at pk + blk_off[b], S state slots).
struct RunRef { const u64* lo; const u64* hi; u32 rows; int S; const char* pk; const u32* blk_off; };

// ---- run codec (isa_codec.cu) -------------------------------------------
#define PK_ROWS 1024
struct PackSrc { const u64* lo; const u64* hi; const u64* st; u32 n; int kw; int S; u32 fmask; };
struct UnpackBlk { u64 src_off; u32 e0, e1, dst, pad; };   // src_off: absolute device address of the block
u32 pack_blocks(u32 n);
// per-block headers (ncol x 2 u64) and byte sizes
void pack_sizes(const PackSrc& p, u64* hdr, u32* blk_bytes, cudaStream_t st);
void pack_write(const PackSrc& p, const u64* hdr, const u32* blk_off, char* out, cudaStream_t st);
// single pass (staged columns + look-back offsets) when <= 8 columns:
// blk_off[nblk + 1] receives the offsets and the total; status = nblk look-back
// words that were zero when allocated (pass epochs keep them valid after)
bool pack_fused_ok(const PackSrc& p);
void pack_fused(const PackSrc& p, u64* status, u32* ticket, u32* blk_off, char* out, cudaStream_t st);
void unpack_blocks(const UnpackBlk* d, u32 nd, const char* src, int kw, int S, u32 fmask, u64* lo, u64* hi, u64* st,
                   cudaStream_t stream);
// rows [s0, s1) of an HBM-resident packed run (blocks at pk + off[b]) -> staged rows from dst;
// blk0 = number of covering blocks of the slices before this one
// raw HBM run slice pieces -> staging columns (isa_codec.cu)
#define RAW_PIECE 8192
struct RawCopy { const u64* lo; const u64* hi; const u64* st; u64 dst; u32 cnt, pad; };
void gather_raw(const RawCopy* d, u32 nd, int kw, int S, u64* lo, u64* hi, u64* st, cudaStream_t stream);
struct UnpackSlice { const char* pk; const u32* off; u32 s0, s1, dst, blk0; };
void unpack_slices(const UnpackSlice* sl, int ns, u32 nblk, int kw, int S, u32 fmask, u64* lo, u64* hi, u64* st,
                   cudaStream_t stream);

// exclusive scan of nb per-block counts in place, starting at *base (null: 0); *total = *base + sum
void block_counts_scan(u32* counts, u32 nb, u32* total, const u32* base, cudaStream_t st);
// ---- dense-window wide merge (isa_codec.cu) -------------------------------
// a (run, window) slice: rows [s0, s1) of an HBM-resident run, bit-packed
// (pk, off) or raw (lo, st); blk0 = its first 1,024-row block in the window's
// block numbering
struct DenseSlice { const char* pk; const u32* off; const u64* lo; const u64* st; u32 s0, s1, blk0, pad; };
void dense_init(u64* dense, unsigned char* occ, const SlotDesc& sd, u32 D, cudaStream_t st);
void dense_accum(const DenseSlice* sl, int ns, u32 nblk, const SlotDesc& sd, u64 key_lo, u32 D, u64* dense,
                 unsigned char* occ, cudaStream_t st);
u32 dense_blocks(u32 D);
void dense_count(const u64* dense, const unsigned char* occ, int S, int cnt_slot, u32 D, u32* counts, cudaStream_t st);
void dense_emit(u64* dense, unsigned char* occ, const SlotDesc& sd, int cnt_slot, u32 D, u64 key_lo, const u32* bbase,
                u64* out_lo, u64* out_st, cudaStream_t st);
void run_key_range(const RunRef* runs, int nruns, u64* out, cudaStream_t st);

// ---- reference page format (isa_pages.cu, runstore.py:1-20, 120-142) ----
struct PageSpec {
  int kw, arity, S, P;
  u32 body_full;   // 8 * arity + P * 8 * (arity + S)
  int shift[ISA_MAX_KEY_COLS], width[ISA_MAX_KEY_COLS], sgn[ISA_MAX_KEY_COLS];
};
struct PageRef { u64 src_off; u32 rows, e0, e1, dst; };
u32 page_run_bytes(const PageSpec& ps, u32 n);
void page_encode(const PageSpec& ps, const u64* lo, const u64* hi, const u64* st, u32 n, char* out, u32* bad,
                 cudaStream_t stream);
void page_decode(const PageSpec& ps, const PageRef* refs, u32 nrefs, const char* src, u64* lo, u64* hi, u64* st,
                 u32* bad, cudaStream_t stream);
// keys of rows 0, F, 2F, ... of every run into out (run r's samples from soff_dev[r])
void run_samples(int KW, const RunRef* runs_dev, int nruns, const int64_t* soff_dev, int64_t F, int64_t total,
                 u64* out_lo, u64* out_hi, cudaStream_t st);
void run_lower_bounds(int KW, const RunRef* runs_dev, int nruns, const u64* b_lo, const u64* b_hi,
                      int nb, u32* out, cudaStream_t st);

// ---- wide merge by key-range tiles (isa_merge.cu) ---------------------------
// Monotone bucket function of the normalized key, fixed per execute:
// bucket = clamp((key - g) >> shift, 0, nb - 1) (keys below g -> 0).
struct Bucketing { u64 g_lo, g_hi; int shift; u32 nb; };
// dir[b], b in [0, nb]: first row of the sorted run (lo/hi, n rows) whose bucket is >= b
// tmp: dir_tmp_bytes() of device scratch (list of long bucket ranges)
size_t dir_tmp_bytes();
void dir_build(int KW, const u64* lo, const u64* hi, u32 n, const Bucketing& bk, u32* dir, void* tmp, cudaStream_t st);
// D[b * k + r] = dirs[r][b] (dirs_dev: device array of k device pointers)
void dir_transpose(u32* const* dirs_dev, int k, u32 nb1, u32* D, cudaStream_t st);
// P[b] = sum_r D[b * k + r]
void dir_rowsum(const u32* D, int k, u32 nb1, u64* P, cudaStream_t st);
// Where the tile merge reads run r: raw rows (an HBM-resident run, or its
// slice staged from host memory) at lo/hi/st[off + p] for run row p, or a
// bit-packed HBM-resident run (pk != nullptr) decoded in place.
struct MergeSrc {
  const u64* lo; const u64* hi; const u64* st;
  i64 off;
  const char* pk; const u32* blk_off;
};
struct TileMergeArgs {
  const u64* P;            // [nb + 1] rows below bucket b (all runs)
  const u32* D;            // [nb + 1][k] first row of run r at bucket >= b
  const MergeSrc* src;     // [k] run sources
  u32 fmask;               // f64 state slots (codec transform of packed runs)
  int k;
  u32 b_lo, b_hi;          // the window's buckets [b_lo, b_hi)
  u32 target;              // rows per tile (planned from P)
  u32 ntiles;
  u32 cap;                 // rows a tile may hold (tile_merge_cap)
  SlotDesc sd;             // nslots, op, type
  u64* out_lo; u64* out_hi; u64* out_st;                // first output group
  u64* status; u32 epoch; u32* ticket;                  // look-back words (ntiles, epoch-tagged), tile counter
  u32* total;              // groups written by the window
  u32* overflow;           // set when a tile holds more than cap rows (the window must be redone)
  int pbits;               // sort-word prefix bits (set by tile_merge)
  u32* tb;                 // [ntiles + 1] scratch: the tiles' bucket bounds (filled by tile_merge)
};
// tile capacity in rows for KW key words, S slots and k runs (0: not possible)
u32 tile_merge_cap(int KW, int S, int k);
void tile_merge(int KW, TileMergeArgs& a, cudaStream_t st);

// ---- result export --------------------------------------------------------
// key column c of rows [0, n) -> out (column dtype); slot s -> out (8 bytes)
void export_key_col(const u64* lo, const u64* hi, u32 n, int dtype, int shift, int width,
                    void* out, cudaStream_t st);
void export_slot(const u64* states, int S, int s, u32 n, u64* out, cudaStream_t st);
struct ExportDesc {
  int ncols, nslots;
  int shift[ISA_MAX_KEY_COLS], width[ISA_MAX_KEY_COLS], is_signed[ISA_MAX_KEY_COLS];
  void* key_dst[ISA_MAX_KEY_COLS];
  void* slot_dst[ISA_MAX_SLOTS];
};
// all key columns + all slots in one kernel (null destinations are skipped)
void export_all(const u64* lo, const u64* hi, const u64* states, u32 n, const ExportDesc& ed, cudaStream_t st);
// dense-window merge emitting straight into the caller's columns (see dense_emit): rows >= cap set *over
void dense_emit_cols(u64* dense, unsigned char* occ, const SlotDesc& sd, int cnt_slot, u32 D, u64 key_lo,
                     const u32* bbase, const ExportDesc& ed, u32 cap, u32* over, cudaStream_t st);

// ---- partition (multi-GPU range split) -----------------------------------
void sample_keys(const KeyDesc& kd, int64_t n, int64_t stride, u64* out_lo, u64* out_hi, cudaStream_t st);
// dest[i] = #splitters <= key(i) -> written as the low key word for a 1-pass radix sort
void partition_dest(int KW, const KeyDesc& kd, u32 n, const u64* s_lo, const u64* s_hi, int ns,
                    u64* dest_lo, u32* val, cudaStream_t st);
void gather_column(const void* src, int elem_bytes, const u32* perm, u32 n, void* dst, cudaStream_t st);
void count_dest(const u64* dest_sorted, u32 n, int ndest, u32* counts, cudaStream_t st);
struct PeerScatter { int ncols; const void* src[ISA_MAX_KEY_COLS + ISA_MAX_VAL_COLS]; int elem[ISA_MAX_KEY_COLS + ISA_MAX_VAL_COLS]; };
void scatter_peers(const PeerScatter& ps, const u32* perm, const u64* dest, u32 n, void* const* peer_cols,
                   const u64* peer_off, const u32* seg_start, cudaStream_t st);

}  // namespace isa
