// Host runtime of the B200 sort-based aggregation operator + the C ABI.
//
// Algorithm (exact read-sort-write semantics of the reference):
//
//   index_run_generation (sortagg.py:300-376, RSW branch :344-351):
//     rows stream into an ordered index of at most M groups; duplicates are
//     absorbed; the first row whose key is new while M groups are resident
//     flushes the whole index as one sorted unique run and starts a new
//     fill cycle.  Here the index is a sorted group table T in HBM and rows
//     are processed in chunks:
//       * |T| <= 8: the "absorb" kernel probes every row against T held in
//         registers and aggregates hits in place; only misses are sorted.
//       * otherwise: the chunk's (key, row) pairs are radix-sorted on their
//         varying bits.
//     From the sorted chunk, every key that is absent from T contributes its
//     first row position to a bitmap; if |T| + new keys > M, the flush
//     position f is the (M - |T| + 1)-th set bit — exactly the row at which
//     the reference's insert_or_aggregate returns NEEDS_EVICTION.  Rows
//     before f are collapsed (segmented reduce) and merged into T; T becomes
//     a run of exactly M groups; the next chunk starts at f.
//   wide_merge (sortagg.py:588-674):
//     all runs are merged in one step.  The forecasting priority queue +
//     strict watermark of the reference emit a key only once every run has
//     advanced past it; on the GPU this is a partition of the key space into
//     windows: window [s_i, s_{i+1}) is final as soon as every run's slice of
//     it has been read.  Each window's slices are staged (H2D for host-tier
//     runs), radix-sorted and collapsed; 128-bit keys merge their windows
//     tile by tile in shared memory (isa_merge.cu); dense integer key
//     domains accumulate every window by direct addressing into an
//     L2-resident state array, reading the HBM-resident runs in place
//     (dense_merge, isa_codec.cu).  With an output allocator the groups go
//     straight to the caller's columns (device input) or leave for the
//     caller's pinned host columns window by window while the merge runs.
#include "isa_kernels.h"
#include "../../include/insortagg_b200.h"

#include <algorithm>
#include <cmath>
#include <chrono>
#include <fcntl.h>
#include <unistd.h>
#include <deque>
#include <functional>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using namespace isa;

struct IsaError : std::runtime_error {
  int code;
  IsaError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw IsaError(ISA_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

static thread_local std::string g_create_error;

// ------------------------------------------------------------ buffers ----
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t need) {
    if (need <= bytes) return;
    if (p) CK(cudaFree(p));
    size_t nb = std::max(need, bytes + bytes / 2);
    nb = (nb + 255) & ~(size_t)255;
    p = nullptr;
    CK(cudaMalloc(&p, nb));
    bytes = nb;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T> T* as() { return (T*)p; }
};

// pinned host blocks, bump-allocated per execute and reused across executes
struct PinnedPool {
  struct Block { char* p; size_t bytes; size_t used; };
  std::vector<Block> blocks;
  void reset() { for (auto& b : blocks) b.used = 0; }
  char* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    for (auto& b : blocks)
      if (b.bytes - b.used >= bytes) { char* r = b.p + b.used; b.used += bytes; return r; }
    size_t nb = std::max(bytes, (size_t)256 << 20);
    void* p = nullptr;
    CK(cudaHostAlloc(&p, nb, cudaHostAllocMapped | cudaHostAllocPortable));
    blocks.push_back({(char*)p, nb, bytes});
    return (char*)p;
  }
  void release() {
    for (auto& b : blocks) cudaFreeHost(b.p);
    blocks.clear();
  }
};

// device blocks for HBM-tier runs, same discipline
struct DevicePool {
  struct Block { char* p; size_t bytes; size_t used; };
  std::vector<Block> blocks;
  void reset() { for (auto& b : blocks) b.used = 0; }
  size_t capacity() const {
    size_t c = 0;
    for (auto& b : blocks) c += b.bytes;
    return c;
  }
  char* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    for (auto& b : blocks)
      if (b.bytes - b.used >= bytes) { char* r = b.p + b.used; b.used += bytes; return r; }
    size_t nb = std::max(bytes, (size_t)1 << 30);
    void* p = nullptr;
    CK(cudaMalloc(&p, nb));
    blocks.push_back({(char*)p, nb, bytes});
    return (char*)p;
  }
  void release() {
    for (auto& b : blocks) cudaFree(b.p);
    blocks.clear();
  }
};

// sorted unique group table (keys SoA, states AoS) in device memory
struct Table {
  DevBuf lo, hi, st;
  DevBuf pk;   // packed image of the table while it is being spilled
  u32 n = 0;
  u64* plo() { return lo.as<u64>(); }
  u64* phi() { return hi.as<u64>(); }
  u64* pst() { return st.as<u64>(); }
  void reserve(size_t cap, int KW, int S) {
    lo.ensure(cap * 8);
    if (KW == 2) hi.ensure(cap * 8);
    if (S) st.ensure(cap * 8 * S);
  }
  void release() { lo.release(); hi.release(); st.release(); pk.release(); n = 0; }
};

struct Run {
  u32* dir = nullptr;  // bucket directory (isa_merge.cu), device memory, nb + 1 entries
  u64* lo = nullptr;   // host-mapped or device pointer usable by kernels
  u64* hi = nullptr;
  const u64* host_lo = nullptr;   // host view of host-tier runs
  const u64* host_hi = nullptr;
  u64* st = nullptr;
  u32 rows = 0;
  bool host = true;
  int level = 0;
  // packed host run (isa_codec.cu): blocks of PK_ROWS rows
  const char* pk_host = nullptr;   // host view
  const char* pk_dev = nullptr;    // mapped device view (slice search)
  const u32* off_host = nullptr;   // block byte offsets (nblk + 1)
  const u32* off_dev = nullptr;
  u32 nblk = 0;
  // FileStore-tier run: reference page format in `path`
  std::string path;
  u32 npages = 0;
  std::vector<u64> hk_lo, hk_hi;   // normalized high key of every page
};

struct Window {      // staged host input
  int64_t start = 0, end = 0;
  std::vector<DevBuf> keys, vals;
  cudaEvent_t ready = nullptr;
  bool staged = false;
};

struct Engine {
  isa_config cfg;
  isa_schema sch;
  int KW = 1, S = 0, key_bits = 0;
  KeyDesc kd0;
  SlotDesc sd0;
  int ops[ISA_MAX_SLOTS], types[ISA_MAX_SLOTS];
  int dev = 0, num_sms = 148;
  cudaStream_t st = nullptr;          // caller's stream for the current call
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::string err;

  // workspace
  DevBuf s_lo[2], s_hi[2], s_val[2], tile_hist, scan_tmp;
  DevBuf scal;   // small device scalars (u64 varying[2], u32 counters)
  u32* h_scal = nullptr;   // pinned, mapped mirror (64 u64 words)
  u32* h_hist = nullptr;   // pinned, mapped: radix histograms for the ranking choice
  // per-execute cache of the onesweep ranking choice, per sort context
  // (0: run-generation chunks, 1: wide-merge windows / other)
  struct RankHint { signed char h[16]; int bit_lo = -1, npass = 0; };
  RankHint rank_hint[2];
  int sort_ctx = 1;
  u32* d_hist_mapped = nullptr;
  u32* d_scal_mapped = nullptr;
  // device -> h_scal through a kernel (see read_words)
  void to_host(const void* dsrc, size_t bytes, size_t host_word_off = 0) {
    read_words(d_scal_mapped + host_word_off, (const u32*)dsrc, (u32)((bytes + 3) / 4), st);
  }
  DevBuf bitmap, word_tmp;
  DevBuf cl_flags, cl_partial, cl_pslot, cl_status, cl_pay;
  DevBuf mg_rank_a, mg_match_a, mg_rank_b, mg_match_b;
  DevBuf ab_partials, ab_miss_buf, ab_miss_cnt, ab_miss_off, miss_list;
  Table T, U;       // resident table, chunk collapse
  // tables whose buffers are still being copied to the host tier (event =
  // copy done) and free tables; a spill never blocks the compute stream
  // unless three copies are still in flight
  struct BusyTable { Table t; cudaEvent_t ev; };
  std::deque<BusyTable> busy;
  std::vector<Table> spare;
  std::vector<cudaEvent_t> busy_ev_pool;
  Table take_table() {
    while (!busy.empty() && cudaEventQuery(busy.front().ev) == cudaSuccess) {
      spare.push_back(busy.front().t);
      busy_ev_pool.push_back(busy.front().ev);
      busy.pop_front();
    }
    Table t;
    if (!spare.empty()) {
      t = spare.back();
      spare.pop_back();
    } else if (busy.size() >= 3) {
      CK(cudaStreamWaitEvent(st, busy.front().ev, 0));
      t = busy.front().t;
      busy_ev_pool.push_back(busy.front().ev);
      busy.pop_front();
    }
    t.n = 0;
    return t;
  }
  TinyTable tiny;   // host mirror of T keys when |T| <= 8
  // runs
  PinnedPool pinned;
  DevicePool devpool;
  std::vector<Run> runs;
  cudaEvent_t spill_done = nullptr;
  // tile merge (isa_merge.cu): bucketing of this execute, run directories
  Bucketing bk{};
  bool bk_ready = false;
  DevicePool dirpool;
  DevBuf tm_D, tm_P, tm_base, tm_status, tm_dirptrs, tm_scal, tm_gap, tm_tb;
  char* tm_base_pin = nullptr;   // pinned MergeSrc[k] of the current window
  size_t tm_base_cap = 0;
  size_t tm_status_bytes = 0;
  int64_t in_n = 0;                 // rows of the current execute's input
  bool in_on_host = false;
  const void* in_keys[ISA_MAX_KEY_COLS] = {};
  // ISA_TILE_MERGE=1/0 forces the tile merge on/off; default: on for
  // 128-bit keys (config 4: wide merge 77 -> 43 ms), off otherwise (the
  // radix-sorted windows are faster on configs 3 and 5, profiles/r2_ab_merge_collapse.txt)
  static int tile_merge_env() {   // read per execute (tests switch it)
    const char* e = getenv("ISA_TILE_MERGE");
    return !e ? -1 : (e[0] == '0' ? 0 : 1);
  }
  int tm_mode = -1;   // tile_merge_env() at the start of the current execute
  bool dirs_wanted() const {
    const int e = tm_mode;
    const bool on = e < 0 ? KW == 2 : e == 1;
    return on && cfg.merge_mode == ISA_MERGE_WIDE && cfg.run_tier != ISA_TIER_FILE;
  }
  // Bucketing for the run directories, chosen at the first spill: the key
  // range of the first run (a sorted table: first and last key), widened by
  // the sampled range of the whole input when it is on the device; nb
  // buckets of ~ a quarter tile each.
  void ensure_bucketing() {
    if (bk_ready) return;
    to_host(T.plo(), 8, 0);
    to_host(T.plo() + (T.n - 1), 8, 2);
    if (KW == 2) { to_host(T.phi(), 8, 4); to_host(T.phi() + (T.n - 1), 8, 6); }
    sync();
    const u64* hw = (const u64*)h_scal;
    u64 mnl = hw[0], mxl = hw[1], mnh = KW == 2 ? hw[2] : 0, mxh = KW == 2 ? hw[3] : 0;
    auto less = [](u64 ah, u64 al, u64 bh, u64 bl) { return ah < bh || (ah == bh && al < bl); };
    if (!in_on_host && in_n > 0) {
      const int64_t want = 1 << 16;
      const int64_t stride = std::max<int64_t>(1, in_n / want);
      const int64_t ns = (in_n + stride - 1) / stride;
      tm_scal.ensure((size_t)ns * 16 + 64);
      u64* dlo = tm_scal.as<u64>();
      u64* dhi = dlo + ns;
      isa::sample_keys(kd_at(in_keys), in_n, stride, dlo, dhi, st);
      std::vector<u64> hl(ns), hh(ns, 0);
      CK(cudaMemcpyAsync(hl.data(), dlo, 8 * ns, cudaMemcpyDeviceToHost, st));
      if (KW == 2) CK(cudaMemcpyAsync(hh.data(), dhi, 8 * ns, cudaMemcpyDeviceToHost, st));
      sync();
      for (int64_t i = 0; i < ns; ++i) {
        if (less(hh[i], hl[i], mnh, mnl)) { mnh = hh[i]; mnl = hl[i]; }
        if (less(mxh, mxl, hh[i], hl[i])) { mxh = hh[i]; mxl = hl[i]; }
      }
    }
    // range and a 1/16 margin on both sides (saturating)
    unsigned __int128 mn = ((unsigned __int128)mnh << 64) | mnl, mx = ((unsigned __int128)mxh << 64) | mxl;
    const unsigned __int128 top = KW == 2 ? ~(unsigned __int128)0 : (unsigned __int128)(~0ull);
    const unsigned __int128 span = mx - mn, pad = span / 16;
    mn = mn > pad ? mn - pad : 0;
    mx = top - mx > pad ? mx + pad : top;
    const unsigned __int128 range = mx - mn;
    int rbits = 0;
    for (unsigned __int128 x = range; x; x >>= 1) ++rbits;
    const int64_t kest = std::max<int64_t>(2, in_n / std::max<int64_t>(1, cfg.memory_budget) + 2);
    const u32 cap = std::max<u32>(256, tile_merge_cap(KW, S, (int)std::min<int64_t>(kest, 4096)));
    int lnb = 8;
    while (lnb < 22 && ((int64_t)1 << lnb) * (int64_t)cap < 4 * in_n) ++lnb;
    bk.g_lo = (u64)mn;
    bk.g_hi = (u64)(mn >> 64);
    bk.nb = 1u << lnb;
    bk.shift = std::max(0, rbits - lnb);
    bk_ready = true;
  }
  // directory of the sorted table T (about to become a run)
  u32* make_dir() {
    if (!dirs_wanted() || T.n == 0) return nullptr;
    ensure_bucketing();
    u32* d = (u32*)dirpool.alloc((size_t)(bk.nb + 1) * 4);
    tm_gap.ensure(dir_tmp_bytes());
    dir_build(KW, T.plo(), T.phi(), T.n, bk, d, tm_gap.p, st);
    return d;
  }
  // wide merge
  std::vector<std::pair<u64, u64>> sampled_bounds;   // (hi, lo) window bounds of the sampled plan
  DevBuf stg_lo[2], stg_hi[2], stg_st[2];
  cudaEvent_t stg_ready[2] = {nullptr, nullptr}, stg_free[2] = {nullptr, nullptr};
  DevBuf runref_dev, bounds_lo, bounds_hi, bounds_out;
  DevBuf pk_hdr, pk_sz, pk_status;          // codec: block headers, byte sizes -> offsets, look-back words
  DevBuf stg_pk[2], stg_desc[2];            // wide merge: packed bytes and unpack descriptors per slot
  std::vector<UnpackBlk> desc_host[2];
  std::vector<UnpackSlice> slice_host[2];         // HBM-resident packed runs' slices per staging slot
  UnpackSlice* slice_pinned[2] = {nullptr, nullptr};
  size_t slice_cap[2] = {0, 0};
  cudaEvent_t slice_done[2] = {nullptr, nullptr};
  DevBuf stg_slices[2];
  std::vector<RawCopy> raw_host[2];             // HBM-resident raw runs' slice pieces per staging slot
  RawCopy* raw_pinned[2] = {nullptr, nullptr};
  size_t raw_cap[2] = {0, 0};
  cudaEvent_t raw_done[2] = {nullptr, nullptr};
  DevBuf stg_raw[2];
  UnpackBlk* desc_pinned[2] = {nullptr, nullptr};
  size_t desc_cap[2] = {0, 0};
  cudaEvent_t desc_done[2] = {nullptr, nullptr};
  u32 fmask = 0;                            // f64 state slots (codec transform)
  DevBuf t_backup;                          // T's states before a speculative absorb fold
  // FileStore tier
  PageSpec ps0;
  std::string spill_dir;
  int64_t next_run_id = 0;
  char* file_pin = nullptr;                 // pinned staging of a run's pages (spill)
  size_t file_pin_cap = 0;
  char* fstage[2] = {nullptr, nullptr};     // pinned staging of a window's pages (merge)
  size_t fstage_cap[2] = {0, 0};
  cudaEvent_t fstage_done[2] = {nullptr, nullptr};
  std::vector<PageRef> pref_host[2];
  PageRef* pref_pinned[2] = {nullptr, nullptr};
  size_t pref_cap[2] = {0, 0};
  DevBuf stg_pref[2];
  Table result;
  DevBuf out_tmp;
  // host input windows
  Window win[2];
  // accounting
  struct PhaseRec { int ph; cudaEvent_t a, b; int64_t rows, bytes; };
  std::vector<PhaseRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  isa_phase phases[ISA_PH_COUNT];
  int open_ph[ISA_PH_COUNT];
  cudaEvent_t ev_get() {
    if (!ev_pool.empty()) { cudaEvent_t e = ev_pool.back(); ev_pool.pop_back(); return e; }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  void ph_begin(int ph) {
    PhaseRec r{ph, ev_get(), ev_get(), 0, 0};
    CK(cudaEventRecord(r.a, st));
    open_ph[ph] = (int)recs.size();
    recs.push_back(r);
  }
  void ph_end(int ph, int64_t rows = 0, int64_t bytes = 0) {
    PhaseRec& r = recs[open_ph[ph]];
    r.rows = rows;
    r.bytes = bytes;
    CK(cudaEventRecord(r.b, st));
  }
  void ph_collect() {   // after the stream is synchronized
    for (auto& r : recs) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      phases[r.ph].ms += ms;
      phases[r.ph].calls += 1;
      phases[r.ph].rows += r.rows;
      phases[r.ph].bytes += r.bytes;
      ev_pool.push_back(r.a);
      ev_pool.push_back(r.b);
    }
    recs.clear();
  }
  int64_t absorb_row_bytes = 0;   // algorithmic bytes read per absorbed row
  int64_t value_row_bytes = 0;    // distinct value-column bytes per input row
  isa_ledger led;
  std::vector<int64_t> cycles;

  // Output columns allocated by the caller (isa_set_output_allocator): with
  // host input the wide merge streams every window's groups into them over
  // PCIe while the next window merges, instead of a device-side export and
  // one device -> host copy per column after the merge.
  isa_alloc_fn out_alloc = nullptr;
  void* out_user = nullptr;
  cudaStream_t xs = nullptr;
  cudaEvent_t xs_ev = nullptr;
  ExportDesc stream_ed;
  bool streaming = false, streamed_ok = false;
  u32 stream_cap = 0;

  Engine(const isa_config& c, const isa_schema& s) : cfg(c), sch(s) {
    validate();
    CK(cudaSetDevice(cfg.device));
    dev = cfg.device;
    CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&spill_done, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&stg_ready[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&stg_free[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&desc_done[i], cudaEventDisableTiming));
      CK(cudaEventRecord(desc_done[i], 0));
      CK(cudaEventCreateWithFlags(&slice_done[i], cudaEventDisableTiming));
      CK(cudaEventRecord(slice_done[i], 0));
      CK(cudaEventCreateWithFlags(&raw_done[i], cudaEventDisableTiming));
      CK(cudaEventRecord(raw_done[i], 0));
      CK(cudaEventCreateWithFlags(&fstage_done[i], cudaEventDisableTiming));
      CK(cudaEventRecord(fstage_done[i], 0));
      CK(cudaEventCreateWithFlags(&win[i].ready, cudaEventDisableTiming));
    }
    CK(cudaHostAlloc((void**)&h_scal, 64 * sizeof(u64), cudaHostAllocMapped));
    CK(cudaHostAlloc((void**)&h_hist, 16 * 256 * sizeof(u32), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&d_hist_mapped, h_hist, 0));
    CK(cudaHostGetDevicePointer((void**)&d_scal_mapped, h_scal, 0));
    scal.ensure(64 * sizeof(u64));
    memset(&led, 0, sizeof(led));
  }
  ~Engine() {
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    DevBuf* bufs[] = {&s_lo[0], &s_lo[1], &s_hi[0], &s_hi[1], &s_val[0], &s_val[1], &tile_hist, &scan_tmp,
                      &scal, &bitmap, &word_tmp, &cl_flags, &cl_partial, &cl_pslot, &cl_status, &cl_pay, &mg_rank_a, &mg_match_a,
                      &mg_rank_b, &mg_match_b, &ab_partials, &ab_miss_buf, &ab_miss_cnt, &ab_miss_off,
                      &miss_list, &stg_lo[0], &stg_lo[1], &stg_hi[0], &stg_hi[1], &stg_st[0], &stg_st[1],
                      &runref_dev, &bounds_lo, &bounds_hi, &bounds_out, &out_tmp, &pk_hdr, &pk_sz,
                      &stg_pk[0], &stg_pk[1], &stg_desc[0], &stg_desc[1], &t_backup, &pk_status, &rec_buf,
                      &tm_D, &tm_P, &tm_base, &tm_status, &tm_dirptrs, &tm_scal, &tm_gap, &tm_tb,
                      &hb_klo, &hb_khi, &hb_idx, &hot_hit, &ct_cuts, &ct_out, &ct_len, &ct_lo, &ct_st,
                      &sq_st[0], &sq_st[1], &sq_st[2], &sq_st[3], &sq_grp, &sq_runlo, &sq_runst, &sq_off, &sq_len,
                      &sq_cyc, &sq_keys, &sq_out, &ha_lo, &ha_hi, &ha_st, &ha_occ, &ha_first, &ha_slot,
                      &dn_state, &dn_occ, &dn_counts, &dn_slices, &rec_sorted};
    for (int i = 0; i < 2; ++i) {
      if (desc_pinned[i]) cudaFreeHost(desc_pinned[i]);
      if (desc_done[i]) cudaEventDestroy(desc_done[i]);
      if (slice_pinned[i]) cudaFreeHost(slice_pinned[i]);
      if (slice_done[i]) cudaEventDestroy(slice_done[i]);
      stg_slices[i].release();
      if (raw_pinned[i]) cudaFreeHost(raw_pinned[i]);
      if (raw_done[i]) cudaEventDestroy(raw_done[i]);
      stg_raw[i].release();
      if (fstage[i]) cudaFreeHost(fstage[i]);
      if (pref_pinned[i]) cudaFreeHost(pref_pinned[i]);
      if (fstage_done[i]) cudaEventDestroy(fstage_done[i]);
      stg_pref[i].release();
    }
    if (file_pin) cudaFreeHost(file_pin);
    for (auto* b : bufs) b->release();
    for (auto& w : win) { for (auto& b : w.keys) b.release(); for (auto& b : w.vals) b.release(); }
    for (auto& r : recs) { ev_pool.push_back(r.a); ev_pool.push_back(r.b); }
    for (auto e : ev_pool) cudaEventDestroy(e);
    T.release(); U.release(); U2.release(); result.release();
    g_lo.release(); g_hi.release(); g_first.release(); g_st.release(); g_count.release(); g_off.release();
    for (auto& t : spare) t.release();
    for (auto& b : busy) { b.t.release(); cudaEventDestroy(b.ev); }
    for (auto e : busy_ev_pool) cudaEventDestroy(e);
    pinned.release();
    devpool.release();
    dirpool.release();
    if (tm_base_pin) cudaFreeHost(tm_base_pin);
    if (h_scal) cudaFreeHost(h_scal);
    if (h_hist) cudaFreeHost(h_hist);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (xs) cudaStreamDestroy(xs);
    if (dn_emit) cudaStreamDestroy(dn_emit);
    for (int i = 0; i < 2; ++i) { if (dn_acc_done[i]) cudaEventDestroy(dn_acc_done[i]); if (dn_emit_done[i]) cudaEventDestroy(dn_emit_done[i]); }
    if (xs_ev) cudaEventDestroy(xs_ev);
    for (auto e : stream_cnt_ev) if (e) cudaEventDestroy(e);
    if (spill_done) cudaEventDestroy(spill_done);
    for (int i = 0; i < 2; ++i) {
      if (stg_ready[i]) cudaEventDestroy(stg_ready[i]);
      if (stg_free[i]) cudaEventDestroy(stg_free[i]);
      if (win[i].ready) cudaEventDestroy(win[i].ready);
    }
  }

  // ---------------------------------------------------------- validate --
  void validate() {
    // SortAggConfig.__post_init__ (sortagg.py:69-82)
    if (cfg.page_capacity < 1) throw IsaError(ISA_ERR_INVALID_INPUT, "page capacity must be positive");
    if (cfg.memory_budget < 2 * cfg.page_capacity)
      throw IsaError(ISA_ERR_INVALID_INPUT, "memory budget must cover two pages");
    if (cfg.memory_budget / cfg.page_capacity < 2) throw IsaError(ISA_ERR_INVALID_INPUT, "fan-in must be at least 2");
    if (cfg.memory_budget > (int64_t)1 << 30)
      throw IsaError(ISA_ERR_INVALID_INPUT, "memory budget above 2^30 groups is not supported");
    if (cfg.preaggregate < 0 || cfg.preaggregate > 2) throw IsaError(ISA_ERR_INVALID_INPUT, "unknown preaggregate mode");
    if (cfg.hot_absorb < 0 || cfg.hot_absorb > 2) throw IsaError(ISA_ERR_INVALID_INPUT, "unknown hot_absorb mode");
    if (cfg.run_generation != ISA_RUNGEN_RSW && cfg.run_generation != ISA_RUNGEN_RS)
      throw IsaError(ISA_ERR_INVALID_INPUT, "unknown run generation mode");
    if (cfg.eviction_chunk < 0) throw IsaError(ISA_ERR_INVALID_INPUT, "eviction chunk must be positive");
    if (cfg.merge_mode < ISA_MERGE_WIDE || cfg.merge_mode > ISA_MERGE_SEPARATE) throw IsaError(ISA_ERR_INVALID_INPUT, "unknown merge mode");
    if (cfg.run_codec < 0 || cfg.run_codec > 2) throw IsaError(ISA_ERR_INVALID_INPUT, "unknown run codec");
    if (cfg.run_tier != ISA_TIER_HOST && cfg.run_tier != ISA_TIER_HBM && cfg.run_tier != ISA_TIER_FILE &&
        cfg.run_tier != ISA_TIER_AUTO)
      throw IsaError(ISA_ERR_INVALID_INPUT, "unknown run tier");
    if (cfg.hbm_run_budget < 0) throw IsaError(ISA_ERR_INVALID_INPUT, "hbm_run_budget must be >= 0");
    if (cfg.run_tier == ISA_TIER_FILE && cfg.merge_mode != ISA_MERGE_WIDE)
      throw IsaError(ISA_ERR_INVALID_INPUT, "the FileStore tier supports merge_mode wide");
    if (sch.n_key_cols < 1) throw IsaError(ISA_ERR_INVALID_INPUT, "schema needs at least one key column");
    if (sch.n_key_cols > ISA_MAX_KEY_COLS) throw IsaError(ISA_ERR_INVALID_INPUT, "too many key columns");
    if (sch.n_slots < 0 || sch.n_slots > ISA_MAX_SLOTS) throw IsaError(ISA_ERR_INVALID_INPUT, "too many state slots");
    if (sch.n_val_cols < 0 || sch.n_val_cols > ISA_MAX_VAL_COLS)
      throw IsaError(ISA_ERR_INVALID_INPUT, "too many value columns");
    key_bits = 0;
    for (int c = 0; c < sch.n_key_cols; ++c) {
      int dt = sch.key_dtypes[c];
      if (dt < ISA_U8 || dt > ISA_I64) throw IsaError(ISA_ERR_INVALID_INPUT, "key columns must be integer");
      key_bits += dtype_bits(dt);
    }
    if (key_bits > 128) throw IsaError(ISA_ERR_INVALID_INPUT, "composite key wider than 128 bits");
    KW = key_bits > 64 ? 2 : 1;
    memset(&kd0, 0, sizeof(kd0));
    kd0.ncols = sch.n_key_cols;
    kd0.total_bits = key_bits;
    int pos = key_bits;
    for (int c = 0; c < sch.n_key_cols; ++c) {
      int w = dtype_bits(sch.key_dtypes[c]);
      pos -= w;
      kd0.dtype[c] = sch.key_dtypes[c];
      kd0.width[c] = w;
      kd0.shift[c] = pos;
    }
    for (int j = 0; j < sch.n_val_cols; ++j)
      if (sch.val_dtypes[j] < ISA_U8 || sch.val_dtypes[j] > ISA_F64)
        throw IsaError(ISA_ERR_INVALID_INPUT, "unknown value column dtype");
    S = sch.n_slots;
    memset(&ps0, 0, sizeof(ps0));
    ps0.kw = KW;
    ps0.arity = sch.n_key_cols;
    ps0.S = S;
    ps0.P = (int)std::min<int64_t>(cfg.page_capacity, 1 << 30);
    ps0.body_full = (u32)(8 * ps0.arity + (int64_t)ps0.P * 8 * (ps0.arity + S));
    for (int c = 0; c < sch.n_key_cols; ++c) {
      ps0.shift[c] = kd0.shift[c];
      ps0.width[c] = kd0.width[c];
      ps0.sgn[c] = dtype_signed(kd0.dtype[c]) ? 1 : 0;
    }
    memset(&sd0, 0, sizeof(sd0));
    sd0.nslots = S;
    for (int s = 0; s < S; ++s) {
      int op = sch.slot_op[s], ty = sch.slot_type[s], src = sch.slot_src[s];
      if (op < 0 || op > 2) throw IsaError(ISA_ERR_INVALID_INPUT, "unknown aggregate op");
      if (ty != ISA_SLOT_I64 && ty != ISA_SLOT_F64) throw IsaError(ISA_ERR_INVALID_INPUT, "unknown slot type");
      if (src != ISA_SRC_ONE && src != ISA_SRC_COLUMN) throw IsaError(ISA_ERR_INVALID_INPUT, "unknown slot source");
      sd0.op[s] = ops[s] = op;
      sd0.type[s] = types[s] = ty;
      if (ty == ISA_SLOT_F64) fmask |= 1u << s;
      if (ty == ISA_SLOT_F64 && cfg.run_tier == ISA_TIER_FILE)
        throw IsaError(ISA_ERR_INVALID_INPUT,
                       "FileStore pages hold int64 state slots only (runstore.py:96, 101); use a host or hbm run tier");
      sd0.src[s] = src;
      if (src == ISA_SRC_COLUMN) {
        int col = sch.slot_col[s];
        if (col < 0 || col >= sch.n_val_cols) throw IsaError(ISA_ERR_INVALID_INPUT, "slot column out of range");
        int dt = sch.val_dtypes[col];
        if (ty == ISA_SLOT_I64 && dtype_float(dt))
          throw IsaError(ISA_ERR_INVALID_INPUT, "integer aggregate slot fed by a float column");
        sd0.dtype[s] = dt;
      }
    }
    for (int s = 0; s < S; ++s) {
      sd0.alias[s] = -1;
      if (sd0.src[s] != SRC_COL) continue;
      for (int q = 0; q < s; ++q)
        if (sd0.src[q] == SRC_COL && sch.slot_col[q] == sch.slot_col[s] && sd0.type[q] == sd0.type[s]) {
          sd0.alias[s] = q;
          break;
        }
    }
    // 32-bit byte counts: packed run images (block offsets are u32) and
    // FileStore page images (page_run_bytes) of a run of up to M groups
    {
      const int64_t M = cfg.memory_budget, ncol = KW + S;
      const int64_t pack_bound = M * 8 * ncol + ((M + 1023) / 1024 + 1) * (ncol * 16 + 8) + 4096;
      pack_u32_ok = pack_bound < (int64_t)0xF0000000ll;
      const int64_t pages = (M + cfg.page_capacity - 1) / cfg.page_capacity;
      const int64_t page_bound = pages * (12 + 8 * (int64_t)sch.n_key_cols) + M * 8 * (sch.n_key_cols + S);
      if (cfg.run_tier == ISA_TIER_FILE && page_bound >= (int64_t)0xF0000000ll)
        throw IsaError(ISA_ERR_INVALID_INPUT, "a run of memory_budget groups exceeds 4 GiB of pages; lower memory_budget");
    }
    if (cfg.run_generation == ISA_RUNGEN_RS) {
      if (cfg.merge_mode != ISA_MERGE_WIDE)
        throw IsaError(ISA_ERR_INVALID_INPUT, "replacement selection is supported with merge_mode 'wide'");
      if (!seq_supported(KW, S, cfg.memory_budget, true))
        throw IsaError(ISA_ERR_INVALID_INPUT,
                       "replacement selection needs a key of <= 64 bits, <= 8 state slots and memory_budget <= 3500");
      if (cfg.run_tier == ISA_TIER_FILE)
        throw IsaError(ISA_ERR_INVALID_INPUT, "replacement selection keeps its runs in HBM (no FileStore tier)");
    }
    absorb_row_bytes = key_bits / 8;
    bool used[ISA_MAX_VAL_COLS] = {false};
    for (int s = 0; s < S; ++s)
      if (sd0.src[s] == SRC_COL && !used[sch.slot_col[s]]) {
        used[sch.slot_col[s]] = true;
        absorb_row_bytes += dtype_bits(sd0.dtype[s]) / 8;
      }
    value_row_bytes = absorb_row_bytes - key_bits / 8;
  }

  // ------------------------------------------------------------ helpers --
  void sync() {
    auto t0 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(st));
    led.ms_host_sync += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  u32 read_u32(const u32* dptr) {
    to_host(dptr, sizeof(u32));
    sync();
    return h_scal[0];
  }
  u32* dscal32(int i) { return (u32*)((u64*)scal.p + 8) + i; }   // u32 counters after 8 u64
  u64* dvary() { return (u64*)scal.p; }

  KeyDesc kd_at(const void* const* key_base) const {
    KeyDesc k = kd0;
    for (int c = 0; c < kd0.ncols; ++c) k.ptr[c] = key_base[c];
    return k;
  }
  SlotDesc sd_at(const void* const* val_base) const {
    SlotDesc s = sd0;
    for (int k = 0; k < S; ++k) s.ptr[k] = (sd0.src[k] == SRC_COL) ? val_base[sch.slot_col[k]] : nullptr;
    return s;
  }

  void ensure_sort(size_t n) {
    for (int i = 0; i < 2; ++i) {
      s_lo[i].ensure(n * 8);
      if (KW == 2) s_hi[i].ensure(n * 8);
      s_val[i].ensure(n * 4);
    }
    const size_t had = tile_hist.bytes;
    tile_hist.ensure(sort_aux_bytes((u32)n) + 64);
    if (tile_hist.bytes != had) CK(cudaMemsetAsync(tile_hist.p, 0, tile_hist.bytes, st));   // look-back epochs start at 0
    scan_tmp.ensure((scan_tmp_words((u32)n + 1) + 64) * 4);
  }
  void ensure_collapse(size_t m) {
    {
      const size_t nt = collapse_tiles((u32)m, S) + 1;
      const size_t had = cl_status.bytes;
      cl_status.ensure(nt * 8 + 64);
      if (cl_status.bytes != had) CK(cudaMemsetAsync(cl_status.p, 0, cl_status.bytes, st));   // epochs start at 0
      cl_pay.ensure(nt * 2 * std::max(S, 1) * 8 + 64);
    }
    cl_flags.ensure((m + 1) * 4);
    cl_pslot.ensure(((size_t)collapse_threads((u32)m, S) + 1) * 4);
    if (S) cl_partial.ensure(((size_t)collapse_threads((u32)m, S) + 1) * 8 * S);
    scan_tmp.ensure((scan_tmp_words((u32)m + 1) + 64) * 4);
  }
  void ensure_merge(size_t na, size_t nb) {
    mg_rank_a.ensure((na + 1) * 4);
    mg_match_a.ensure((2 * na + 2) * 4);
    mg_rank_b.ensure((nb + 1) * 4);
    mg_match_b.ensure((2 * nb + 2) * 4);
    scan_tmp.ensure((scan_tmp_words((u32)std::max(na, nb) + 1) + 64) * 4);
  }

  // Sort (key, pos) pairs of rows row0 + pos[i] (pos == nullptr: row0 + i),
  // i < m.  Returns the buffer index holding the sorted result.
  // assume: sort on the varying-bit mask of the execute's earlier chunks
  // instead of reading this chunk's mask back first (one host round trip
  // less); the caller then verifies it at its next synchronization
  // (sort_assumed, verify_assumed_mask)
  u64 sticky_vlo = 0, sticky_vhi = 0;
  bool sticky_ok = false, sort_assume = false, sort_assumed = false;
  int pend_hist_lo = -1, pend_hist_np = 0;   // histograms counted by build_keys for the pending sort
  static bool hist_fuse_env() {   // ISA_HIST_FUSE=0 (read per sort): the histogram kernel always runs
    const char* e = getenv("ISA_HIST_FUSE");
    return !(e && e[0] == '0');
  }
  int sort_rows(const KeyDesc& kd, int64_t row0, const u32* pos, u32 m, bool assume = false) {
    sort_assume = assume && sticky_ok && assume_env();
    ensure_sort(m);
    ph_begin(ISA_PH_SORT);
    CK(cudaMemsetAsync(dvary(), 0, 2 * sizeof(u64), st));
    // with the mask assumed the sort's bit range is known here: the key-building
    // pass counts the all-pass histograms itself (one read of the keys less)
    pend_hist_lo = -1;
    pend_hist_np = 0;
    u32* gh = nullptr;
    if (sort_assume && sticky_vhi == 0 && sticky_vlo != 0 && build_keys_counts_histograms(KW, kd, pos) &&
        hist_fuse_env()) {
      const int hb = 63 - __builtin_clzll(sticky_vlo);
      int lb = __builtin_ctzll(sticky_vlo);
      if (sort_partial_ok && hb - lb + 1 > 48 && m >= (1u << 20) && partial_env()) lb = hb - 47;   // as sort_built
      const int np = (hb + 1 - lb + 7) / 8;
      if (np >= 1 && np <= 16) {
        gh = sort_aux_hist(tile_hist.p);
        CK(cudaMemsetAsync(gh, 0, sort_aux_hist_bytes(), st));
        pend_hist_lo = lb;
        pend_hist_np = np;
      }
    }
    build_keys(KW, kd, row0, pos, m, s_lo[0].as<u64>(), s_hi[0].as<u64>(), s_val[0].as<u32>(), dvary(), st, gh,
               pend_hist_lo, pend_hist_np);
    sort_ctx = 0;
    sort_val_iota = pos == nullptr;
    int cur = sort_built(m);
    sort_ctx = 1;
    ph_end(ISA_PH_SORT, m, 0);
    return cur;
  }
  // known_v: the varying-bit mask is known on the host (a key-range window
  // [L, U): every key shares the bits above L ^ (U - 1)), no read-back
  bool sort_val_iota = false;   // the pending sort's payload is 0..m-1 (consumed by the next sort_built)
  static bool assume_env() {   // ISA_ASSUME_MASK=0 (read per sort): always read the chunk's mask back
    const char* e = getenv("ISA_ASSUME_MASK");
    return !(e && e[0] == '0');
  }
  // after a synchronization that followed to_host(dvary(), 16, 104): did the
  // chunk's varying bits stay inside the assumed mask?  (widens the mask if not)
  bool verify_assumed_mask() {
    const u64 alo = ((volatile u64*)h_scal)[52], ahi = ((volatile u64*)h_scal)[53];
    const bool ok = !(alo & ~sticky_vlo) && !(ahi & ~sticky_vhi);
    sticky_vlo |= alo;
    sticky_vhi |= ahi;
    return ok;
  }
  // the pending sort may carry a 4-byte value per row (in row order) with the keys and leave it in sorted
  // order in sort_carry_out; sort_carried tells whether it did (packed passes only)
  const u32* sort_carry_in = nullptr;
  u32* sort_carry_out = nullptr;
  bool sort_carried = false;
  int sort_built(u32 m, const u64* known_v = nullptr) {
    const bool iota = sort_val_iota;
    sort_val_iota = false;
    const int ph_lo = pend_hist_lo, ph_np = pend_hist_np;   // consumed by this sort on every path
    pend_hist_lo = -1;
    pend_hist_np = 0;
    sort_assumed = false;
    sort_partial_used = false;
    const bool partial_ok = sort_partial_ok;
    sort_partial_ok = false;
    const u32* cin = sort_carry_in;
    u32* cout = sort_carry_out;
    sort_carry_in = nullptr;
    sort_carry_out = nullptr;
    sort_carried = false;
    u64 vlo, vhi;
    if (known_v) {
      vlo = known_v[0];
      vhi = known_v[1];
    } else if (key_bits <= 16 || (key_bits <= 32 && m <= (1u << 20))) {
      // at most two 8-bit passes, or a small chunk of <= 32-bit keys: sort
      // every key bit instead of a host round trip for the varying bits
      vlo = key_bits == 64 ? ~0ull : ((1ull << key_bits) - 1);
      vhi = 0;
    } else if (sort_assume) {
      vlo = sticky_vlo;
      vhi = sticky_vhi;
      sort_assumed = true;
    } else {
      to_host(dvary(), 2 * sizeof(u64));
      sync();
      vlo = ((u64*)h_scal)[0];
      vhi = ((u64*)h_scal)[1];
      sticky_vlo |= vlo;
      sticky_vhi |= vhi;
      sticky_ok = true;
    }
    sort_assume = false;
    int hb = -1, lb = 128;
    if (vhi) { hb = 127 - __builtin_clzll(vhi); }
    else if (vlo) { hb = 63 - __builtin_clzll(vlo); }
    if (vlo) lb = __builtin_ctzll(vlo);
    else if (vhi) lb = 64 + __builtin_ctzll(vhi);
    if (hb < 0) return 0;   // all keys equal: already sorted (stable)
    SortBufs b;
    for (int i = 0; i < 2; ++i) { b.lo[i] = s_lo[i].as<u64>(); b.hi[i] = s_hi[i].as<u64>(); b.val[i] = s_val[i].as<u32>(); }
    b.aux = tile_hist.p;
    b.map_dev = d_hist_mapped;
    b.map_host = h_hist;
    b.pack_ok = true;   // bits outside [lb, hb] do not vary (see above)
    b.val_iota = iota;
    b.hist_bit_lo = ph_lo;
    b.hist_npass = ph_np;
    b.carry_in = cin;
    b.carry_out = cout;
    struct CarryBack { bool& f; SortBufs& b; ~CarryBack() { f = b.carried; } } carry_back{sort_carried, b};
    RankHint& rh = rank_hint[sort_ctx];
    b.hint = rh.h;
    b.hint_bit_lo = rh.bit_lo;
    b.hint_npass = rh.npass;
    struct HintBack {   // copy the (possibly updated) choice back on every return path
      RankHint& rh; SortBufs& b;
      ~HintBack() { rh.bit_lo = b.hint_bit_lo; rh.npass = b.hint_npass; }
    } hint_back{rh, b};
    if (KW == 2 && hb >= 64 && lb < 64) {
      // 128-bit keys whose high word varies: sort on the high word, then
      // finish runs of equal high words with a stable sort on the low word
      // (half the radix passes when high words are nearly unique)
      // ... and at most the top 48 bits of it (6 passes): keys sharing those
      // bits are rare and land in the same small run
      int lo_bit = std::max(lb, 64);
      if (hb - lo_bit + 1 > 48 && partial_env()) lo_bit = hb - 47;
      int cur = radix_sort_pairs(KW, b, m, lo_bit, hb + 1, st, nullptr);
      CK(cudaMemsetAsync(dscal32(5), 0, sizeof(u32), st));
      sort_small_segments(b.lo[cur], b.hi[cur], b.val[cur], m, 64, lo_bit > 64 ? lo_bit - 64 : 0, dscal32(5), st);
      if (read_u32(dscal32(5)) == 0) return cur;
      return radix_sort_pairs(KW, b, m, lb, hb + 1, st, nullptr, cur);
    }
    // Wide one-word keys (hashed 64-bit keys: every bit varies): sort on the
    // top 48 varying bits only -- 6 passes instead of 8.  Equal keys keep
    // their row order (stable), and two distinct keys that share 48 bits are
    // rare (about one pair per eight chunks of 2^23 distinct keys); a check
    // pass over the sorted keys reports an inversion to the caller's next
    // synchronization, which then sorts the chunk again on every bit.
    if (partial_ok && KW == 1 && hb - lb + 1 > 48 && m >= (1u << 20) && partial_env()) {
      const int cur = radix_sort_pairs(KW, b, m, hb - 47, hb + 1, st, nullptr);
      ((volatile u32*)h_scal)[111] = 0;
      check_sorted(b.lo[cur], m, d_scal_mapped + 111, st);
      sort_partial_used = true;
      return cur;
    }
    return radix_sort_pairs(KW, b, m, lb, hb + 1, st, nullptr);
  }
  // sort_partial_ok: the caller of the next sort can verify a partial-key
  // sort at its next synchronization (sort_partial_used, h_scal[111])
  bool sort_partial_ok = false, sort_partial_used = false;
  static bool partial_env() {   // ISA_PARTIAL_SORT=0 (read per sort): always sort every varying bit
    const char* e = getenv("ISA_PARTIAL_SORT");
    return !(e && e[0] == '0');
  }

  // Flush analysis on a sorted chunk of `span` rows: number of keys absent
  // from T; if |T| + new > M returns the chunk-relative flush row, else span.
  // absent_from_T: the sorted keys are known not to be in T (hash-image
  // misses), so no head needs the binary search over T
  u32 flush_point(int cur, u32 m, u32 span, const u32* firstpos = nullptr, bool absent_from_T = false) {
    const u32 tn_search = absent_from_T ? 0u : T.n;
    if (!firstpos && flush_small_ok(span)) {
      const u32 k = (u32)(cfg.memory_budget - (int64_t)T.n + 1);   // >= 1: |T| <= M
      ph_begin(ISA_PH_FLUSH);
      flush_small(KW, s_lo[cur].as<u64>(), s_hi[cur].as<u64>(), s_val[cur].as<u32>(), m, T.plo(), T.phi(), tn_search, span,
                  k, d_scal_mapped, st);
      ph_end(ISA_PH_FLUSH, m, 0);
      sync();
      const u32 n_new = ((volatile u32*)h_scal)[0], f = ((volatile u32*)h_scal)[1];
      last_new = n_new;
      return (int64_t)T.n + n_new <= cfg.memory_budget ? span : f;
    }
    u32 nw = (span + 31) / 32;
    bitmap.ensure((size_t)nw * 4 + 4);
    word_tmp.ensure((size_t)nw * 4 + 4);
    scan_tmp.ensure((scan_tmp_words(nw + 1) + 64) * 4);
    ph_begin(ISA_PH_FLUSH);
    CK(cudaMemsetAsync(bitmap.p, 0, (size_t)nw * 4, st));
    CK(cudaMemsetAsync(dscal32(0), 0, sizeof(u32), st));
    // chunks of mostly new keys (the previous chunk tells) mark the rows that
    // are not new heads and select in the complement: far fewer bitmap atomics
    const bool invert = !firstpos && m == span && new_frac_hint > 0.5 && flush_invert_env();
    new_heads(KW, s_lo[cur].as<u64>(), s_hi[cur].as<u64>(), s_val[cur].as<u32>(), m, T.plo(), T.phi(), tn_search,
              bitmap.as<u32>(), dscal32(0), st, firstpos, invert);
    const int64_t M = cfg.memory_budget;
    u32 k = (u32)(M - (int64_t)T.n + 1);   // >= 1: |T| <= M
    if (span <= (1u << 20) || expect_flush) {
      // small chunks, and chunks sized to end just past the next flush (the
      // previous chunk flushed): select the k-th new head speculatively and
      // read both numbers with one synchronization
      select_kth_bit(bitmap.as<u32>(), span, k, word_tmp.as<u32>(), scan_tmp.as<u32>(), dscal32(1), st, invert);
      to_host(dscal32(0), 2 * sizeof(u32));
      ph_end(ISA_PH_FLUSH, m, 0);
      sync();
      const u32 n_new = h_scal[0], f = h_scal[1];
      last_new = n_new;
      new_frac_hint = (double)n_new / (double)std::max<u32>(m, 1);
      return (int64_t)T.n + n_new <= M ? span : f;
    }
    to_host(dscal32(0), sizeof(u32));
    ph_end(ISA_PH_FLUSH, m, 0);
    sync();
    u32 n_new = h_scal[0];
    last_new = n_new;
    new_frac_hint = (double)n_new / (double)std::max<u32>(m, 1);
    if ((int64_t)T.n + n_new <= M) return span;
    ph_begin(ISA_PH_FLUSH);
    select_kth_bit(bitmap.as<u32>(), span, k, word_tmp.as<u32>(), scan_tmp.as<u32>(), dscal32(1), st, invert);
    to_host(dscal32(1), sizeof(u32));
    ph_end(ISA_PH_FLUSH, 0, 0);
    sync();
    return h_scal[0];
  }
  u32 last_new = 0;
  bool expect_flush = false;   // the current chunk was sized from the last fill cycle: a flush is likely
  double new_frac_hint = 0;   // new keys / rows of the last large flush analysis (per execute)
  static bool flush_invert_env() {   // ISA_FLUSH_INVERT=0 (read per call): always mark the new heads
    const char* e = getenv("ISA_FLUSH_INVERT");
    return !(e && e[0] == '0');
  }
  // large-table absorb (isa_hot.cu): hash image of T, rebuilt when T changed
  DevBuf hb_klo, hb_khi, hb_idx, hot_hit;
  HotHash hh{};
  u64 t_ver = 1, hash_ver = 0;   // T version (bumped on every change) / version the image was built from
  int hot_mode = 0;              // per execute: -1 auto (undecided), 0 off, 1 on
  double hot_miss_rate = 0;      // misses / rows of the last hot chunk
  static constexpr u32 kHotMinT = 1u << 15;   // smallest table worth a hash image
  bool hot_ready() const { return hot_mode == 1 && T.n > 8 && (cfg.hot_absorb == 1 || T.n >= kHotMinT); }
  // K1 tile pre-aggregation: slotted groups of the current chunk
  DevBuf g_lo, g_hi, g_first, g_st, g_count, g_off;
  Table U2;           // groups of the partial tile before a flush row
  int k1_mode = 0;    // per execute: -1 undecided, 0 off, 1 on
  size_t tcap = 1;   // capacity of every run-generation table: min(M, n) + 1

  // U <- collapse(sorted chunk restricted to positions < limit)
  // known_n >= 0: the caller knows the group count (no host round trip)
  bool collapse_by_pos = false;   // the next collapse_chunk reads value columns by sorted position (carried values)
  void collapse_chunk(int cur, u32 m, u32 limit, const SlotDesc& sd, int64_t row0, const u64* st_in, Table& out,
                      size_t out_cap, bool merge_phase = true, int64_t known_n = -1) {
    ensure_collapse(m);
    out.reserve(out_cap, KW, S);
    CollapseTmp ct;
    ct.flags = cl_flags.as<u32>();
    ct.scan_tmp = scan_tmp.as<u32>();
    ct.partial = cl_partial.as<u64>();
    ct.partial_slot = cl_pslot.as<u32>();
    ct.total = dscal32(2);
    ct.status = cl_status.as<u64>();
    ct.pay = cl_pay.as<u64>();
    ct.ticket = dscal32(22);
    ct.by_pos = collapse_by_pos;
    collapse_by_pos = false;
    const int phc = (st_in && merge_phase) ? ISA_PH_WM_COLLAPSE : ISA_PH_COLLAPSE;
    ph_begin(phc);
    kt_begin(KF_COLLAPSE, st);
    collapse(KW, s_lo[cur].as<u64>(), s_hi[cur].as<u64>(), s_val[cur].as<u32>(), m, limit, sd, row0, st_in,
             out.plo(), out.phi(), out.pst(), ct, st);
    // algorithmic bytes: every sorted (key, row id) read once, the rows'
    // values (or staged states) read once, the groups written once
    kt_end(KF_COLLAPSE, (int64_t)m * (8 * KW + 4 + (st_in ? 8 * S : value_row_bytes)), st);
    const int64_t out_row = 8 * KW + 8 * S;
    if (known_n >= 0) {
      ph_end(phc, m, 0);
      out.n = (u32)known_n;
      kt_add_bytes(KF_COLLAPSE, known_n * out_row);
      return;
    }
    to_host(dscal32(2), sizeof(u32));
    ph_end(phc, m, 0);
    sync();
    out.n = h_scal[0];
    kt_add_bytes(KF_COLLAPSE, (int64_t)out.n * out_row);
  }

  // out <- merge_combine(A, B); A's buffers become spare, B is emptied
  Table merge_tables(Table& A, Table& B) {
    ensure_merge(A.n, B.n);
    Table out = take_table();
    out.reserve(tcap, KW, S);   // |A ∪ B| <= min(M, n) by the flush analysis
    MergeTmp mt;
    mt.rank_a = mg_rank_a.as<u32>(); mt.match_a = mg_match_a.as<u32>();
    mt.rank_b = mg_rank_b.as<u32>(); mt.match_b = mg_match_b.as<u32>();
    mt.scan_tmp = scan_tmp.as<u32>();
    mt.total = dscal32(4);
    ph_begin(ISA_PH_TABLE_MERGE);
    merge_combine(KW, S, ops, types, A.plo(), A.phi(), A.pst(), A.n, B.plo(), B.phi(), B.pst(), B.n, out.plo(),
                  out.phi(), out.pst(), mt, st);
    to_host(dscal32(4), sizeof(u32));
    ph_end(ISA_PH_TABLE_MERGE, (int64_t)A.n + B.n, 0);
    sync();
    u32 matches = h_scal[0];
    out.n = A.n + B.n - matches;
    spare.push_back(A);
    A = Table();
    B.n = 0;
    return out;
  }

  // T <- merge_combine(T, U)
  void merge_into_T() {
    if (U.n == 0) return;
    ++t_ver;
    if (T.n == 0) { std::swap(T, U); U.n = 0; return; }
    T = merge_tables(T, U);
  }

  void refresh_tiny() {
    tiny_ok = false;
    if (T.n == 0 || T.n > 8) return;
    memset(&tiny, 0, sizeof(tiny));
    to_host(T.plo(), (size_t)T.n * 8);
    if (KW == 2) to_host(T.phi(), (size_t)T.n * 8, 16);
    sync();
    for (u32 j = 0; j < T.n; ++j) {
      tiny.lo[j] = ((u64*)h_scal)[j];
      tiny.hi[j] = KW == 2 ? ((u64*)h_scal)[8 + j] : 0;
    }
    tiny_ok = true;
  }
  bool tiny_ok = false;

  // allocate run storage (pinned host pool or device pool) for `rows` rows
  // run placement of the auto tier: HBM while the runs fit hbm_left bytes
  int64_t hbm_left = 0;
  bool run_to_device(size_t bytes) {
    if (cfg.run_tier == ISA_TIER_HBM) return true;
    if (cfg.run_tier != ISA_TIER_AUTO) return false;
    if ((int64_t)bytes > hbm_left) return false;
    hbm_left -= (int64_t)bytes;
    return true;
  }
  Run alloc_run(u32 rows) {
    Run r;
    r.rows = rows;
    const size_t nb_key = std::max<size_t>((size_t)rows * 8, 8), nb_st = std::max<size_t>((size_t)rows * 8 * S, 8);
    if (!run_to_device(nb_key * KW + (S ? nb_st : 0))) {
      r.host = true;
      char* klo = pinned.alloc(nb_key);
      char* khi = KW == 2 ? pinned.alloc(nb_key) : nullptr;
      char* kst = S ? pinned.alloc(nb_st) : nullptr;
      u64 *dlo = nullptr, *dhi = nullptr, *dst = nullptr;
      CK(cudaHostGetDevicePointer((void**)&dlo, klo, 0));
      if (khi) CK(cudaHostGetDevicePointer((void**)&dhi, khi, 0));
      if (kst) CK(cudaHostGetDevicePointer((void**)&dst, kst, 0));
      r.lo = dlo; r.hi = dhi; r.st = dst;
      r.host_lo = (const u64*)klo;
      r.host_hi = (const u64*)khi;
    } else {
      r.host = false;
      r.lo = (u64*)devpool.alloc(nb_key);
      r.hi = KW == 2 ? (u64*)devpool.alloc(nb_key) : nullptr;
      r.st = S ? (u64*)devpool.alloc(nb_st) : nullptr;
    }
    return r;
  }

  // copy `n` table rows into run storage at row offset `off` (on stream s)
  void copy_into_run(Run& r, Table& t, u32 n, size_t off, cudaStream_t s) {
    const size_t nb_key = (size_t)n * 8, nb_st = (size_t)n * 8 * S;
    CK(cudaMemcpyAsync(r.lo + off, t.plo(), nb_key, cudaMemcpyDefault, s));
    if (KW == 2) CK(cudaMemcpyAsync(r.hi + off, t.phi(), nb_key, cudaMemcpyDefault, s));
    if (S) CK(cudaMemcpyAsync(r.st + off * S, t.pst(), nb_st, cudaMemcpyDefault, s));
    if (r.host) led.bytes_d2h += nb_key * KW + nb_st;
  }

  void account_written(const Run& r) {
    led.rows_spilled += r.rows;
    led.pages_written += (r.rows + cfg.page_capacity - 1) / cfg.page_capacity;
  }

  // small runs are not worth the extra synchronization (their link time is tiny)
  bool pack_u32_ok = true;   // packed images of the largest run fit 32-bit offsets
  bool pack_runs(u32 rows) const {
    if ((cfg.run_tier != ISA_TIER_HOST && cfg.run_tier != ISA_TIER_AUTO) || cfg.merge_mode != ISA_MERGE_WIDE ||
        !pack_u32_ok)
      return false;
    return cfg.run_codec == 2 || (cfg.run_codec == 0 && rows >= kPackMinRows);
  }
  static constexpr u32 kPackMinRows = 1u << 15;

  // Auto tier: keep a run raw in HBM (no pack / unpack) when it fits next to
  // the estimated packed size of everything still to spill (at most the input
  // rows not yet read, at the packed/raw ratio measured on earlier runs); the
  // first run is packed to learn the ratio.
  int64_t rows_left = 0;              // input rows not yet consumed (updated per chunk)
  double packed_ratio = -1;           // packed / raw bytes of the last packed run
  // Raw runs pay off when the wide merge reads them in place -- the
  // dense-window merge (predicted from the first run: one key word, integer
  // slots, a key span of at most 4 keys per input row): no pack, and the
  // accumulate kernel reads 8 * (KW + S) bytes per row instead of decoding.
  // For the sort-based windows they do not (config 5 at 1e9 rows 189 -> 192
  // ms: the D2D slice copies cost more than unpacking).  Raw runs take at most
  // 45% of the memory free at the start of the execute (all runs together up
  // to 50%, hbm_left): the caller's output columns, and a result table when
  // the merge needs one, still have to fit.  ISA_RAW_RUNS=1 / 0 forces raw
  // runs whenever they fit hbm_left / off.
  int dense_pred = -1;     // per execute: -1 unknown, 0 / 1 the dense-window merge is expected
  double raw_left = 0;     // bytes of raw runs still allowed
  bool raw_fits_hbm(u32 rows) {
    const char* e = getenv("ISA_RAW_RUNS");
    if ((e && e[0] == '0') || cfg.run_tier != ISA_TIER_AUTO || packed_ratio < 0) return false;
    const double row_b = 8.0 * (KW + S);
    const double need = (double)rows * row_b + (double)rows_left * row_b * packed_ratio;
    if (need > (double)hbm_left) return false;
    if (e && e[0] == '1') return true;
    if (dense_pred != 1 || (double)rows * row_b > raw_left) return false;
    raw_left -= (double)rows * row_b;
    return true;
  }
  // first run: is the dense-window merge likely (see dense_merge)?
  void predict_dense() {
    if (dense_pred >= 0) return;
    dense_pred = 0;
    if (KW != 1 || T.n < 2 || cfg.run_tier != ISA_TIER_AUTO) return;
    for (int s = 0; s < S; ++s)
      if (sd0.type[s] != ST_I64) return;
    u64 ends[2];
    CK(cudaMemcpyAsync(&ends[0], T.plo(), 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&ends[1], T.plo() + (T.n - 1), 8, cudaMemcpyDeviceToHost, st));
    sync();
    dense_pred = (double)(ends[1] - ends[0]) < 4.0 * (double)in_n ? 1 : 0;
  }

  // T packed on the GPU (isa_codec.cu), then the packed bytes cross PCIe.
  // One host synchronization learns the packed size.
  Run spill_packed(Table& t) {
    PackSrc ps{t.plo(), t.phi(), t.pst(), t.n, KW, S, fmask};
    const u32 nblk = pack_blocks(t.n);
    const int ncol = KW + S;
    pk_sz.ensure((size_t)(nblk + 2) * 4 + 16);
    u32 bytes = 0;
    size_t off_at = 0;
    kt_begin(KF_PACK, st);
    if (pack_fused_ok(ps)) {
      // one pass; the output is bounded by the raw size
      const size_t bound = (size_t)nblk * ncol * 16 + (size_t)t.n * ncol * 8 + 64;
      t.pk.ensure(bound + (size_t)(nblk + 1) * 4 + 32);
      const size_t had = pk_status.bytes;
      pk_status.ensure((size_t)nblk * 8 + 16);
      if (pk_status.bytes != had) CK(cudaMemsetAsync(pk_status.p, 0, pk_status.bytes, st));   // epochs start at 0
      pack_fused(ps, pk_status.as<u64>(), pk_sz.as<u32>() + nblk + 1, pk_sz.as<u32>(), t.pk.as<char>(), st);
      kt_end(KF_PACK, (int64_t)t.n * 8 * ncol, st);
      bytes = read_u32(pk_sz.as<u32>() + nblk);   // offsets[nblk] = total
      off_at = ((size_t)bytes + 15) & ~(size_t)15;
    } else {
      pk_hdr.ensure((size_t)nblk * ncol * 16 + 16);
      scan_tmp.ensure((scan_tmp_words(nblk + 1) + 64) * 4);
      pack_sizes(ps, pk_hdr.as<u64>(), pk_sz.as<u32>(), st);
      scan_exclusive_u32(pk_sz.as<u32>(), nblk, scan_tmp.as<u32>(), pk_sz.as<u32>() + nblk, st);
      bytes = read_u32(pk_sz.as<u32>() + nblk);   // offsets[nblk] = total
      off_at = ((size_t)bytes + 15) & ~(size_t)15;
      t.pk.ensure(off_at + (size_t)(nblk + 1) * 4 + 16);
      pack_write(ps, pk_hdr.as<u64>(), pk_sz.as<u32>(), t.pk.as<char>(), st);
      kt_end(KF_PACK, (int64_t)t.n * 8 * ncol * 2, st);
    }
    kt_add_bytes(KF_PACK, bytes);
    packed_ratio = (double)bytes / std::max(1.0, (double)t.n * 8.0 * (KW + S));
    // packed blocks, then the block offsets: both owned by the table until
    // its D2H copies are done (pk_sz is reused by the next spill)
    CK(cudaMemcpyAsync(t.pk.as<char>() + off_at, pk_sz.p, (size_t)(nblk + 1) * 4, cudaMemcpyDeviceToDevice, st));
    Run r;
    r.rows = t.n;
    r.nblk = nblk;
    if (run_to_device((size_t)bytes + (size_t)(nblk + 1) * 4 + 512)) {
      // auto tier: the packed image stays in HBM (one D2D copy on the
      // compute stream; the table is free again right after it)
      r.host = false;
      char* db = devpool.alloc((size_t)bytes + 16);
      u32* doff = (u32*)devpool.alloc((size_t)(nblk + 1) * 4 + 16);
      u32* hoff = (u32*)pinned.alloc((size_t)(nblk + 1) * 4 + 16);
      CK(cudaMemcpyAsync(db, t.pk.p, bytes, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(doff, t.pk.as<char>() + off_at, (size_t)(nblk + 1) * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(hoff, t.pk.as<char>() + off_at, (size_t)(nblk + 1) * 4, cudaMemcpyDeviceToHost, st));
      r.pk_dev = db; r.off_dev = doff; r.off_host = hoff;
      dev_packed = true;
      return r;
    }
    r.host = true;
    char* hb = pinned.alloc((size_t)bytes + 16);
    u32* hoff = (u32*)pinned.alloc((size_t)(nblk + 1) * 4 + 16);
    const char* db = nullptr;
    const u32* doff = nullptr;
    CK(cudaHostGetDevicePointer((void**)&db, hb, 0));
    CK(cudaHostGetDevicePointer((void**)&doff, hoff, 0));
    r.pk_host = hb; r.pk_dev = db; r.off_host = hoff; r.off_dev = doff;
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, st));
    CK(cudaStreamWaitEvent(d2h, ev, 0));
    cudaEventDestroy(ev);
    CK(cudaMemcpyAsync(hb, t.pk.p, bytes, cudaMemcpyDeviceToHost, d2h));
    CK(cudaMemcpyAsync(hoff, t.pk.as<char>() + off_at, (size_t)(nblk + 1) * 4, cudaMemcpyDeviceToHost, d2h));
    led.bytes_d2h += bytes + (size_t)(nblk + 1) * 4;
    return r;
  }

  static void grow_pinned(char*& p, size_t& cap, size_t need) {
    if (need <= cap) return;
    if (p) CK(cudaFreeHost(p));
    cap = std::max(need, cap + cap / 2);
    CK(cudaHostAlloc((void**)&p, cap, cudaHostAllocDefault));
  }

  // FileStore tier: T encoded as reference pages on the GPU, copied out and
  // written to run_NNNNNN.bin (RunWriter + FileStore.append_page,
  // runstore.py:205-220, 239-301).  Synchronous: the file is complete when
  // this returns.
  Run spill_file(Table& t) {
    if (spill_dir.empty()) throw IsaError(ISA_ERR_INVALID_INPUT, "FileStore tier without a spill directory");
    const u32 n = t.n;
    const u32 bytes = page_run_bytes(ps0, n);
    const u32 npages = (n + ps0.P - 1) / ps0.P;
    t.pk.ensure((size_t)bytes + 16);
    CK(cudaMemsetAsync(dscal32(6), 0, sizeof(u32), st));
    page_encode(ps0, t.plo(), t.phi(), t.pst(), n, t.pk.as<char>(), dscal32(6), st);
    grow_pinned(file_pin, file_pin_cap, bytes);
    CK(cudaMemcpyAsync(file_pin, t.pk.p, bytes, cudaMemcpyDeviceToHost, st));
    Run r;
    r.rows = n;
    r.host = true;
    r.npages = npages;
    r.hk_lo.resize(npages);
    if (KW == 2) r.hk_hi.resize(npages);
    // page high keys: rows P-1, 2P-1, ... and the last row
    if (npages > 1) {
      CK(cudaMemcpy2DAsync(r.hk_lo.data(), 8, t.plo() + (ps0.P - 1), (size_t)ps0.P * 8, 8, npages - 1,
                           cudaMemcpyDeviceToHost, st));
      if (KW == 2)
        CK(cudaMemcpy2DAsync(r.hk_hi.data(), 8, t.phi() + (ps0.P - 1), (size_t)ps0.P * 8, 8, npages - 1,
                             cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(r.hk_lo.data() + npages - 1, t.plo() + n - 1, 8, cudaMemcpyDeviceToHost, st));
    if (KW == 2) CK(cudaMemcpyAsync(r.hk_hi.data() + npages - 1, t.phi() + n - 1, 8, cudaMemcpyDeviceToHost, st));
    to_host(dscal32(6), sizeof(u32));
    sync();
    if (h_scal[0])
      throw IsaError(ISA_ERR_INVALID_INPUT, "a uint64 key value >= 2^63 cannot be written as an int64 page column");
    char name[32];
    snprintf(name, sizeof(name), "run_%06lld.bin", (long long)next_run_id++);
    r.path = spill_dir + "/" + name;
    int fd = ::open(r.path.c_str(), O_CREAT | O_WRONLY | O_TRUNC, 0644);
    if (fd < 0) throw IsaError(ISA_ERR_RESOURCE, "cannot create " + r.path);
    size_t done = 0;
    while (done < bytes) {
      ssize_t w = ::write(fd, file_pin + done, bytes - done);
      if (w <= 0) { ::close(fd); throw IsaError(ISA_ERR_RESOURCE, "short write to " + r.path); }
      done += (size_t)w;
    }
    ::close(fd);
    led.bytes_d2h += bytes;
    t.n = 0;
    return r;
  }

  // int64 page column value -> normalized key bits of column c (host)
  u64 page_field(int c, i64 v) const {
    const int w = ps0.width[c];
    u64 f = (u64)v;
    if (ps0.sgn[c]) f ^= 1ull << (w - 1);
    if (w < 64) f &= (1ull << w) - 1;
    return f;
  }
  static void pread_all(const std::string& path, char* dst, size_t bytes, size_t off) {
    int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) throw IsaError(ISA_ERR_RESOURCE, "cannot open " + path);
    size_t done = 0;
    while (done < bytes) {
      ssize_t r = ::pread(fd, dst + done, bytes - done, (off_t)(off + done));
      if (r <= 0) { ::close(fd); throw IsaError(ISA_ERR_CORRUPTION, "truncated run file " + path); }
      done += (size_t)r;
    }
    ::close(fd);
  }
  size_t page_off(u32 p) const { return (size_t)p * (12 + ps0.body_full); }
  u32 page_rows(const Run& r, u32 p) const { return std::min<u32>((u32)ps0.P, r.rows - p * (u32)ps0.P); }
  size_t page_len(const Run& r, u32 p) const {
    return 12 + 8 * (size_t)ps0.arity + (size_t)page_rows(r, p) * 8 * (ps0.arity + S);
  }
  // first row of file run r whose key >= (bhi, blo): page high keys, then
  // the keys of one page read back (host; the slice search of the merge)
  u32 file_lower_bound(const Run& r, u64 bhi, u64 blo) {
    u32 l = 0, h = r.npages;
    auto less_b = [&](u64 khi, u64 klo) { return KW == 2 ? (khi < bhi || (khi == bhi && klo < blo)) : klo < blo; };
    while (l < h) {
      u32 m = (l + h) / 2;
      if (less_b(KW == 2 ? r.hk_hi[m] : 0, r.hk_lo[m])) l = m + 1; else h = m;
    }
    if (l == r.npages) return r.rows;
    std::vector<char> pg(page_len(r, l));
    pread_all(r.path, pg.data(), pg.size(), page_off(l));
    const u32 rows = page_rows(r, l);
    const char* body = pg.data() + 12;
    for (u32 i = 0; i < rows; ++i) {
      const char* row = body + 8 * ps0.arity + (size_t)i * 8 * (ps0.arity + S);
      u64 klo = 0, khi = 0;
      for (int c = 0; c < ps0.arity; ++c) {
        i64 v;
        memcpy(&v, row + 8 * c, 8);
        const u64 f = page_field(c, v);
        const int s = ps0.shift[c], w = ps0.width[c];
        if (s < 64) {
          klo |= f << s;
          if (s > 0 && s + w > 64) khi |= f >> (64 - s);
        } else {
          khi |= f << (s - 64);
        }
      }
      if (!less_b(khi, klo)) return l * (u32)ps0.P + i;
    }
    return l * (u32)ps0.P + rows;
  }

  // T becomes a run (RunWriter of a read-sort-write flush, sortagg.py:344-350)
  bool dev_packed = false;   // a packed run of this execute went to HBM (spill_T: no busy table)
  void spill_T() {
    if (T.n == 0) return;
    ++t_ver;
    if (cfg.run_tier == ISA_TIER_FILE) {
      Run r = spill_file(T);
      runs.push_back(r);
      account_written(r);
      return;
    }
    u32* dir = make_dir();
    predict_dense();
    if (pack_runs(T.n) && !raw_fits_hbm(T.n)) {
      Run r = spill_packed(T);
      r.dir = dir;
      if (!r.host) {   // stream-ordered D2D copy: T's buffers are reusable right away
        T.n = 0;
        runs.push_back(r);
        account_written(r);
        return;
      }
      CK(cudaEventRecord(spill_done, d2h));
      cudaEvent_t bev;
      if (!busy_ev_pool.empty()) { bev = busy_ev_pool.back(); busy_ev_pool.pop_back(); }
      else CK(cudaEventCreateWithFlags(&bev, cudaEventDisableTiming));
      CK(cudaEventRecord(bev, d2h));
      busy.push_back({T, bev});
      T = take_table();
      runs.push_back(r);
      account_written(r);
      return;
    }
    Run r = alloc_run(T.n);
    r.dir = dir;
    if (r.host) {
      // copy on the d2h stream after the table is complete; the table's
      // buffers are recycled only after the copy finished (busy list)
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CK(cudaEventRecord(ev, st));
      CK(cudaStreamWaitEvent(d2h, ev, 0));
      cudaEventDestroy(ev);
      copy_into_run(r, T, T.n, 0, d2h);
      CK(cudaEventRecord(spill_done, d2h));
      cudaEvent_t bev;
      if (!busy_ev_pool.empty()) { bev = busy_ev_pool.back(); busy_ev_pool.pop_back(); }
      else CK(cudaEventCreateWithFlags(&bev, cudaEventDisableTiming));
      CK(cudaEventRecord(bev, d2h));
      busy.push_back({T, bev});
      T = take_table();
    } else {
      copy_into_run(r, T, T.n, 0, st);
      T.n = 0;
    }
    runs.push_back(r);
    account_written(r);
  }

  // ------------------------------------------------------------ chunks --
  // Process rows [a, b) (absolute), columns addressed by (kd, sd) with
  // row0_base = absolute row of column element 0.  Returns the absolute row
  // at which the next chunk starts (b, or the flush row).
  int64_t process_chunk(const KeyDesc& kd, const SlotDesc& sd, int64_t base, int64_t a, int64_t b) {
    const u32 span = (u32)(b - a);
    const int64_t row0 = a - base;   // column element of row a
    led.chunks++;
    if (T.n > 0 && T.n <= 8 && tiny_ok && absorb_supported((int)T.n, S)) return absorb_chunk(kd, sd, row0, a, span);
    // tiny chunks are not worth the extra pass in auto mode; "always" keeps
    // it down to 4 tiles (also what the parity tests exercise)
    if (hot_ready()) return hot_chunk(kd, sd, row0, a, span);
    const u32 k1_min = (cfg.preaggregate == 1 ? 4 : 64) * tile_rows();
    if (k1_mode != 0 && span >= k1_min) return k1_chunk(kd, sd, row0, a, span);
    // one int64 value column: an int32 copy of the chunk's values, carried
    // through the packed sort passes as the payload so that the collapse
    // reads every row's value at its sorted position (no random gather); when
    // the sort cannot carry it (key bits spanning more than 32) the collapse
    // gathers from the int32 copy.  The fit check rides on the flush
    // analysis's host round trip.
    const void* ncol = span >= (1u << 20) ? narrow_candidate(sd) : nullptr;
    if (ncol) {
      rec_buf.ensure((size_t)span * 4 + 64);
      ((volatile u32*)h_scal)[110] = 0;
      narrow_i64(ncol, row0, span, rec_buf.as<int>(), d_scal_mapped + 110, st);
      if (collapse_by_pos_ok(span, S)) {
        rec_sorted.ensure((size_t)span * 4 + 64);
        sort_carry_in = rec_buf.as<u32>();
        sort_carry_out = rec_sorted.as<u32>();
      }
    }
    sort_partial_ok = true;
    int cur = sort_rows(kd, row0, nullptr, span, /*assume=*/true);
    bool carried = sort_carried;
    const bool assumed = sort_assumed, partial = sort_partial_used;
    if (assumed) to_host(dvary(), 2 * sizeof(u64), 104);
    const bool t_empty = T.n == 0;
    u32 f = flush_point(cur, span, span);
    const bool mask_ok = !assumed || verify_assumed_mask();
    if (!mask_ok || (partial && ((volatile u32*)h_scal)[111] != 0)) {
      // key bits outside the assumed mask vary in this chunk, or two keys
      // that share the sorted top bits came out of order: sort again on the
      // chunk's own mask, every bit
      cur = sort_rows(kd, row0, nullptr, span);
      carried = sort_carried;
      f = flush_point(cur, span, span);
    }
    // with T empty every group of the chunk before f is new: M of them on a
    // flush, else the new-key count the flush analysis already returned
    const int64_t known = t_empty ? (f < span ? cfg.memory_budget : (int64_t)last_new) : -1;
    SlotDesc sdc = sd;
    int64_t r0c = row0;
    if (ncol && ((volatile u32*)h_scal)[110] == 0) {
      for (int s = 0; s < S; ++s)
        if (sd.src[s] == SRC_COL && sd.ptr[s] == ncol) {
          sdc.ptr[s] = carried ? rec_sorted.p : rec_buf.p;
          sdc.dtype[s] = ISA_I32;
        }
      r0c = 0;
      collapse_by_pos = carried;
    } else if (f >= (1u << 20) && pack_records(sd, sdc, f)) {
      // >= 2 value columns: one record per row, so the collapse's random
      // gather touches one sector per row instead of one per column
      row_pack(rpk, row0, f, rec_buf.as<char>(), st);
      r0c = 0;
    }
    // a flush into an empty table whose run stays raw in HBM: the collapse
    // writes the run's rows in place (no table, no device-to-device copy)
    if (t_empty && f < span && cfg.run_tier == ISA_TIER_AUTO && dense_pred == 1 && !dirs_wanted() &&
        pack_runs((u32)cfg.memory_budget) && raw_fits_hbm((u32)cfg.memory_budget)) {
      Run r = alloc_run((u32)cfg.memory_budget);
      if (!r.host) {
        Table view;   // borrows the run's storage (DevBuf owns nothing by itself)
        view.lo.p = r.lo; view.lo.bytes = (size_t)r.rows * 8;
        view.st.p = r.st; view.st.bytes = (size_t)r.rows * 8 * S;
        collapse_chunk(cur, span, f, sdc, r0c, nullptr, view, r.rows, true, known);
        ++t_ver;
        runs.push_back(r);
        account_written(r);
        return a + f;
      }
      // (not reached: raw_fits_hbm reserved the space) fall through with the host run unused
    }
    collapse_chunk(cur, span, f, sdc, r0c, nullptr, U, tcap, true, known);
    merge_into_T();
    if (f < span) {
      spill_T();
      return a + f;
    }
    refresh_tiny();
    return b;
  }

  // First chunk into an empty T: one single-CTA kernel finds the chunk's
  // groups when there are few of them (<= 8 and <= M: no flush possible),
  // writes T and hands the keys to the absorb kernel; false = use the sort path.
  bool probe_chunk(const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 span) {
    u32 max_nt = 0;
    for (int t = 8; t >= 1; --t)
      if (t <= cfg.memory_budget && absorb_supported(t, S)) { max_nt = (u32)t; break; }
    if (max_nt == 0) return false;
    ph_begin(ISA_PH_PROBE);
    probe_tiny(KW, kd, sd, row0, span, max_nt, T.plo(), T.phi(), T.pst(), (u64*)d_scal_mapped, st);
    ph_end(ISA_PH_PROBE, span, 0);
    sync();
    const volatile u64* hw = (const volatile u64*)h_scal;
    if (hw[0] == ~0ull) return false;
    T.n = (u32)hw[0];
    last_new = T.n;
    memset(&tiny, 0, sizeof(tiny));
    for (u32 j = 0; j < T.n; ++j) {
      tiny.lo[j] = hw[8 + j];
      tiny.hi[j] = KW == 2 ? hw[16 + j] : 0;
    }
    tiny_ok = true;
    return true;
  }

  // Sort path with tile-local pre-aggregation (K1): sort the tiles' groups
  // instead of the rows.  Exact read-sort-write semantics: each group knows
  // its first row, so the flush row f is exact; groups are excluded at tile
  // granularity (tile < f / TILE, i.e. slotted index < (f / TILE) * TILE) and
  // the rows of f's tile before f are collapsed from the raw rows.
  int64_t k1_chunk(const KeyDesc& kd, const SlotDesc& sd, int64_t row0, int64_t a, u32 span) {
    const u32 TR = tile_rows();
    const u32 tiles = (span + TR - 1) / TR;
    const size_t slots = (size_t)tiles * TR;
    g_lo.ensure(slots * 8);
    if (KW == 2) g_hi.ensure(slots * 8);
    g_first.ensure(slots * 4);
    if (S) g_st.ensure(slots * 8 * S);
    g_count.ensure((size_t)(tiles + 1) * 4);
    g_off.ensure((size_t)(tiles + 1) * 4);
    scan_tmp.ensure((scan_tmp_words(tiles + 1) + 64) * 4);
    ph_begin(ISA_PH_SORT);
    tile_collapse(KW, kd, sd, row0, span, g_lo.as<u64>(), g_hi.as<u64>(), g_first.as<u32>(), g_st.as<u64>(),
                  g_count.as<u32>(), st);
    CK(cudaMemcpyAsync(g_off.p, g_count.p, (size_t)tiles * 4, cudaMemcpyDeviceToDevice, st));
    scan_exclusive_u32(g_off.as<u32>(), tiles, scan_tmp.as<u32>(), dscal32(6), st);
    const u32 groups = read_u32(dscal32(6));
    // auto mode: keep pre-aggregating only if tiles collapse at least 2x
    // (measured: on config 3, Zipf(1.1), tiles reach ~0.65 and the extra
    // pass costs more than the smaller sort saves)
    if (k1_mode < 0) k1_mode = (double)groups <= 0.5 * (double)span ? 1 : 0;
    ensure_sort(groups);
    CK(cudaMemsetAsync(dvary(), 0, 2 * sizeof(u64), st));
    compact_groups(KW, g_lo.as<u64>(), g_hi.as<u64>(), g_count.as<u32>(), g_off.as<u32>(), tiles, s_lo[0].as<u64>(),
                   s_hi[0].as<u64>(), s_val[0].as<u32>(), dvary(), st);
    const int cur = sort_built(groups);
    ph_end(ISA_PH_SORT, span, 0);
    const u32 f = flush_point(cur, groups, span, g_first.as<u32>());
    if (f >= span) {
      collapse_chunk(cur, groups, 0xFFFFFFFFu, sd, 0, g_st.as<u64>(), U, tcap, /*merge_phase=*/false);
      merge_into_T();
      refresh_tiny();
      return a + span;
    }
    const u32 tau = f / TR;
    collapse_chunk(cur, groups, tau * TR, sd, 0, g_st.as<u64>(), U, tcap, false);
    if (f > tau * TR) {   // rows of the flush row's tile before it, from the raw rows
      const u32 m2 = f - tau * TR;
      const int c2 = sort_rows(kd, row0 + (int64_t)tau * TR, nullptr, m2);
      collapse_chunk(c2, m2, 0xFFFFFFFFu, sd, row0 + (int64_t)tau * TR, nullptr, U2, tcap);
      if (U2.n) {
        if (U.n == 0) std::swap(U, U2);
        else U = merge_tables(U, U2);
        U2.n = 0;
      }
    }
    merge_into_T();
    spill_T();
    return a + f;
  }

  // one absorb pass over rows [row0, row0 + n) of the chunk -> per-CTA partials + miss lists
  void absorb_pass(const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, u32* grid_out, u32* rpc_out) {
    const int nt = (int)T.n;
    u32 grid, rpc;
    absorb_geometry(n, num_sms, &grid, &rpc);
    ab_partials.ensure((size_t)grid * nt * std::max(S, 1) * 8 + 64);
    ab_miss_buf.ensure((size_t)grid * rpc * 4 + 64);
    ab_miss_cnt.ensure((size_t)(grid + 1) * 4);
    ab_miss_off.ensure((size_t)(grid + 1) * 4);
    ph_begin(ISA_PH_ABSORB);
    kt_begin(KF_ABSORB, st);
    absorb_tiny(KW, nt, kd, sd, row0, n, tiny, grid, rpc, ab_partials.as<u64>(), ab_miss_buf.as<u32>(),
                ab_miss_cnt.as<u32>(), st);
    kt_end(KF_ABSORB, (int64_t)n * absorb_row_bytes, st);
    ph_end(ISA_PH_ABSORB, n, (int64_t)n * absorb_row_bytes);
    *grid_out = grid;
    *rpc_out = rpc;
  }

  int64_t absorb_chunk(const KeyDesc& kd, const SlotDesc& sd, int64_t row0, int64_t a, u32 span) {
    const int nt = (int)T.n;
    u32 grid, rpc;
    absorb_pass(kd, sd, row0, span, &grid, &rpc);
    scan_tmp.ensure((scan_tmp_words(grid + 1) + 64) * 4);
    CK(cudaMemcpyAsync(ab_miss_off.p, ab_miss_cnt.p, (size_t)grid * 4, cudaMemcpyDeviceToDevice, st));
    scan_exclusive_u32(ab_miss_off.as<u32>(), grid, scan_tmp.as<u32>(), dscal32(3), st);
    // fold speculatively (the common case: no misses) before the one host
    // round trip; T's states are kept to undo it when the chunk has misses
    const size_t tst_bytes = (size_t)nt * S * 8;
    if (S) {
      t_backup.ensure(tst_bytes + 8);
      CK(cudaMemcpyAsync(t_backup.p, T.pst(), tst_bytes, cudaMemcpyDeviceToDevice, st));
    }
    fold_partials(nt, sd, ab_partials.as<u64>(), grid, T.pst(), st);
    u32 nmiss = read_u32(dscal32(3));
    if (nmiss == 0) {
      last_new = 0;
      return a + span;
    }
    if (S) CK(cudaMemcpyAsync(T.pst(), t_backup.p, tst_bytes, cudaMemcpyDeviceToDevice, st));
    miss_list.ensure((size_t)nmiss * 4 + 64);
    compact_misses(ab_miss_buf.as<u32>(), ab_miss_cnt.as<u32>(), ab_miss_off.as<u32>(), grid, rpc,
                   miss_list.as<u32>(), st);
    int cur = sort_rows(kd, row0, miss_list.as<u32>(), nmiss);
    u32 f = flush_point(cur, nmiss, span);
    if (f >= span) {
      fold_partials(nt, sd, ab_partials.as<u64>(), grid, T.pst(), st);
      collapse_chunk(cur, nmiss, span, sd, row0, nullptr, U, tcap);
      merge_into_T();
      refresh_tiny();
      return a + span;
    }
    // a flush inside this chunk: the optimistic partials include hits at or
    // after f; recompute them for [a, a + f) only
    if (f > 0) {
      u32 g2, r2;
      absorb_pass(kd, sd, row0, f, &g2, &r2);
      fold_partials(nt, sd, ab_partials.as<u64>(), g2, T.pst(), st);
    }
    collapse_chunk(cur, nmiss, f, sd, row0, nullptr, U, tcap);
    merge_into_T();
    spill_T();
    return a + f;
  }

  // Chunk with a large resident table: rows whose key is in T are absorbed
  // through T's hash image (memindex.py:209-215), only the misses -- the
  // chunk's new keys -- are sorted; the flush row comes from the sorted
  // misses exactly as on the sort path, and only hits before it are absorbed.
  int64_t hot_chunk(const KeyDesc& kd, const SlotDesc& sd, int64_t row0, int64_t a, u32 span) {
    ph_begin(ISA_PH_HOT);
    if (hash_ver != t_ver) {
      const u32 cap = hot_hash_capacity(T.n);
      hb_idx.ensure((size_t)cap * 4);
      hb_klo.ensure((size_t)cap * 8);
      if (KW == 2) hb_khi.ensure((size_t)cap * 8);
      hh = HotHash{hb_klo.as<u64>(), KW == 2 ? hb_khi.as<u64>() : nullptr, hb_idx.as<u32>(), cap - 1};
      hot_hash_build(KW, T.plo(), T.phi(), T.n, hh, st);
      hash_ver = t_ver;
    }
    u32 grid, rpc;
    hot_probe_geometry(span, num_sms, &grid, &rpc);
    hot_hit.ensure((size_t)span * 4 + 64);
    ab_miss_buf.ensure((size_t)grid * rpc * 4 + 64);
    ab_miss_cnt.ensure((size_t)(grid + 1) * 4);
    ab_miss_off.ensure((size_t)(grid + 1) * 4);
    scan_tmp.ensure((scan_tmp_words(grid + 1) + 64) * 4);
    kt_begin(KF_HOT_PROBE, st);
    hot_probe(KW, kd, row0, span, hh, grid, rpc, hot_hit.as<u32>(), ab_miss_buf.as<u32>(), ab_miss_cnt.as<u32>(), st);
    kt_end(KF_HOT_PROBE, (int64_t)span * (key_bits / 8 + 4), st);
    CK(cudaMemcpyAsync(ab_miss_off.p, ab_miss_cnt.p, (size_t)grid * 4, cudaMemcpyDeviceToDevice, st));
    scan_exclusive_u32(ab_miss_off.as<u32>(), grid, scan_tmp.as<u32>(), dscal32(3), st);
    ph_end(ISA_PH_HOT, span, 0);
    const u32 nmiss = read_u32(dscal32(3));
    hot_miss_rate = (double)nmiss / (double)std::max<u32>(span, 1);
    u32 f = span;
    int cur = 0;
    if (nmiss) {
      miss_list.ensure((size_t)nmiss * 4 + 64);
      compact_misses(ab_miss_buf.as<u32>(), ab_miss_cnt.as<u32>(), ab_miss_off.as<u32>(), grid, rpc,
                     miss_list.as<u32>(), st);
      cur = sort_rows(kd, row0, miss_list.as<u32>(), nmiss);
      f = flush_point(cur, nmiss, span, nullptr, /*absent_from_T=*/true);
    } else {
      last_new = 0;
    }
    // hits before the flush row, into T (T's indices: before the merge)
    ph_begin(ISA_PH_HOT);
    kt_begin(KF_HOT_ABSORB, st);
    hot_absorb(sd, row0, f, hot_hit.as<u32>(), T.pst(), num_sms, st);
    kt_end(KF_HOT_ABSORB, (int64_t)f * (4 + value_row_bytes), st);
    ph_end(ISA_PH_HOT, f, 0);
    if (nmiss) {
      collapse_chunk(cur, nmiss, f, sd, row0, nullptr, U, tcap);
      merge_into_T();
    }
    if (f < span) {
      spill_T();
      return a + f;
    }
    refresh_tiny();
    return a + span;
  }

  // next chunk length (rows) for the sort path
  static constexpr int64_t kProbeRows = 4096;  // = one radix-sort tile (RS_TILE)
  int64_t chunk_len(int64_t remaining, int64_t last_len, bool last_flushed, int64_t last_cycle, int64_t since_cycle) {
    const int64_t M = cfg.memory_budget;
    int64_t cmax = cfg.chunk_rows_max > 0 ? cfg.chunk_rows_max : ((int64_t)64 << 20);
    int64_t len;
    if (T.n > 0 && T.n <= 8 && tiny_ok && absorb_supported((int)T.n, S)) {
      // one streaming pass over everything staged: the absorb kernel has no
      // per-chunk memory beyond a per-CTA miss list
      return std::min<int64_t>(remaining, cfg.chunk_rows_max > 0 ? cfg.chunk_rows_max : ((int64_t)1 << 30));
    } else if (last_len == 0) {
      // probe chunk: one sort tile (no histogram/scan passes); it measures
      // the new-group rate for the next chunk and, when the input has only
      // a handful of groups, hands the rest to the absorb kernel
      len = kProbeRows;
    } else if (last_flushed && hot_mode == 1) {
      // large-table absorb: sort the first eighth of the cycle (the table
      // fills with the frequent keys), absorb the rest through its hash image
      static int frac = -1;
      if (frac < 0) { const char* e = getenv("ISA_HOT_FIRST"); frac = e ? std::max(2, atoi(e)) : 8; }
      len = last_cycle / frac + 4096;
    } else if (last_flushed) {
      // the next flush ~ one fill cycle away; the margin follows how much
      // consecutive cycles have varied (rows past the flush are sorted for
      // nothing; a chunk that ends short costs an extra table merge)
      len = last_cycle + (int64_t)((double)last_cycle * cycle_slack()) + 4096;
    } else if (hot_ready() && !cycles.empty() && since_cycle < last_cycle) {
      // the rest of the fill cycle in one hot chunk
      const int64_t rest = last_cycle - since_cycle;
      len = rest + (int64_t)((double)last_cycle * cycle_slack()) + 4096;
    } else if (last_new > 0) {
      double rate = (double)last_new / (double)last_len;
      double need = (double)(M - (int64_t)T.n + 1) / rate;
      len = (int64_t)(need * 1.125) + 4096;
      if (last_len > kProbeRows) len = std::min(len, last_len * 4);
    } else {
      len = last_len * 4;
    }
    len = std::max<int64_t>(len, 4096);
    len = std::min(len, cmax);
    return std::min(len, remaining);
  }

  // relative margin past the predicted flush row: how much consecutive fill
  // cycles have varied (rows past the flush are processed for nothing; a
  // chunk that ends short costs an extra table merge)
  double cycle_slack() const {
    double dev = 0.03;
    if (cycles.size() >= 2) {
      dev = 0;
      for (size_t i = 1; i < cycles.size(); ++i)
        dev = std::max(dev, std::fabs((double)cycles[i] / (double)std::max<int64_t>(cycles[i - 1], 1) - 1.0));
    }
    return std::min(0.125, 0.01 + 4.0 * dev);
  }

  // ------------------------------------------------------- host windows --
  size_t key_elem(int c) const { return dtype_bits(sch.key_dtypes[c]) / 8; }
  size_t val_elem(int j) const { return dtype_bits(sch.val_dtypes[j]) / 8; }

  void stage_window(Window& w, const void* const* key_cols, const void* const* val_cols, int64_t start,
                    int64_t end) {
    w.start = start;
    w.end = end;
    size_t rows = (size_t)(end - start);
    w.keys.resize(sch.n_key_cols);
    w.vals.resize(sch.n_val_cols);
    for (int c = 0; c < sch.n_key_cols; ++c) {
      w.keys[c].ensure(rows * key_elem(c));
      CK(cudaMemcpyAsync(w.keys[c].p, (const char*)key_cols[c] + start * key_elem(c), rows * key_elem(c),
                         cudaMemcpyHostToDevice, h2d));
      led.bytes_h2d += rows * key_elem(c);
    }
    for (int j = 0; j < sch.n_val_cols; ++j) {
      w.vals[j].ensure(rows * val_elem(j));
      CK(cudaMemcpyAsync(w.vals[j].p, (const char*)val_cols[j] + start * val_elem(j), rows * val_elem(j),
                         cudaMemcpyHostToDevice, h2d));
      led.bytes_h2d += rows * val_elem(j);
    }
    CK(cudaEventRecord(w.ready, h2d));
    w.staged = true;
  }

  // the one int64 value column every column-fed slot reads (null: none, or
  // several columns / another dtype / strided records)
  const void* narrow_candidate(const SlotDesc& sd) const {
    { const char* e = getenv("ISA_NARROW"); if (e && e[0] == '0') return nullptr; }   // A/B
    const void* col = nullptr;
    for (int s = 0; s < S; ++s) {
      if (sd.src[s] != SRC_COL) continue;
      if (sd.dtype[s] != ISA_I64 || sd.stride[s] != 0) return nullptr;
      if (col && sd.ptr[s] != col) return nullptr;
      col = sd.ptr[s];
    }
    return col;
  }

  // Row-record layout for the collapse of a large sort-path chunk: true
  // (and sdc pointing into rec_buf) when the slots read >= 2 distinct
  // value columns that fit a 16-byte record.
  RowPack rpk;
  DevBuf rec_buf, rec_sorted;
  bool pack_records(const SlotDesc& sd, SlotDesc& sdc, u32 rows) {
    memset(&rpk, 0, sizeof(rpk));
    int off = 0;
    int col_of[ISA_MAX_SLOTS];
    for (int s = 0; s < S; ++s) {
      col_of[s] = -1;
      if (sd.src[s] != SRC_COL || sd.alias[s] >= 0) continue;
      int found = -1;
      for (int c = 0; c < rpk.nc; ++c)
        if (rpk.src[c] == sd.ptr[s]) found = c;
      if (found < 0) {
        const int el = dtype_bits(sd.dtype[s]) / 8;
        off = (off + el - 1) / el * el;
        rpk.src[rpk.nc] = sd.ptr[s];
        rpk.elem[rpk.nc] = el;
        rpk.off[rpk.nc] = off;
        off += el;
        found = rpk.nc++;
      }
      col_of[s] = found;
    }
    if (rpk.nc < 2 || off > 16) return false;
    rpk.R = off <= 8 ? 8 : 16;
    rec_buf.ensure((size_t)rows * rpk.R + 64);
    for (int s = 0; s < S; ++s) {
      if (col_of[s] < 0) continue;
      sdc.ptr[s] = rec_buf.as<char>() + rpk.off[col_of[s]];
      sdc.stride[s] = rpk.R;
    }
    return true;
  }

  // -------------------------------------------------------- wide merge --
  // Merge `rs` window by window (key-range windows planned from sampled
  // keys, slices staged double-buffered, each window radix-sorted); every
  // window's sorted output -- collapsed into unique groups, or with
  // duplicates kept -- is handed to emit(table, distinct keys).
  // Windows from run directories (tile merge): window w = buckets
  // [wb[w], wb[w + 1]); lb[r * nbound + i] = first row of run r at bucket
  // wb[i + 1]; P at the window boundaries.
  struct TilePlan {
    int nbound = 0;
    std::vector<u32> wb;
    std::vector<u64> pw;
    std::vector<u32> lb;
    u32 cap = 0;
  };
  // Output size estimate for the result's first allocation: the largest
  // run and the OutputEstimator's read-sort-write inversion of the mean fill
  // cycle, C = O ln(O / (O - M)) (sortagg.py:129-144), capped at the rows.
  int64_t estimate_groups(int64_t total_rows) {
    int64_t est = 1;
    for (auto& r : runs) est = std::max<int64_t>(est, r.rows);
    if (!cycles.empty()) {
      double mean = 0;
      for (auto c : cycles) mean += (double)c;
      mean /= (double)cycles.size();
      const double M = (double)cfg.memory_budget;
      if (mean <= M * (1 + 1e-9)) return total_rows;
      auto clen = [&](double o) { return o * std::log(o / (o - M)); };
      double lo = M * (1 + 1e-12), hi = 2 * M;
      while (clen(hi) > mean && hi < 1e18) hi *= 2;
      for (int i = 0; i < 80; ++i) {
        const double mid = 0.5 * (lo + hi);
        if (clen(mid) > mean) lo = mid; else hi = mid;
      }
      est = std::max<int64_t>(est, (int64_t)(0.5 * (lo + hi)));
    }
    return std::min(est, total_rows);
  }

  // Run directories -> D (transposed), P (rows below each bucket), windows
  // of <= W rows on a coarse grid of bucket boundaries, and the per-run
  // slice bounds at the window boundaries.  False: use the sampled-window
  // path (a run without a directory, too many runs for a tile).
  bool build_tile_plan(TilePlan& tp) {
    const int k = (int)runs.size();
    if (!dirs_wanted() || !bk_ready || k < 1) return false;
    for (auto& r : runs)
      if (!r.dir) return false;
    const u32 cap = tile_merge_cap(KW, S, k);
    if (cap < 512) return false;
    const u32 nb1 = bk.nb + 1;
    std::vector<u32*> ptrs(k);
    for (int r = 0; r < k; ++r) ptrs[r] = runs[r].dir;
    tm_dirptrs.ensure(sizeof(u32*) * k + 16);
    CK(cudaMemcpyAsync(tm_dirptrs.p, ptrs.data(), sizeof(u32*) * k, cudaMemcpyHostToDevice, st));
    tm_D.ensure((size_t)nb1 * k * 4 + 64);
    tm_P.ensure((size_t)nb1 * 8 + 64);
    dir_transpose((u32* const*)tm_dirptrs.p, k, nb1, tm_D.as<u32>(), st);
    dir_rowsum(tm_D.as<u32>(), k, nb1, tm_P.as<u64>(), st);
    const u32 C = std::min<u32>(1024, bk.nb);   // nb is a power of two >= 256
    const u32 nc = bk.nb / C + 1;                // coarse points 0, C, 2C, ..., nb
    std::vector<u64> pc(nc);
    CK(cudaMemcpy2DAsync(pc.data(), 8, tm_P.p, (size_t)C * 8, 8, nc, cudaMemcpyDeviceToHost, st));
    sync();
    int64_t W = cfg.merge_window_rows > 0 ? cfg.merge_window_rows : ((int64_t)48 << 20);
    tp.wb.assign(1, 0u);
    tp.pw.assign(1, pc[0]);
    for (u32 c = 1; c < nc; ++c) {
      // cut before coarse step c when it would take the window past W rows
      if ((int64_t)(pc[c] - tp.pw.back()) > W && tp.wb.back() != (c - 1) * C) {
        tp.wb.push_back((c - 1) * C);
        tp.pw.push_back(pc[c - 1]);
      }
    }
    tp.wb.push_back(bk.nb);
    tp.pw.push_back(pc[nc - 1]);
    tp.nbound = (int)tp.wb.size() - 2;
    std::vector<u32> rowsb((size_t)std::max(tp.nbound, 1) * k);
    for (int i = 0; i < tp.nbound; ++i)
      CK(cudaMemcpyAsync(rowsb.data() + (size_t)i * k, tm_D.as<u32>() + (size_t)tp.wb[i + 1] * k, (size_t)k * 4,
                         cudaMemcpyDeviceToHost, st));
    sync();
    tp.lb.assign((size_t)k * std::max(tp.nbound, 1), 0u);
    for (int i = 0; i < tp.nbound; ++i)
      for (int r = 0; r < k; ++r) tp.lb[(size_t)r * tp.nbound + i] = rowsb[(size_t)i * k + r];
    tp.cap = cap;
    return true;
  }

  // One staged window through the tile merge, groups appended to the
  // result in place.  False: a tile overflowed its capacity (skewed
  // buckets); the caller merges the window with the radix-sort path.
  bool tile_window(TilePlan& tp, int w, u32 m, int slot, const std::vector<int64_t>& soff) {
    const int k = (int)runs.size();
    if (tm_base_cap < (size_t)k) {
      if (tm_base_pin) CK(cudaFreeHost(tm_base_pin));
      tm_base_cap = (size_t)k + 64;
      CK(cudaHostAlloc((void**)&tm_base_pin, tm_base_cap * sizeof(MergeSrc), cudaHostAllocDefault));
    }
    // run sources: HBM-resident runs in place (raw or bit-packed), the
    // others from this window's staged slice (staged row = soff + (p - s0))
    MergeSrc* msrc = (MergeSrc*)tm_base_pin;
    for (int r = 0; r < k; ++r) {
      const Run& rn = runs[r];
      MergeSrc q;
      memset(&q, 0, sizeof(q));
      if (!rn.host && rn.path.empty() && rn.pk_dev) {
        q.pk = rn.pk_dev;
        q.blk_off = rn.off_dev;
      } else if (!rn.host && rn.path.empty()) {
        q.lo = rn.lo; q.hi = rn.hi; q.st = rn.st;
        q.off = 0;
      } else {
        const i64 s0 = w == 0 ? 0 : (i64)tp.lb[(size_t)r * tp.nbound + (w - 1)];
        q.lo = stg_lo[slot].as<u64>();
        q.hi = KW == 2 ? stg_hi[slot].as<u64>() : nullptr;
        q.st = S ? stg_st[slot].as<u64>() : nullptr;
        q.off = (i64)soff[r] - s0;
      }
      msrc[r] = q;
    }
    tm_base.ensure((size_t)k * sizeof(MergeSrc) + 16);
    CK(cudaMemcpyAsync(tm_base.p, msrc, (size_t)k * sizeof(MergeSrc), cudaMemcpyHostToDevice, st));
    const u32 target = tp.cap / 2;
    const u64 rows = tp.pw[w + 1] - tp.pw[w];
    const u32 ntiles = (u32)((rows + target - 1) / target);
    if ((size_t)result.n + m > result.lo.bytes / 8) grow_result((size_t)result.n + m);
    const size_t need = (size_t)ntiles * 8 + 64;
    if (tm_status_bytes < need) {
      tm_status.ensure(need);
      tm_status_bytes = tm_status.bytes;
      CK(cudaMemsetAsync(tm_status.p, 0, tm_status.bytes, st));   // epoch 0: never a live status word
    }
    TileMergeArgs a;
    memset(&a, 0, sizeof(a));
    a.P = tm_P.as<u64>();
    a.D = tm_D.as<u32>();
    a.src = (const MergeSrc*)tm_base.p;
    a.fmask = fmask;
    a.k = k;
    a.b_lo = tp.wb[w];
    a.b_hi = tp.wb[w + 1];
    a.target = target;
    a.ntiles = ntiles;
    a.cap = tp.cap;
    a.sd = sd0;
    a.out_lo = result.plo() + result.n;
    a.out_hi = KW == 2 ? result.phi() + result.n : nullptr;
    a.out_st = S ? result.pst() + (size_t)result.n * S : nullptr;
    a.status = tm_status.as<u64>();
    a.ticket = dscal32(19);
    a.total = dscal32(20);
    a.overflow = dscal32(21);
    tm_tb.ensure((size_t)(ntiles + 2) * 4);
    a.tb = tm_tb.as<u32>();
    CK(cudaMemsetAsync(dscal32(20), 0, 2 * sizeof(u32), st));
    ph_begin(ISA_PH_WM_COLLAPSE);
    kt_begin(KF_MERGE, st);
    tile_merge(KW, a, st);
    kt_end(KF_MERGE, (int64_t)m * (8 * KW + 8 * S), st);
    to_host(dscal32(20), 2 * sizeof(u32));
    ph_end(ISA_PH_WM_COLLAPSE, m, 0);
    sync();
    const u32 groups = h_scal[0], over = h_scal[1];
    if (over) return false;
    kt_add_bytes(KF_MERGE, (int64_t)groups * (8 * KW + 8 * S));
    result.n += groups;
    return true;
  }

  // direct != nullptr (wide merge, no tile plan): every window collapses
  // straight into `direct`, numbered on the device after the groups of the
  // windows before it -- no per-window host round trip; the host only reads
  // the count when the rows staged so far could exceed direct's capacity.
  void merge_runs(std::vector<Run>& rs, bool collapse, const std::function<void(Table&, u32)>& emit,
                  TilePlan* tp = nullptr, Table* direct = nullptr) {
    auto& runs = rs;
    const int k = (int)runs.size();
    int64_t total = 0;
    for (auto& r : runs) total += r.rows;
    CK(cudaStreamWaitEvent(st, spill_done, 0));
    int64_t W = cfg.merge_window_rows > 0 ? cfg.merge_window_rows : ((int64_t)48 << 20);
    W = std::max<int64_t>(W, (int64_t)k * 64);
    CK(cudaEventSynchronize(spill_done));   // the host reads host-tier runs directly
    int nb = 0;
    std::vector<u32> lb;
    if (tp) {
      nb = tp->nbound;
      lb = tp->lb;
    } else {
      // ---- plan windows from sampled keys (every F-th row of each run)
      int64_t F = std::max<int64_t>(1, W / (8 * (int64_t)k));
      std::vector<std::pair<u64, u64>> samples;   // (hi, lo)
      int64_t total_s = 0;
      for (auto& r : runs) total_s += (r.rows + F - 1) / F;
      std::vector<u64> tmp_lo(std::max<int64_t>(total_s, 1)), tmp_hi(std::max<int64_t>(total_s, 1), 0);
      {
        // FileStore runs: the high key of the page holding each sampled row
        // (>= its key; split points only need to be keys in range, slice
        // bounds are searched exactly); every other run: the sampled rows'
        // keys, read by one kernel (HBM, mapped host memory, packed blocks)
        std::vector<int64_t> soff(k + 1, 0);
        std::vector<RunRef> refs(k);
        for (int i = 0; i < k; ++i) {
          const Run& r = runs[i];
          const int64_t ns = r.path.empty() ? (r.rows + F - 1) / F : 0;
          soff[i + 1] = soff[i] + ns;
          refs[i] = RunRef{r.lo, r.hi, r.rows, S, r.pk_dev, r.off_dev};
        }
        const int64_t dev_s = soff[k];
        if (dev_s > 0) {
          runref_dev.ensure(sizeof(RunRef) * k);
          bounds_out.ensure(8 * (size_t)(k + 1));
          bounds_lo.ensure(8 * (size_t)dev_s);
          bounds_hi.ensure(8 * (size_t)dev_s);
          CK(cudaMemcpyAsync(runref_dev.p, refs.data(), sizeof(RunRef) * k, cudaMemcpyHostToDevice, st));
          CK(cudaMemcpyAsync(bounds_out.p, soff.data(), 8 * (size_t)(k + 1), cudaMemcpyHostToDevice, st));
          run_samples(KW, runref_dev.as<RunRef>(), k, (const int64_t*)bounds_out.p, F, dev_s, bounds_lo.as<u64>(),
                      bounds_hi.as<u64>(), st);
          CK(cudaMemcpyAsync(tmp_lo.data(), bounds_lo.p, 8 * (size_t)dev_s, cudaMemcpyDeviceToHost, st));
          if (KW == 2) CK(cudaMemcpyAsync(tmp_hi.data(), bounds_hi.p, 8 * (size_t)dev_s, cudaMemcpyDeviceToHost, st));
        }
        int64_t o = dev_s;
        for (auto& r : runs) {
          if (r.path.empty()) continue;
          const int64_t ns = (r.rows + F - 1) / F;
          for (int64_t i = 0; i < ns; ++i) {
            const u32 pg = (u32)((i * F) / ps0.P);
            tmp_lo[o + i] = r.hk_lo[pg];
            if (KW == 2) tmp_hi[o + i] = r.hk_hi[pg];
          }
          o += ns;
        }
        sync();
        samples.reserve(total_s);
        for (int64_t i = 0; i < total_s; ++i) samples.push_back({tmp_hi[i], tmp_lo[i]});
      }
      std::sort(samples.begin(), samples.end());
      std::vector<std::pair<u64, u64>>& bounds = sampled_bounds;
      bounds.clear();
      int64_t acc = (int64_t)k * F;
      for (auto& s : samples) {
        if (acc + F > W && (bounds.empty() || bounds.back() != s)) {
          bounds.push_back(s);
          acc = (int64_t)k * F;
        }
        acc += F;
      }
      nb = (int)bounds.size();
      // ---- exact slice boundaries: lower_bound of every bound in every run
      lb.assign((size_t)k * std::max(nb, 1), 0u);
      if (nb > 0) {
        std::vector<RunRef> refs(k);
        for (int i = 0; i < k; ++i)
          refs[i] = runs[i].path.empty() ? RunRef{runs[i].lo, runs[i].hi, runs[i].rows, S, runs[i].pk_dev, runs[i].off_dev}
                                         : RunRef{nullptr, nullptr, 0u, S, nullptr, nullptr};
        runref_dev.ensure(sizeof(RunRef) * k);
        bounds_lo.ensure(8 * nb);
        bounds_hi.ensure(8 * nb);
        bounds_out.ensure(4 * (size_t)k * nb);
        std::vector<u64> blo(nb), bhi(nb);
        for (int i = 0; i < nb; ++i) { bhi[i] = bounds[i].first; blo[i] = bounds[i].second; }
        CK(cudaMemcpyAsync(runref_dev.p, refs.data(), sizeof(RunRef) * k, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(bounds_lo.p, blo.data(), 8 * nb, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(bounds_hi.p, bhi.data(), 8 * nb, cudaMemcpyHostToDevice, st));
        run_lower_bounds(KW, runref_dev.as<RunRef>(), k, bounds_lo.as<u64>(), bounds_hi.as<u64>(), nb,
                         bounds_out.as<u32>(), st);
        CK(cudaMemcpyAsync(lb.data(), bounds_out.p, 4 * (size_t)k * nb, cudaMemcpyDeviceToHost, st));
        sync();
        for (int i = 0; i < k; ++i)   // FileStore runs: searched on the host (page high keys + one page)
          if (!runs[i].path.empty())
            for (int b = 0; b < nb; ++b) lb[(size_t)i * nb + b] = file_lower_bound(runs[i], bhi[b], blo[b]);
      }
    }
    const int nwin = nb + 1;
    auto slice = [&](int r, int w, u32& s0, u32& s1) {
      s0 = (w == 0) ? 0 : lb[(size_t)r * nb + (w - 1)];
      s1 = (w == nwin - 1) ? runs[r].rows : lb[(size_t)r * nb + w];
    };
    int64_t wmax = 0;
    for (int w = 0; w < nwin; ++w) {
      int64_t rows = 0;
      for (int r = 0; r < k; ++r) { u32 s0, s1; slice(r, w, s0, s1); rows += s1 - s0; }
      wmax = std::max(wmax, rows);
    }
    CK(cudaMemsetAsync(dscal32(12), 0, sizeof(u32), st));   // page checksum failures (FileStore runs)
    for (int i = 0; i < 2; ++i) {
      stg_lo[i].ensure(wmax * 8 + 8);
      if (KW == 2) stg_hi[i].ensure(wmax * 8 + 8);
      if (S) stg_st[i].ensure(wmax * 8 * S + 8);
      CK(cudaEventRecord(stg_free[i], st));
    }
    bool any_packed = false;
    for (auto& r : runs) any_packed |= r.pk_host != nullptr || !r.path.empty();
    if (any_packed) {
      // packed bytes per window: at most the covering blocks (or pages) of every slice
      size_t pmax = 0;
      for (int w = 0; w < nwin; ++w) {
        size_t b = 0;
        for (int r = 0; r < k; ++r) {
          u32 s0, s1;
          slice(r, w, s0, s1);
          if (s1 <= s0) continue;
          if (runs[r].pk_host) {
            b += runs[r].off_host[(s1 - 1) / PK_ROWS + 1] - runs[r].off_host[s0 / PK_ROWS];
          } else if (!runs[r].path.empty()) {
            const u32 p0 = s0 / ps0.P, p1 = (s1 - 1) / ps0.P;
            b += page_off(p1) + page_len(runs[r], p1) - page_off(p0) + 16;
          }
        }
        pmax = std::max(pmax, b);
      }
      for (int i = 0; i < 2; ++i) {
        stg_pk[i].ensure(pmax + 16);
        if (cfg.run_tier == ISA_TIER_FILE && fstage_cap[i] < pmax + 16) {
          CK(cudaEventSynchronize(fstage_done[i]));   // no copy out of it is pending
          grow_pinned(fstage[i], fstage_cap[i], pmax + 16);
        }
      }
    }
    std::vector<int64_t> soffs[2];   // staged row of each run's slice, per staging slot
    soffs[0].assign(k, 0);
    soffs[1].assign(k, 0);
    // HBM-resident runs are read in place by the tile merge (no staging copy)
    const bool inplace = tp && collapse;
    auto resident = [&](const Run& r) { return !r.host && r.path.empty(); };
    // mode 0: every run (h2d stream); 1: all but the HBM-resident runs (the
    // tile merge reads those in place); 2: only the HBM-resident runs, on the
    // compute stream (a window whose tiles overflowed goes to the radix path)
    auto stage = [&](int w, int slot, int mode) -> int64_t {
      cudaStream_t ss = mode == 2 ? st : h2d;
      if (mode != 2) CK(cudaStreamWaitEvent(h2d, stg_free[slot], 0));
      int64_t off = 0;
      size_t poff = 0;
      auto& desc = desc_host[slot];
      desc.clear();
      int64_t unpack_bytes = 0;   // packed bytes read + rows written
      auto& prefs = pref_host[slot];
      prefs.clear();
      size_t fbytes = 0;
      auto& slices = slice_host[slot];
      slices.clear();
      auto& raws = raw_host[slot];
      raws.clear();
      u32 slice_blocks = 0;
      for (int r = 0; r < k; ++r) {
        u32 s0, s1;
        slice(r, w, s0, s1);
        size_t cnt = s1 - s0;
        soffs[slot][r] = off;
        if (!cnt) continue;
        if ((mode == 1 && resident(runs[r])) || (mode == 2 && !resident(runs[r]))) {
          off += cnt;
          continue;
        }
        if (!runs[r].path.empty()) {
          // FileStore run: read the covering pages back from its file
          // (read_page / parse_page, runstore.py:132-142, 315-333)
          const u32 p0 = s0 / ps0.P, p1 = (s1 - 1) / ps0.P;
          const size_t o0 = page_off(p0), len = page_off(p1) + page_len(runs[r], p1) - o0;
          if (fbytes == 0) CK(cudaEventSynchronize(fstage_done[slot]));   // its previous H2D is done
          if (fbytes + len > fstage_cap[slot]) throw IsaError(ISA_ERR_CONTRACT, "page staging overflow");
          pread_all(runs[r].path, fstage[slot] + fbytes, len, o0);
          for (u32 pg = p0; pg <= p1; ++pg) {
            const u32 r0 = pg * (u32)ps0.P;
            PageRef pr;
            pr.src_off = fbytes + (page_off(pg) - o0);
            pr.rows = page_rows(runs[r], pg);
            pr.e0 = std::max(s0, r0) - r0;
            pr.e1 = std::min<u32>(s1, r0 + pr.rows) - r0;
            pr.dst = (u32)(off + (r0 + pr.e0 - s0));
            prefs.push_back(pr);
          }
          fbytes += (len + 15) & ~(size_t)15;
          led.bytes_h2d += len;
          off += cnt;
          continue;
        }
        if (runs[r].pk_host || runs[r].pk_dev) {
          // covering blocks' bytes (host runs: copied into the staging
          // area; HBM runs: read in place), one unpack descriptor per block
          const u32 b0 = s0 / PK_ROWS, b1 = (s1 - 1) / PK_ROWS;
          const u32 o0 = runs[r].off_host[b0], o1 = runs[r].off_host[b1 + 1];
          const bool on_host = runs[r].pk_host != nullptr;
          if (on_host) {
            CK(cudaMemcpyAsync(stg_pk[slot].as<char>() + poff, runs[r].pk_host + o0, o1 - o0, cudaMemcpyHostToDevice, ss));
            led.bytes_h2d += o1 - o0;
          }
          if (!on_host) {
            // HBM-resident: one slice descriptor, the blocks are found on the device
            UnpackSlice sl{runs[r].pk_dev, runs[r].off_dev, s0, s1, (u32)off, slice_blocks};
            slices.push_back(sl);
            slice_blocks += b1 - b0 + 1;
            unpack_bytes += (int64_t)(o1 - o0) + (int64_t)cnt * 8 * (KW + S);
            off += cnt;
            continue;
          }
          const u64 src0 = on_host ? (u64)(uintptr_t)(stg_pk[slot].as<char>() + poff) : (u64)(uintptr_t)(runs[r].pk_dev + o0);
          for (u32 b = b0; b <= b1; ++b) {
            const u32 r0 = b * PK_ROWS;
            UnpackBlk d;
            d.src_off = src0 + (runs[r].off_host[b] - o0);
            d.e0 = std::max(s0, r0) - r0;
            d.e1 = std::min<u32>(s1, std::min<u32>(r0 + PK_ROWS, runs[r].rows)) - r0;
            d.dst = (u32)(off + (r0 + d.e0 - s0));
            d.pad = 0;
            desc.push_back(d);
          }
          if (on_host) poff += o1 - o0;
          unpack_bytes += (int64_t)(o1 - o0) + (int64_t)cnt * 8 * (KW + S);
          off += cnt;
          continue;
        }
        if (!runs[r].host) {   // HBM-resident raw run: pieces for one gather kernel
          for (u32 q = 0; q < cnt; q += RAW_PIECE) {
            RawCopy rc;
            rc.lo = runs[r].lo + s0 + q;
            rc.hi = KW == 2 ? runs[r].hi + s0 + q : nullptr;
            rc.st = S ? runs[r].st + (size_t)(s0 + q) * S : nullptr;
            rc.dst = (u64)(off + q);
            rc.cnt = std::min<u32>(RAW_PIECE, (u32)cnt - q);
            rc.pad = 0;
            raws.push_back(rc);
          }
          off += cnt;
          continue;
        }
        cudaMemcpyKind kind = runs[r].host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        CK(cudaMemcpyAsync(stg_lo[slot].as<u64>() + off, runs[r].lo + s0, cnt * 8, cudaMemcpyDefault, ss));
        if (KW == 2) CK(cudaMemcpyAsync(stg_hi[slot].as<u64>() + off, runs[r].hi + s0, cnt * 8, cudaMemcpyDefault, ss));
        if (S) CK(cudaMemcpyAsync(stg_st[slot].as<u64>() + off * S, runs[r].st + (size_t)s0 * S, cnt * 8 * S, cudaMemcpyDefault, ss));
        if (kind == cudaMemcpyHostToDevice) led.bytes_h2d += cnt * 8 * (KW + S);
        off += cnt;
      }
      if (!prefs.empty()) {
        CK(cudaMemcpyAsync(stg_pk[slot].p, fstage[slot], fbytes, cudaMemcpyHostToDevice, ss));
        if (pref_cap[slot] < prefs.size()) {
          if (pref_pinned[slot]) CK(cudaFreeHost(pref_pinned[slot]));
          pref_cap[slot] = prefs.size() + prefs.size() / 2 + 64;
          CK(cudaHostAlloc((void**)&pref_pinned[slot], pref_cap[slot] * sizeof(PageRef), cudaHostAllocDefault));
        }
        memcpy(pref_pinned[slot], prefs.data(), prefs.size() * sizeof(PageRef));
        stg_pref[slot].ensure(prefs.size() * sizeof(PageRef) + 16);
        CK(cudaMemcpyAsync(stg_pref[slot].p, pref_pinned[slot], prefs.size() * sizeof(PageRef),
                           cudaMemcpyHostToDevice, ss));
        CK(cudaEventRecord(fstage_done[slot], ss));
        page_decode(ps0, stg_pref[slot].as<PageRef>(), (u32)prefs.size(), stg_pk[slot].as<char>(),
                    stg_lo[slot].as<u64>(), stg_hi[slot].as<u64>(), stg_st[slot].as<u64>(), dscal32(12), ss);
      }
      if (!desc.empty()) {
        // descriptors through a pinned buffer (its previous copy must be done)
        CK(cudaEventSynchronize(desc_done[slot]));
        if (desc_cap[slot] < desc.size()) {
          if (desc_pinned[slot]) CK(cudaFreeHost(desc_pinned[slot]));
          desc_cap[slot] = desc.size() + desc.size() / 2 + 64;
          CK(cudaHostAlloc((void**)&desc_pinned[slot], desc_cap[slot] * sizeof(UnpackBlk), cudaHostAllocDefault));
        }
        memcpy(desc_pinned[slot], desc.data(), desc.size() * sizeof(UnpackBlk));
        stg_desc[slot].ensure(desc.size() * sizeof(UnpackBlk) + 16);
        CK(cudaMemcpyAsync(stg_desc[slot].p, desc_pinned[slot], desc.size() * sizeof(UnpackBlk),
                           cudaMemcpyHostToDevice, ss));
        CK(cudaEventRecord(desc_done[slot], ss));
        kt_begin(KF_UNPACK, ss);
        unpack_blocks(stg_desc[slot].as<UnpackBlk>(), (u32)desc.size(), stg_pk[slot].as<char>(), KW, S, fmask,
                      stg_lo[slot].as<u64>(), stg_hi[slot].as<u64>(), stg_st[slot].as<u64>(), ss);
        kt_end(KF_UNPACK, unpack_bytes, ss);
      }
      if (!slices.empty()) {
        CK(cudaEventSynchronize(slice_done[slot]));   // the pinned buffer's previous copy is done
        if (slice_cap[slot] < slices.size()) {
          if (slice_pinned[slot]) CK(cudaFreeHost(slice_pinned[slot]));
          slice_cap[slot] = slices.size() + slices.size() / 2 + 64;
          CK(cudaHostAlloc((void**)&slice_pinned[slot], slice_cap[slot] * sizeof(UnpackSlice), cudaHostAllocDefault));
        }
        memcpy(slice_pinned[slot], slices.data(), slices.size() * sizeof(UnpackSlice));
        stg_slices[slot].ensure(slices.size() * sizeof(UnpackSlice) + 16);
        CK(cudaMemcpyAsync(stg_slices[slot].p, slice_pinned[slot], slices.size() * sizeof(UnpackSlice),
                           cudaMemcpyHostToDevice, ss));
        CK(cudaEventRecord(slice_done[slot], ss));
        kt_begin(KF_UNPACK, ss);
        unpack_slices(stg_slices[slot].as<UnpackSlice>(), (int)slices.size(), slice_blocks, KW, S, fmask,
                      stg_lo[slot].as<u64>(), stg_hi[slot].as<u64>(), stg_st[slot].as<u64>(), ss);
        kt_end(KF_UNPACK, unpack_bytes, ss);
      }
      if (!raws.empty()) {
        CK(cudaEventSynchronize(raw_done[slot]));   // the pinned buffer's previous copy is done
        if (raw_cap[slot] < raws.size()) {
          if (raw_pinned[slot]) CK(cudaFreeHost(raw_pinned[slot]));
          raw_cap[slot] = raws.size() + raws.size() / 2 + 64;
          CK(cudaHostAlloc((void**)&raw_pinned[slot], raw_cap[slot] * sizeof(RawCopy), cudaHostAllocDefault));
        }
        memcpy(raw_pinned[slot], raws.data(), raws.size() * sizeof(RawCopy));
        stg_raw[slot].ensure(raws.size() * sizeof(RawCopy) + 16);
        CK(cudaMemcpyAsync(stg_raw[slot].p, raw_pinned[slot], raws.size() * sizeof(RawCopy), cudaMemcpyHostToDevice, ss));
        CK(cudaEventRecord(raw_done[slot], ss));
        gather_raw(stg_raw[slot].as<RawCopy>(), (u32)raws.size(), KW, S, stg_lo[slot].as<u64>(),
                   stg_hi[slot].as<u64>(), stg_st[slot].as<u64>(), ss);
      }
      if (mode != 2) CK(cudaEventRecord(stg_ready[slot], h2d));
      return off;
    };
    std::vector<int64_t> wrows(nwin);
    // sampled windows [bounds[w-1], bounds[w]) are sorted on key - bounds[w-1]
    // (window 0: key - 0): with a known upper bound (every window but the
    // last) the varying bits are those of the span, known on the host
    auto window_low = [&](int w) -> std::pair<u64, u64> {
      if (tp || w == 0 || w > nb) return {0ull, 0ull};
      return sampled_bounds[w - 1];
    };
    auto window_mask = [&](int w, u64* v) -> bool {
      if (tp || w >= nb) return false;
      const auto L = window_low(w), U = sampled_bounds[w];   // (hi, lo), U exclusive
      u64 uh = U.first, ul = U.second;
      if (ul == 0) { if (uh == 0) return false; --uh; }
      --ul;
      const u64 sh = uh - L.first - (ul < L.second ? 1ull : 0ull), sl = ul - L.second;   // U - 1 - L
      if (sh) { const int b = 63 - __builtin_clzll(sh); v[1] = b == 63 ? ~0ull : ((1ull << (b + 1)) - 1); v[0] = ~0ull; }
      else { v[1] = 0; v[0] = sl ? (63 - __builtin_clzll(sl) == 63 ? ~0ull : ((1ull << (64 - __builtin_clzll(sl))) - 1)) : 1ull; }
      return true;
    };
    const bool dir_mode = direct && collapse && !tp;
    int64_t ub = 0;
    if (dir_mode) {
      ub = direct->n;
      CK(cudaMemcpyAsync(dscal32(25), &direct->n, sizeof(u32), cudaMemcpyHostToDevice, st));
      sync();
      if (stream_want && direct->n == 0) stream_setup();
    }
    const int smode = inplace ? 1 : 0;
    wrows[0] = stage(0, 0, smode);
    for (int w = 0; w < nwin; ++w) {
      const int slot = w & 1;
      if (w + 1 < nwin) wrows[w + 1] = stage(w + 1, slot ^ 1, smode);
      CK(cudaStreamWaitEvent(st, stg_ready[slot], 0));
      const u32 m = (u32)wrows[w];
      led.rows_read_back += m;
      led.merge_windows++;
      if (m == 0) { CK(cudaEventRecord(stg_free[slot], st)); continue; }
      if (inplace) {
        if (tile_window(*tp, w, m, slot, soffs[slot])) {
          CK(cudaEventRecord(stg_free[slot], st));
          continue;
        }
        stage(w, slot, 2);   // the radix path below needs every row staged
      }
      // sort the window's rows by key: keys copied into sort buffers, value = staged row index
      ensure_sort(m);
      const auto wl = dir_mode ? window_low(w) : std::pair<u64, u64>{0ull, 0ull};
      window_keys(KW, stg_lo[slot].as<u64>(), stg_hi[slot].as<u64>(), m, wl.second, wl.first, s_lo[0].as<u64>(),
                  s_hi[0].as<u64>(), s_val[0].as<u32>(), st);
      ph_begin(ISA_PH_WM_SORT);
      u64 vm[2];
      const bool known = dir_mode && window_mask(w, vm);
      if (!known) {
        CK(cudaMemsetAsync(dvary(), 0, 2 * sizeof(u64), st));
        keys_varying(KW, s_lo[0].as<u64>(), s_hi[0].as<u64>(), m, dvary(), st);
      }
      sort_val_iota = true;   // window_keys numbered the staged rows
      int cur = sort_built(m, known ? vm : nullptr);
      ph_end(ISA_PH_WM_SORT, m, 0);
      u32 distinct;
      if (dir_mode) {
        // room for every row of this window after the groups so far
        if (ub + m > (int64_t)(direct->lo.bytes / 8)) {
          direct->n = read_u32(dscal32(25));
          ub = direct->n;
          if (ub + m > (int64_t)(direct->lo.bytes / 8)) {
            if (streaming) { stream_flush(nullptr); CK(cudaStreamSynchronize(xs)); }   // exports read the table that is about to move
            grow_table(*direct, (size_t)ub + m);
          }
        }
        collapse_direct(cur, m, stg_st[slot].as<u64>(), *direct, wl.second, wl.first);
        if (streaming) stream_window(m);
        ub += m;
        CK(cudaEventRecord(stg_free[slot], st));
        continue;
      }
      if (collapse) {
        collapse_chunk(cur, m, 0xFFFFFFFFu, sd0, 0, stg_st[slot].as<u64>(), U, m);
        distinct = U.n;
      } else {
        U.reserve(m, KW, S);
        CK(cudaMemsetAsync(dscal32(7), 0, sizeof(u32), st));
        materialize(KW, s_lo[cur].as<u64>(), s_hi[cur].as<u64>(), s_val[cur].as<u32>(), m, sd0, 0,
                    stg_st[slot].as<u64>(), U.plo(), U.phi(), U.pst(), dscal32(7), st);
        U.n = m;
        distinct = read_u32(dscal32(7));
      }
      CK(cudaEventRecord(stg_free[slot], st));
      emit(U, distinct);
    }
    U.n = 0;
    if (dir_mode) direct->n = read_u32(dscal32(25));
  }

  // one window's collapse straight into t, numbered after *dscal32(25) groups
  // (device count updated in place)
  void collapse_direct(int cur, u32 m, const u64* st_in, Table& t, u64 add_lo, u64 add_hi) {
    ensure_collapse(m);
    CollapseTmp ct;
    ct.flags = cl_flags.as<u32>();
    ct.scan_tmp = scan_tmp.as<u32>();
    ct.partial = cl_partial.as<u64>();
    ct.partial_slot = cl_pslot.as<u32>();
    ct.total = dscal32(26);
    ct.dev_base = dscal32(25);
    ct.key_add_lo = add_lo;
    ct.key_add_hi = add_hi;
    ph_begin(ISA_PH_WM_COLLAPSE);
    kt_begin(KF_COLLAPSE, st);
    collapse(KW, s_lo[cur].as<u64>(), s_hi[cur].as<u64>(), s_val[cur].as<u32>(), m, 0xFFFFFFFFu, sd0, 0, st_in,
             t.plo(), t.phi(), t.pst(), ct, st);
    kt_end(KF_COLLAPSE, (int64_t)m * (8 * KW + 4 + 8 * S), st);
    CK(cudaMemcpyAsync(dscal32(25), dscal32(26), sizeof(u32), cudaMemcpyDeviceToDevice, st));
    ph_end(ISA_PH_WM_COLLAPSE, m, 0);
  }

  // ---- streamed output (isa_set_output_allocator) ----
  // Window w's groups leave for the caller's pinned columns while window
  // w + 1 merges: its group count goes to mapped host memory right after its
  // collapse (one word, written by a kernel), the host -- one window ahead
  // with its enqueues, so the GPU never waits for it -- reads it once the
  // collapse's event completed, and the export stream converts rows
  // [count before, count after) into column slices (device staging) and
  // copies them out with the copy engine.  The allocator is asked after the
  // first window, for max(the OutputEstimator's inversion of the mean fill
  // cycle, total run rows x the first window's groups / rows) plus a margin;
  // a result that outgrows the columns falls back to isa_result_copy.
  bool stream_want = false;
  bool stream_alloc_called = false;   // the allocator is asked at most once per execute
  bool streamed_during_merge = false;
  int64_t stream_total = 0, stream_est = 0, stream_rows0 = 0;
  u32 stream_prev = 0;          // groups exported so far
  int stream_pending = -1;      // h_scal slot of the window whose export is still to be issued
  cudaEvent_t stream_cnt_ev[2] = {nullptr, nullptr};
  void stream_setup() {
    if (!xs) {
      CK(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&xs_ev, cudaEventDisableTiming));
      for (auto& e : stream_cnt_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    stream_prev = 0;
    stream_pending = -1;
    stream_rows0 = 0;
    streaming = true;
    stream_cap = 0;
  }
  bool stream_alloc(u32 groups0) {
    int64_t est = stream_est;
    if (stream_rows0 > 0)
      est = std::max<int64_t>(est, (int64_t)((double)stream_total * (double)groups0 / (double)stream_rows0));
    const int64_t cap = std::min<int64_t>({stream_total, est + est / 32 + 65536, (int64_t)0xFFFFFFF0ll});
    void* kptr[ISA_MAX_KEY_COLS] = {nullptr};
    void* sptr[ISA_MAX_SLOTS] = {nullptr};
    stream_alloc_called = true;
    if (out_alloc(out_user, cap, kptr, sptr) != 0) return false;
    memset(&stream_ed, 0, sizeof(stream_ed));
    stream_ed.ncols = kd0.ncols;
    stream_ed.nslots = S;
    for (int c = 0; c < kd0.ncols; ++c) {
      stream_ed.shift[c] = kd0.shift[c];
      stream_ed.width[c] = kd0.width[c];
      stream_ed.is_signed[c] = dtype_signed(kd0.dtype[c]) ? 1 : 0;
      stream_ed.key_dst[c] = kptr[c];
    }
    for (int s = 0; s < S; ++s) stream_ed.slot_dst[s] = sptr[s];
    stream_cap = (u32)cap;
    return true;
  }
  // the window that just collapsed into the table: publish its count
  void stream_window(u32 m) {
    if (stream_rows0 == 0) stream_rows0 = m;
    const int slot = stream_pending < 0 ? 0 : (stream_pending ^ 1);
    stream_flush(nullptr);                        // the window before it (its count is complete by now)
    to_host(dscal32(26), sizeof(u32), 100 + slot);
    CK(cudaEventRecord(stream_cnt_ev[slot], st));
    stream_pending = slot;
  }
  // issue the pending window's export; t: the table when it may have moved
  void stream_flush(Table* moved) {
    (void)moved;
    if (stream_pending < 0 || !streaming) return;
    const int slot = stream_pending;
    stream_pending = -1;
    CK(cudaEventSynchronize(stream_cnt_ev[slot]));
    const u32 c1 = ((volatile u32*)h_scal)[100 + slot], c0 = stream_prev;
    if (stream_cap == 0 && !stream_alloc(c1)) { streaming = false; return; }
    if (c1 > stream_cap) { streaming = false; return; }   // the columns are too small: isa_result_copy
    const u32 n = c1 - c0;
    if (n == 0) return;
    size_t off = 0;
    ExportDesc ed = stream_ed;
    std::vector<size_t> koff(kd0.ncols), soff(S);
    for (int c = 0; c < kd0.ncols; ++c) { koff[c] = off; off += (((size_t)n * key_elem(c)) + 255) & ~(size_t)255; }
    for (int s = 0; s < S; ++s) { soff[s] = off; off += (((size_t)n * 8) + 255) & ~(size_t)255; }
    if (off + 256 > out_tmp.bytes) {
      CK(cudaStreamSynchronize(xs));   // copies out of the staging area still in flight
      out_tmp.ensure(off + off / 4 + 256);
    }
    for (int c = 0; c < kd0.ncols; ++c) ed.key_dst[c] = out_tmp.as<char>() + koff[c];
    for (int s = 0; s < S; ++s) ed.slot_dst[s] = out_tmp.as<char>() + soff[s];
    CK(cudaStreamWaitEvent(xs, stream_cnt_ev[slot], 0));
    kt_begin(KF_EXPORT, xs);
    export_all(result.plo() + c0, KW == 2 ? result.phi() + c0 : nullptr, result.pst() + (size_t)c0 * S, n, ed, xs);
    kt_end(KF_EXPORT, (int64_t)n * 2 * (8 * KW + 8 * S), xs);
    for (int c = 0; c < kd0.ncols; ++c)
      CK(cudaMemcpyAsync((char*)stream_ed.key_dst[c] + (size_t)c0 * key_elem(c), out_tmp.as<char>() + koff[c],
                         (size_t)n * key_elem(c), cudaMemcpyDeviceToHost, xs));
    for (int s = 0; s < S; ++s)
      CK(cudaMemcpyAsync((char*)stream_ed.slot_dst[s] + (size_t)c0 * 8, out_tmp.as<char>() + soff[s], (size_t)n * 8,
                         cudaMemcpyDeviceToHost, xs));
    stream_prev = c1;
  }
  void end_stream() {
    stream_flush(nullptr);
    CK(cudaStreamSynchronize(xs));
    streamed_ok = streaming && stream_cap > 0 && stream_prev == result.n;
    streamed_during_merge = streamed_ok;
    streaming = false;
  }

  // ---- dense-window wide merge (isa_codec.cu) ----
  // Applies when every run is HBM-resident, the key is one word, every slot
  // is an integer aggregate and the runs' key range holds at most 4 possible
  // keys per run row.  Windows are equal key slabs of D keys (state array of
  // ~40 MB: it lives in L2); slice bounds come from one batched lower-bound
  // search, every window's slice descriptors are built and uploaded once.
  DevBuf dn_state, dn_occ, dn_counts, dn_slices;
  cudaStream_t dn_emit = nullptr;
  cudaEvent_t dn_acc_done[2] = {nullptr, nullptr}, dn_emit_done[2] = {nullptr, nullptr};
  // allow_direct: with an output allocator and device input the occupied
  // entries are emitted straight into the caller's columns (no result table,
  // no export pass); a result larger than the columns' capacity -- the
  // estimate after the first window was short -- merges again into the table
  bool result_in_caller = false;
  bool dense_merge(int64_t total, int64_t est, bool allow_direct = true) {
    { const char* e = getenv("ISA_DENSE"); if (e && e[0] == '0') return false; }   // A/B: sort-based windows
    const int k = (int)runs.size();
    if (KW != 1 || k < 1 || total < 1) return false;
    for (int s = 0; s < S; ++s)
      if (sd0.type[s] != ST_I64) return false;
    for (auto& r : runs)
      if (r.host || !r.path.empty() || r.rows == 0) return false;
    // key range of the runs
    std::vector<RunRef> refs(k);
    for (int i = 0; i < k; ++i) refs[i] = RunRef{runs[i].lo, runs[i].hi, runs[i].rows, S, runs[i].pk_dev, runs[i].off_dev};
    runref_dev.ensure(sizeof(RunRef) * k);
    bounds_lo.ensure(8 * (size_t)2 * k);
    CK(cudaMemcpyAsync(runref_dev.p, refs.data(), sizeof(RunRef) * k, cudaMemcpyHostToDevice, st));
    run_key_range(runref_dev.as<RunRef>(), k, bounds_lo.as<u64>(), st);
    std::vector<u64> kr(2 * (size_t)k);
    CK(cudaMemcpyAsync(kr.data(), bounds_lo.p, 8 * kr.size(), cudaMemcpyDeviceToHost, st));
    sync();
    u64 kmin = ~0ull, kmax = 0;
    for (int i = 0; i < k; ++i) { kmin = std::min(kmin, kr[2 * i]); kmax = std::max(kmax, kr[2 * i + 1]); }
    const u64 span = kmax - kmin;   // keys kmin .. kmin + span
    if (span >= (u64)total * 4) return false;
    const int cnt_slot = dense_count_slot();
    const size_t entry = (size_t)8 * S + (cnt_slot < 0 ? 1 : 0);
    u32 D = 1u << 12;
    while (D < (1u << 26) && (size_t)(2 * D) * std::max<size_t>(entry, 1) <= ((size_t)40 << 20)) D *= 2;
    while (D > (1u << 12) && (u64)(D / 2) > span) D /= 2;
    if (const char* e = getenv("ISA_DENSE_D")) D = std::max<u32>(64u, (u32)atoi(e));   // tests: many small windows
    const u64 nwin64 = span / D + 1;
    if (nwin64 > (1u << 16)) return false;
    const int nwin = (int)nwin64, nb = nwin - 1;
    // exact slice bounds: lower_bound of every window boundary in every run
    std::vector<u32> lb((size_t)k * std::max(nb, 1), 0u);
    if (nb > 0) {
      std::vector<u64> blo(nb), bhi(nb, 0ull);
      for (int i = 0; i < nb; ++i) blo[i] = kmin + (u64)(i + 1) * D;
      bounds_lo.ensure(8 * (size_t)nb);
      bounds_hi.ensure(8 * (size_t)nb);
      bounds_out.ensure(4 * (size_t)k * nb);
      CK(cudaMemcpyAsync(bounds_lo.p, blo.data(), 8 * (size_t)nb, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(bounds_hi.p, bhi.data(), 8 * (size_t)nb, cudaMemcpyHostToDevice, st));
      run_lower_bounds(KW, runref_dev.as<RunRef>(), k, bounds_lo.as<u64>(), bounds_hi.as<u64>(), nb,
                       bounds_out.as<u32>(), st);
      CK(cudaMemcpyAsync(lb.data(), bounds_out.p, 4 * (size_t)k * nb, cudaMemcpyDeviceToHost, st));
      sync();
    }
    // every window's slices, uploaded once
    std::vector<DenseSlice> slices;
    std::vector<size_t> soff(nwin + 1, 0);
    std::vector<u32> wblk(nwin, 0);
    std::vector<int64_t> wrows(nwin, 0), wbytes(nwin, 0);
    slices.reserve((size_t)k * nwin);
    for (int w = 0; w < nwin; ++w) {
      u32 blocks = 0;
      for (int r = 0; r < k; ++r) {
        const u32 s0 = w == 0 ? 0u : lb[(size_t)r * nb + (w - 1)];
        const u32 s1 = w == nwin - 1 ? runs[r].rows : lb[(size_t)r * nb + w];
        if (s1 <= s0) continue;
        DenseSlice d{};
        d.s0 = s0; d.s1 = s1; d.blk0 = blocks;
        if (runs[r].pk_dev) {
          d.pk = runs[r].pk_dev;
          d.off = runs[r].off_dev;
          const u32 b0 = s0 / PK_ROWS, b1 = (s1 - 1) / PK_ROWS;
          blocks += b1 - b0 + 1;
          wbytes[w] += (int64_t)(runs[r].off_host[b1 + 1] - runs[r].off_host[b0]);
        } else {
          d.lo = runs[r].lo;
          d.st = runs[r].st;
          blocks += (s1 - s0 + PK_ROWS - 1) / PK_ROWS;
          wbytes[w] += (int64_t)(s1 - s0) * 8 * (KW + S);
        }
        slices.push_back(d);
        wrows[w] += s1 - s0;
      }
      wblk[w] = blocks;
      soff[w + 1] = slices.size();
    }
    dn_slices.ensure(slices.size() * sizeof(DenseSlice) + 64);
    CK(cudaMemcpyAsync(dn_slices.p, slices.data(), slices.size() * sizeof(DenseSlice), cudaMemcpyHostToDevice, st));
    const u32 nblocks = dense_blocks(D);
    dn_counts.ensure((size_t)(nblocks + 1) * 4);
    // two state arrays: window w + 1 accumulates on the compute stream while
    // window w's entries are emitted (and reset) on a second stream
    dn_state.ensure((size_t)2 * D * 8 * std::max(S, 1) + 64);
    if (cnt_slot < 0) dn_occ.ensure((size_t)2 * D + 64);
    u64* dstate2[2] = {dn_state.as<u64>(), dn_state.as<u64>() + (size_t)D * std::max(S, 1)};
    unsigned char* occ2[2] = {cnt_slot < 0 ? dn_occ.as<unsigned char>() : nullptr,
                              cnt_slot < 0 ? dn_occ.as<unsigned char>() + D : nullptr};
    if (!dn_emit) {
      CK(cudaStreamCreateWithFlags(&dn_emit, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&dn_acc_done[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&dn_emit_done[i], cudaEventDisableTiming));
      }
    }
    for (int i = 0; i < 2; ++i) {
      dense_init(dstate2[i], occ2[i], sd0, D, st);
      CK(cudaEventRecord(dn_emit_done[i], st));
    }
    u32 zero = 0;
    CK(cudaMemcpyAsync(dscal32(25), &zero, sizeof(u32), cudaMemcpyHostToDevice, st));
    sync();   // the descriptor vectors are pageable host memory
    result.n = 0;
    bool direct = allow_direct && out_alloc && !in_on_host && !stream_alloc_called;
    { const char* e = getenv("ISA_DIRECT_OUT"); if (e && e[0] == '0') direct = false; }   // A/B: result table + export
    ExportDesc ded;
    u32 dcap = 0;
    const int64_t led_rb0 = led.rows_read_back, led_mw0 = led.merge_windows;
    if (direct) {
      // the first non-empty window is accumulated and counted before anything
      // is emitted: its groups / rows ratio sizes the caller's columns
      int w0 = 0;
      while (w0 < nwin && wrows[w0] == 0) ++w0;
      u32 g0 = 0;
      if (w0 < nwin) {
        dense_accum(dn_slices.as<DenseSlice>() + soff[w0], (int)(soff[w0 + 1] - soff[w0]), wblk[w0], sd0,
                    kmin + (u64)w0 * D, D, dstate2[0], occ2[0], st);
        dense_count(dstate2[0], occ2[0], S, cnt_slot, D, dn_counts.as<u32>(), st);
        block_counts_scan(dn_counts.as<u32>(), nblocks, dscal32(26), dscal32(25), st);
        g0 = read_u32(dscal32(26));
        // put the probed window back: the loop below accumulates it again
        dense_init(dstate2[0], occ2[0], sd0, D, st);
      }
      int64_t e2 = est;
      if (w0 < nwin) e2 = std::max<int64_t>(e2, (int64_t)((double)total * (double)g0 / (double)wrows[w0]));
      const int64_t cap = std::min<int64_t>({total, e2 + e2 / 32 + (int64_t)D + 65536, (int64_t)0xFFFFFFF0ll});
      void* kptr[ISA_MAX_KEY_COLS] = {nullptr};
      void* sptr[ISA_MAX_SLOTS] = {nullptr};
      stream_alloc_called = true;
      if (out_alloc(out_user, cap, kptr, sptr) != 0) {
        direct = false;
      } else {
        memset(&ded, 0, sizeof(ded));
        ded.ncols = kd0.ncols;
        ded.nslots = S;
        for (int c = 0; c < kd0.ncols; ++c) {
          ded.shift[c] = kd0.shift[c];
          ded.width[c] = kd0.width[c];
          ded.is_signed[c] = dtype_signed(kd0.dtype[c]) ? 1 : 0;
          ded.key_dst[c] = kptr[c];
        }
        for (int s = 0; s < S; ++s) ded.slot_dst[s] = sptr[s];
        dcap = (u32)cap;
        CK(cudaMemsetAsync(dscal32(31), 0, sizeof(u32), st));
        CK(cudaEventRecord(dn_emit_done[0], st));
      }
    }
    if (!direct) {   // room for the estimated output in the result table (grown when short)
      const int64_t W = cfg.merge_window_rows > 0 ? cfg.merge_window_rows : ((int64_t)48 << 20);
      result.reserve(std::max<int64_t>(1, std::min<int64_t>(total, est + est / 16 + W)), KW, S);
    }
    if (stream_want) stream_setup();
    int64_t ub = 0;
    cudaStream_t main_st = st;
    int nact = 0;
    ph_begin(ISA_PH_WM_COLLAPSE);
    for (int w = 0; w < nwin; ++w) {
      const int64_t m = wrows[w];
      led.rows_read_back += m;
      led.merge_windows++;
      if (m == 0) continue;
      const int buf = nact++ & 1;
      const int64_t most = std::min<int64_t>(m, D);
      if (!direct && ub + most > (int64_t)(result.lo.bytes / 8)) {
        CK(cudaStreamSynchronize(dn_emit));
        result.n = read_u32(dscal32(25));
        ub = result.n;
        if (ub + most > (int64_t)(result.lo.bytes / 8)) {
          if (streaming) { stream_flush(nullptr); CK(cudaStreamSynchronize(xs)); }
          grow_table(result, (size_t)ub + most);
        }
      }
      // accumulate on the compute stream once this array's previous window was emitted
      CK(cudaStreamWaitEvent(st, dn_emit_done[buf], 0));
      kt_begin(KF_MERGE, st);
      dense_accum(dn_slices.as<DenseSlice>() + soff[w], (int)(soff[w + 1] - soff[w]), wblk[w], sd0, kmin + (u64)w * D, D,
                  dstate2[buf], occ2[buf], st);
      kt_end(KF_MERGE, wbytes[w] + m * 8 * S, st);
      CK(cudaEventRecord(dn_acc_done[buf], st));
      // count, number and emit on the second stream (the helpers launch on `st`)
      st = dn_emit;
      CK(cudaStreamWaitEvent(st, dn_acc_done[buf], 0));
      dense_count(dstate2[buf], occ2[buf], S, cnt_slot, D, dn_counts.as<u32>(), st);
      block_counts_scan(dn_counts.as<u32>(), nblocks, dscal32(26), dscal32(25), st);
      if (direct)
        dense_emit_cols(dstate2[buf], occ2[buf], sd0, cnt_slot, D, kmin + (u64)w * D, dn_counts.as<u32>(), ded, dcap,
                        dscal32(31), st);
      else
        dense_emit(dstate2[buf], occ2[buf], sd0, cnt_slot, D, kmin + (u64)w * D, dn_counts.as<u32>(), result.plo(),
                   result.pst(), st);
      CK(cudaMemcpyAsync(dscal32(25), dscal32(26), sizeof(u32), cudaMemcpyDeviceToDevice, st));
      CK(cudaEventRecord(dn_emit_done[buf], st));
      if (streaming) stream_window((u32)std::min<int64_t>(m, 0xFFFFFFFFll));
      st = main_st;
      ub += most;
    }
    for (int i = 0; i < 2; ++i) CK(cudaStreamWaitEvent(st, dn_emit_done[i], 0));
    ph_end(ISA_PH_WM_COLLAPSE, total, 0);
    result.n = read_u32(dscal32(25));
    if (result.n > 0xFFFFFFF0u) throw IsaError(ISA_ERR_INVALID_INPUT, "more than 2^32-1 output groups are not supported");
    if (direct) {
      if (read_u32(dscal32(31)) || result.n > dcap) {
        // the caller's columns were too small: merge again, into the result
        // table (the caller then reads it with isa_result_copy)
        led.rows_read_back = led_rb0;
        led.merge_windows = led_mw0;
        return dense_merge(total, est, false);
      }
      result_in_caller = true;
      streamed_ok = true;
      streamed_during_merge = false;
      kt_add_bytes(KF_MERGE, (int64_t)result.n * (8 * KW + 8 * S));
    }
    return true;
  }
  // a COUNT-like slot (int64 sum of ones): nonzero exactly for occupied entries
  int dense_count_slot() const {
    for (int s = 0; s < S; ++s)
      if (sd0.src[s] == SRC_ONE && sd0.op[s] == OP_ADD && sd0.type[s] == ST_I64) return s;
    return -1;
  }

  // Final wide merge of all runs into the result (sortagg.py:588-674)
  void wide_merge() {
    int64_t total = 0;
    for (auto& r : runs) total += r.rows;
    const int64_t W = cfg.merge_window_rows > 0 ? cfg.merge_window_rows : ((int64_t)48 << 20);
    result.n = 0;
    TilePlan tp;
    const bool tiles = build_tile_plan(tp);
    const int64_t est = estimate_groups(total);
    stream_want = out_alloc && in_on_host && !tiles && direct_merge_env();
    { const char* e = getenv("ISA_STREAM_OUT"); if (e && e[0] == '0') stream_want = false; }   // A/B: isa_result_copy
    stream_total = total;
    stream_est = est;
    if (tiles || !dense_merge(total, est)) {
      // room for the estimated output (grown when short)
      result.reserve(std::max<int64_t>(1, std::min<int64_t>(total, est + est / 16 + W)), KW, S);
      merge_runs(runs, true, [&](Table& w, u32) { append_result(w); }, tiles ? &tp : nullptr,
                 direct_merge_env() ? &result : nullptr);
    }
    if (streaming) end_stream();
    stream_want = false;
    if (cfg.run_tier == ISA_TIER_FILE && read_u32(dscal32(12)))
      throw IsaError(ISA_ERR_CORRUPTION, "page checksum mismatch");   // parse_page, runstore.py:132-142
    led.pages_read = led.pages_written;
    led.merge_steps += 1;
    led.merge_levels += 1;
    steps.push_back({ISA_STEP_WIDE, 1, (int64_t)runs.size(), total, (int64_t)result.n, 0});
  }

  static bool direct_merge_env() {   // ISA_DIRECT_MERGE=0 (read per merge): per-window host round trips
    const char* e = getenv("ISA_DIRECT_MERGE");
    return !(e && e[0] == '0');
  }
  void append_result(Table& w) {
    size_t need = (size_t)result.n + w.n;
    if (need > 0xFFFFFFFFull) throw IsaError(ISA_ERR_INVALID_INPUT, "more than 2^32-1 output groups are not supported");
    if (need > result.lo.bytes / 8) grow_result(need);
    CK(cudaMemcpyAsync(result.plo() + result.n, w.plo(), (size_t)w.n * 8, cudaMemcpyDeviceToDevice, st));
    if (KW == 2) CK(cudaMemcpyAsync(result.phi() + result.n, w.phi(), (size_t)w.n * 8, cudaMemcpyDeviceToDevice, st));
    if (S) CK(cudaMemcpyAsync(result.pst() + (size_t)result.n * S, w.pst(), (size_t)w.n * 8 * S, cudaMemcpyDeviceToDevice, st));
    result.n += w.n;
  }

  // ------------------------------------------- traditional / separate --
  std::vector<isa_step> steps;
  int64_t pq_observed = 1, pq_max_run = 0;

  // OutputEstimator.estimate without fill cycles (sortagg.py:146-160)
  int64_t pq_estimate(int64_t rows_seen) {
    if (cfg.output_size_hint > 0) return cfg.output_size_hint;
    int64_t est = std::max<int64_t>({pq_observed, pq_max_run, (int64_t)1});
    if (rows_seen) est = std::min(est, rows_seen);
    return std::max<int64_t>(1, est);
  }

  // merge_mode traditional / separate (sortagg.py:788-849): priority-queue
  // run generation, read-sort-write (every M rows -> one sorted run,
  // duplicates kept, sortagg.py:379-455), fan-in-limited merge levels over
  // the smallest runs that collapse only when their input covers the output
  // estimate (never in separate mode), then a final collapsing merge.
  int64_t execute_pq(int64_t n, const void* const* key_cols, const void* const* val_cols, bool on_host) {
    const int64_t M = cfg.memory_budget;
    const int64_t F = cfg.memory_budget / cfg.page_capacity;
    const bool collapse_allowed = cfg.merge_mode != ISA_MERGE_SEPARATE;
    pq_observed = 1;
    pq_max_run = 0;
    int64_t wrows = on_host ? std::max<int64_t>(cfg.window_rows > 0 ? cfg.window_rows : ((int64_t)32 << 20), M) : n;
    if (on_host) wrows = (wrows / M) * M;   // windows hold whole blocks
    Window& w = win[0];
    for (int64_t ws = 0; ws < n; ws += wrows) {
      const int64_t we = std::min(n, ws + wrows);
      const void* kb[ISA_MAX_KEY_COLS];
      const void* vb[ISA_MAX_VAL_COLS];
      int64_t base = 0;
      if (on_host) {
        sync();   // the previous window is fully consumed
        stage_window(w, key_cols, val_cols, ws, we);
        CK(cudaStreamWaitEvent(st, w.ready, 0));
        for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = w.keys[c].p;
        for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = w.vals[j].p;
        base = ws;
      } else {
        for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = key_cols[c];
        for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = val_cols[j];
      }
      KeyDesc kd = kd_at(kb);
      SlotDesc sd = sd_at(vb);
      for (int64_t a = ws; a < we; a += M) {
        const u32 m = (u32)std::min<int64_t>(M, we - a);
        const int cur = sort_rows(kd, a - base, nullptr, m);
        if (n <= M) {   // everything fits: sort + collapse in memory, no runs (sortagg.py:398-404, 793-795)
          collapse_chunk(cur, m, 0xFFFFFFFFu, sd, a - base, nullptr, result, m);
          return result.n;
        }
        U.reserve(m, KW, S);
        materialize(KW, s_lo[cur].as<u64>(), s_hi[cur].as<u64>(), s_val[cur].as<u32>(), m, sd, a - base, nullptr,
                    U.plo(), U.phi(), U.pst(), nullptr, st);
        U.n = m;
        Run r = alloc_run(m);
        copy_into_run(r, U, m, 0, st);
        runs.push_back(r);
        account_written(r);
        pq_max_run = std::max<int64_t>(pq_max_run, m);
        led.chunks++;
      }
    }
    U.n = 0;
    led.runs_after_generation = (int64_t)runs.size();
    sync();
    // traditional merge levels over the smallest runs (sortagg.py:813-837)
    std::vector<Run> pool = runs;
    while ((int64_t)pool.size() > F) {
      const int64_t o_est = pq_estimate(n);
      std::stable_sort(pool.begin(), pool.end(), [](const Run& x, const Run& y) { return x.rows < y.rows; });
      int level = 0;
      for (auto& r : pool) level = std::max(level, r.level);
      ++level;
      std::vector<Run> nxt;
      for (size_t g = 0; g < pool.size(); g += (size_t)F) {
        std::vector<Run> group(pool.begin() + g, pool.begin() + std::min(pool.size(), g + (size_t)F));
        if (group.size() == 1) { nxt.push_back(group[0]); continue; }
        int64_t total = 0;
        for (auto& r : group) total += r.rows;
        if (total > (int64_t)0xFFFFFFFFll)
          throw IsaError(ISA_ERR_INVALID_INPUT, "a traditional merge step of more than 2^32-1 rows is not supported");
        const bool collapse = collapse_allowed && total >= o_est;
        Run out = alloc_run((u32)total);
        out.level = level;
        size_t off = 0;
        int64_t observed = 0;
        merge_runs(group, collapse, [&](Table& t, u32 distinct) {
          copy_into_run(out, t, t.n, off, st);
          off += t.n;
          observed += distinct;
          sync();   // the window table is reused by the next window
        });
        out.rows = (u32)off;
        for (auto& r : group) led.pages_read += (r.rows + cfg.page_capacity - 1) / cfg.page_capacity;
        account_written(out);
        led.merge_steps += 1;
        pq_observed = std::max(pq_observed, observed);
        steps.push_back({ISA_STEP_TRADITIONAL, collapse ? 1 : 0, (int64_t)group.size(), total, (int64_t)out.rows, level});
        nxt.push_back(out);
      }
      led.merge_levels += 1;
      pool = nxt;
    }
    // final merge with collapse into the output (sortagg.py:839-849)
    int64_t total = 0;
    for (auto& r : pool) total += r.rows;
    const int64_t W = cfg.merge_window_rows > 0 ? cfg.merge_window_rows : ((int64_t)48 << 20);
    result.n = 0;
    result.reserve(std::max<int64_t>(1, std::min<int64_t>(total, W)), KW, S);
    merge_runs(pool, true, [&](Table& t, u32) { append_result(t); });
    for (auto& r : pool) led.pages_read += (r.rows + cfg.page_capacity - 1) / cfg.page_capacity;
    led.merge_steps += 1;
    led.merge_levels += 1;
    steps.push_back({ISA_STEP_FINAL, 1, (int64_t)pool.size(), total, (int64_t)result.n, 0});
    return result.n;
  }

  void grow_result(size_t need) { grow_table(result, need); }
  void grow_table(Table& t, size_t need) {
    const size_t have = t.lo.bytes / 8;
    size_t cap = std::max(need, have + have / 4);
    Table nt;
    nt.reserve(cap, KW, S);
    if (t.n) {
      CK(cudaMemcpyAsync(nt.plo(), t.plo(), (size_t)t.n * 8, cudaMemcpyDeviceToDevice, st));
      if (KW == 2) CK(cudaMemcpyAsync(nt.phi(), t.phi(), (size_t)t.n * 8, cudaMemcpyDeviceToDevice, st));
      if (S) CK(cudaMemcpyAsync(nt.pst(), t.pst(), (size_t)t.n * 8 * S, cudaMemcpyDeviceToDevice, st));
    }
    sync();
    nt.n = t.n;
    t.release();
    t = nt;
    nt.lo.p = nt.hi.p = nt.st.p = nullptr;
  }

  // ------------------------------------------------ one-CTA run generation --
  // Small budgets (isa_seq.cu): the whole read-sort-write run generation in
  // one persistent CTA -- a fill cycle of a few thousand rows costs no launch
  // and no host round trip -- and the only replacement-selection path.
  DevBuf sq_st[4], sq_grp, sq_runlo, sq_runst, sq_off, sq_len, sq_cyc, sq_keys, sq_out;
  bool seq_wanted(int64_t n) const {
    if (cfg.run_generation == ISA_RUNGEN_RS) return true;
    // read-sort-write: opt-in (ISA_SEQ=1, read per execute): config 1 measured
    // 33.4 ms one-CTA vs 34.4 ms chunked -- one SM's memory latency per
    // fill cycle costs what the chunked path spends in launches
    const char* e = getenv("ISA_SEQ");
    if (!e || e[0] != '1') return false;
    return cfg.merge_mode == ISA_MERGE_WIDE && (cfg.run_tier == ISA_TIER_AUTO || cfg.run_tier == ISA_TIER_HBM) &&
           cfg.chunk_rows_max == 0 && cfg.preaggregate == 0 && cfg.hot_absorb == 0 && n <= ((int64_t)1 << 22) &&
           cfg.memory_budget <= 4096 && seq_supported(KW, S, cfg.memory_budget, false);
  }
  void execute_seq(int64_t n, const void* const* key_cols, const void* const* val_cols, bool on_host) {
    if (n > ((int64_t)1 << 27))
      throw IsaError(ISA_ERR_INVALID_INPUT, "replacement selection on the B200 operator takes at most 2^27 rows");
    const bool rs = cfg.run_generation == ISA_RUNGEN_RS;
    const u32 M = (u32)cfg.memory_budget;
    const u32 P = (u32)(cfg.eviction_chunk > 0 ? cfg.eviction_chunk : cfg.page_capacity);
    const void* kb[ISA_MAX_KEY_COLS];
    const void* vb[ISA_MAX_VAL_COLS];
    if (on_host) {
      Window& w = win[0];
      CK(cudaStreamSynchronize(h2d));
      w.staged = false;
      stage_window(w, key_cols, val_cols, 0, n);
      CK(cudaStreamWaitEvent(st, w.ready, 0));
      for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = w.keys[c].p;
      for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = w.vals[j].p;
      w.staged = false;
    } else {
      for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = key_cols[c];
      for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = val_cols[j];
    }
    const int Sx = std::max(S, 1);
    for (auto& b : sq_st) b.ensure((size_t)M * Sx * 8 + 64);
    sq_grp.ensure((size_t)4096 * Sx * 8 + 64);
    sq_runlo.ensure((size_t)n * 8 + 64);
    sq_runst.ensure((size_t)n * Sx * 8 + 64);
    const u32 max_runs = (u32)std::min<int64_t>(rs ? n + 16 : n / std::max<u32>(M, 1) + 16, (int64_t)1 << 24);
    sq_off.ensure((size_t)max_runs * 4 + 64);
    sq_len.ensure((size_t)max_runs * 4 + 64);
    sq_cyc.ensure((size_t)max_runs * 4 + 64);
    sq_keys.ensure((size_t)M * 8 + 64);
    sq_out.ensure(256);
    CK(cudaMemsetAsync(sq_out.p, 0, 256, st));
    SeqBufs b{sq_st[0].as<u64>(), sq_st[1].as<u64>(), sq_st[2].as<u64>(), sq_st[3].as<u64>(), sq_grp.as<u64>(),
              sq_runlo.as<u64>(), sq_runst.as<u64>(), sq_off.as<u32>(), sq_len.as<u32>(), sq_cyc.as<u32>(), max_runs,
              sq_keys.as<u64>(), sq_out.p};
    ph_begin(ISA_PH_SORT);
    seq_rungen(rs, kd_at(kb), sd_at(vb), (u32)n, M, P, b, st);
    ph_end(ISA_PH_SORT, n, 0);
    struct { u32 nruns, ncycles, windows, epochs, cur_n, cur_buf, overflow, pad; u64 probes, absorbs, ressum; } o;
    CK(cudaMemcpyAsync(&o, sq_out.p, sizeof(o), cudaMemcpyDeviceToHost, st));
    sync();
    if (o.overflow) throw IsaError(ISA_ERR_RESOURCE, "run directory of the one-CTA run generation overflowed");
    std::vector<u32> off(o.nruns), len(o.nruns), cyc(o.ncycles);
    if (o.nruns) {
      CK(cudaMemcpyAsync(off.data(), sq_off.p, 4 * (size_t)o.nruns, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(len.data(), sq_len.p, 4 * (size_t)o.nruns, cudaMemcpyDeviceToHost, st));
    }
    if (o.ncycles) CK(cudaMemcpyAsync(cyc.data(), sq_cyc.p, 4 * (size_t)o.ncycles, cudaMemcpyDeviceToHost, st));
    sync();
    for (u32 r = 0; r < o.nruns; ++r) {
      Run rr;
      rr.host = false;
      rr.rows = len[r];
      rr.lo = sq_runlo.as<u64>() + off[r];
      rr.hi = nullptr;
      rr.st = S ? sq_runst.as<u64>() + (size_t)off[r] * S : nullptr;
      runs.push_back(rr);
      account_written(rr);
    }
    for (u32 c = 0; c < o.ncycles; ++c) cycles.push_back(cyc[c]);
    led.chunks += o.epochs;
    led.steady_probes = (int64_t)o.probes;
    led.steady_absorbs = (int64_t)o.absorbs;
    led.steady_resident_sum = (int64_t)o.ressum;
    if (o.nruns == 0 && o.cur_n) {   // no spill: the index is the result
      T.reserve(std::max<size_t>(tcap, o.cur_n + 1), KW, S);
      CK(cudaMemcpyAsync(T.plo(), sq_keys.p, (size_t)o.cur_n * 8, cudaMemcpyDeviceToDevice, st));
      if (S) CK(cudaMemcpyAsync(T.pst(), sq_st[o.cur_buf].p, (size_t)o.cur_n * 8 * S, cudaMemcpyDeviceToDevice, st));
      T.n = o.cur_n;
    }
  }

  // ------------------------------------ cut-then-aggregate (isa_seq.cu) --
  // Small budgets: every read-sort-write fill cycle starts from an empty
  // table, so the cycle boundaries follow from the keys alone.  One CTA
  // finds them (k_cut_scan), then every cycle's run is built in parallel
  // (k_cut_runs): two launches and two host synchronizations for the whole
  // run generation instead of a few launches and syncs per cycle.  The scan
  // stops at the first cycle longer than it can sort in shared memory; the
  // chunked loop continues from that cycle's first row (empty table: exact).
  DevBuf ct_cuts, ct_out, ct_len, ct_lo, ct_st;
  bool cut_staged = false;
  int64_t host_window_rows() const { return cfg.window_rows > 0 ? cfg.window_rows : ((int64_t)32 << 20); }
  bool cut_wanted(int64_t n, bool on_host) const {
    const char* e = getenv("ISA_CUT");   // read per execute (A/B and tests)
    if (e && e[0] == '0') return false;
    if (cfg.run_generation != ISA_RUNGEN_RSW || cfg.merge_mode != ISA_MERGE_WIDE) return false;
    if (cfg.run_tier != ISA_TIER_AUTO && cfg.run_tier != ISA_TIER_HBM) return false;
    if (cfg.chunk_rows_max != 0 || cfg.preaggregate == 1 || cfg.hot_absorb == 1) return false;
    if (!cut_supported(KW, S, cfg.memory_budget)) return false;
    if (n <= cfg.memory_budget || n > ((int64_t)1 << 26)) return false;
    if (on_host && n > host_window_rows()) return false;
    return true;
  }
  // returns the first row the chunked loop still has to process
  int64_t execute_cut(int64_t n, const void* const* key_cols, const void* const* val_cols, bool on_host) {
    const u32 M = (u32)cfg.memory_budget;
    const void* kb[ISA_MAX_KEY_COLS];
    const void* vb[ISA_MAX_VAL_COLS];
    if (on_host) {   // the whole input in one window; the chunked loop reuses it
      Window& w = win[0];
      CK(cudaStreamSynchronize(h2d));
      stage_window(w, key_cols, val_cols, 0, n);
      CK(cudaStreamWaitEvent(st, w.ready, 0));
      for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = w.keys[c].p;
      for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = w.vals[j].p;
      cut_staged = true;
    } else {
      for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = key_cols[c];
      for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = val_cols[j];
    }
    const KeyDesc kd = kd_at(kb);
    const SlotDesc sd = sd_at(vb);
    const u32 max_cuts = (u32)(n / M + 4);
    ct_cuts.ensure((size_t)max_cuts * 4 + 64);
    ct_out.ensure(64);
    CK(cudaMemsetAsync(ct_out.p, 0, 64, st));
    ph_begin(ISA_PH_FLUSH);
    cut_scan(kd, (u32)n, M, ct_cuts.as<u32>(), max_cuts, ct_out.p, st);
    ph_end(ISA_PH_FLUSH, n, n * (key_bits / 8));
    struct { u32 ncuts, stop, batches, overflow; } o;
    CK(cudaMemcpyAsync(&o, ct_out.p, sizeof(o), cudaMemcpyDeviceToHost, st));
    sync();
    if (o.overflow) throw IsaError(ISA_ERR_RESOURCE, "cut directory of the small-budget run generation overflowed");
    const bool done = (int64_t)o.stop == n;
    const u32 ncyc = o.ncuts + (done ? 1u : 0u);
    if (ncyc == 0) return 0;
    const int Sx = std::max(S, 1);
    ct_lo.ensure((size_t)ncyc * M * 8 + 64);
    ct_st.ensure((size_t)ncyc * M * 8 * Sx + 64);
    ct_len.ensure((size_t)ncyc * 4 + 64);
    ph_begin(ISA_PH_COLLAPSE);
    cut_runs(kd, sd, ct_cuts.as<u32>(), ncyc, M, ct_lo.as<u64>(), ct_st.as<u64>(), ct_len.as<u32>(), st);
    ph_end(ISA_PH_COLLAPSE, o.stop, 0);
    std::vector<u32> cuts(o.ncuts + 2), len(ncyc);
    CK(cudaMemcpyAsync(cuts.data(), ct_cuts.p, 4 * cuts.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(len.data(), ct_len.p, 4 * (size_t)ncyc, cudaMemcpyDeviceToHost, st));
    sync();
    led.chunks += ncyc;
    if (o.ncuts == 0) {   // done, no flush: the one cycle is the index, i.e. the result
      T.reserve(std::max<size_t>(tcap, (size_t)len[0] + 1), KW, S);
      CK(cudaMemcpyAsync(T.plo(), ct_lo.p, (size_t)len[0] * 8, cudaMemcpyDeviceToDevice, st));
      if (S) CK(cudaMemcpyAsync(T.pst(), ct_st.p, (size_t)len[0] * 8 * S, cudaMemcpyDeviceToDevice, st));
      T.n = len[0];
      return n;
    }
    for (u32 c = 0; c < ncyc; ++c) {
      Run rr;
      rr.host = false;
      rr.rows = len[c];
      rr.lo = ct_lo.as<u64>() + (size_t)c * M;
      rr.hi = nullptr;
      rr.st = S ? ct_st.as<u64>() + (size_t)c * M * S : nullptr;
      runs.push_back(rr);
      account_written(rr);
    }
    for (u32 c = 0; c < o.ncuts; ++c) cycles.push_back(cuts[c + 1] - cuts[c]);
    return o.stop;
  }

  // ------------------------------------------------------------ execute --
  int64_t execute(int64_t n, const void* const* key_cols, const void* const* val_cols, bool on_host,
                  cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    memset(&led, 0, sizeof(led));
    cycles.clear();
    runs.clear();
    pinned.reset();
    devpool.reset();
    T.n = U.n = result.n = 0;
    for (auto& b : busy) {   // the previous execute synchronized: every copy is done
      spare.push_back(b.t);
      busy_ev_pool.push_back(b.ev);
    }
    busy.clear();
    memset(phases, 0, sizeof(phases));
    for (auto& r : recs) { ev_pool.push_back(r.a); ev_pool.push_back(r.b); }
    recs.clear();
    const long long launch0 = g_launches.load();
    if (n < 0) throw IsaError(ISA_ERR_INVALID_INPUT, "negative row count");
    steps.clear();
    for (auto& rh : rank_hint) { memset(rh.h, 0xFF, sizeof(rh.h)); rh.bit_lo = -1; rh.npass = 0; }
    led.rows_seen = n;
    if (n == 0) { led.kernel_launches = 0; return 0; }
    dev_packed = false;
    packed_ratio = -1;
    rows_left = n;
    tm_mode = tile_merge_env();
    hbm_left = 0;
    bk_ready = false;
    dirpool.reset();
    in_n = n;
    in_on_host = on_host;
    streaming = streamed_ok = false;
    stream_alloc_called = false;
    streamed_during_merge = false;
    result_in_caller = false;
    dense_pred = -1;
    raw_left = 0;
    new_frac_hint = 0;
    sticky_vlo = sticky_vhi = 0;
    sticky_ok = false;
    for (int c = 0; c < sch.n_key_cols; ++c) in_keys[c] = key_cols[c];
    if (cfg.run_tier == ISA_TIER_AUTO) {
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      // half of what is free, counting this handle's own run pool (kept
      // from the previous execute, reused before anything new is allocated)
      hbm_left = cfg.hbm_run_budget > 0 ? cfg.hbm_run_budget
                                        : (int64_t)(0.5 * ((double)fr + (double)devpool.capacity()));
      raw_left = 0.9 * (double)hbm_left;
    }
    if (cfg.merge_mode != ISA_MERGE_WIDE) {
      auto t0p = std::chrono::steady_clock::now();
      int64_t g = execute_pq(n, key_cols, val_cols, on_host);
      sync();
      ph_collect();
      led.ms_run_generation = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0p).count();
      led.n_groups = g;
      led.kernel_launches = g_launches.load() - launch0;
      return g;
    }
    // every run-generation table holds up to M groups: size them once so
    // swapping tables never reallocates (cudaFree would synchronize)
    tcap = (size_t)std::min<int64_t>(cfg.memory_budget, n) + 1;
    k1_mode = cfg.preaggregate == 1 ? 1 : (cfg.preaggregate == 2 ? 0 : -1);
    hot_mode = cfg.hot_absorb == 1 ? 1 : (cfg.hot_absorb == 2 ? 0 : -1);
    if (const char* e = getenv("ISA_HOT")) hot_mode = e[0] == 'n' ? 0 : (e[0] == 'a' && e[1] == 'l' ? 1 : hot_mode);   // A/B
    hash_ver = 0;
    ++t_ver;
    U2.reserve(std::min<size_t>(tcap, tile_rows() + 1), KW, S);
    T.reserve(tcap, KW, S);
    U.reserve(tcap, KW, S);
    auto t0 = std::chrono::steady_clock::now();
    cudaEvent_t rg0 = ev_get(), rg1 = ev_get(), wm1 = ev_get();
    CK(cudaEventRecord(rg0, st));

    const bool seq = seq_wanted(n);
    if (seq) execute_seq(n, key_cols, val_cols, on_host);
    cut_staged = false;
    for (auto& w : win) w.staged = false;   // never reuse a window staged from another execute's input
    const int64_t cut_stop = !seq && cut_wanted(n, on_host) ? execute_cut(n, key_cols, val_cols, on_host) : 0;
    int64_t wrows = on_host ? (cut_staged ? n : host_window_rows()) : n;
    int64_t a = seq ? n : cut_stop, cycle_start = a, last_len = 0, last_cycle = 0;
    bool last_flushed = !cycles.empty();
    if (last_flushed) last_len = last_cycle = cycles.back();
    int wi = 0;
    if (on_host && !seq && !cut_staged) stage_window(win[0], key_cols, val_cols, 0, std::min(n, wrows));
    while (a < n) {
      const void* kb[ISA_MAX_KEY_COLS];
      const void* vb[ISA_MAX_VAL_COLS];
      int64_t base = 0, wend = n;
      if (on_host) {
        Window& w = win[wi];
        if (a >= w.end) {
          // advance: the next window was prefetched (or stage it now)
          cudaEvent_t used;
          CK(cudaEventCreateWithFlags(&used, cudaEventDisableTiming));
          CK(cudaEventRecord(used, st));
          wi ^= 1;
          Window& nw = win[wi];
          if (!(nw.staged && nw.start == a)) {
            CK(cudaStreamWaitEvent(h2d, used, 0));
            stage_window(nw, key_cols, val_cols, a, std::min(n, a + wrows));
          }
          cudaEventDestroy(used);
          continue;
        }
        CK(cudaStreamWaitEvent(st, w.ready, 0));
        // prefetch the following window into the other buffer
        Window& ow = win[wi ^ 1];
        if (w.end < n && !(ow.staged && ow.start == w.end)) {
          cudaEvent_t used;
          CK(cudaEventCreateWithFlags(&used, cudaEventDisableTiming));
          CK(cudaEventRecord(used, st));
          CK(cudaStreamWaitEvent(h2d, used, 0));
          cudaEventDestroy(used);
          stage_window(ow, key_cols, val_cols, w.end, std::min(n, w.end + wrows));
        }
        base = w.start;
        wend = w.end;
        for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = w.keys[c].p;
        for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = w.vals[j].p;
      } else {
        for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = key_cols[c];
        for (int j = 0; j < sch.n_val_cols; ++j) vb[j] = val_cols[j];
      }
      KeyDesc kd = kd_at(kb);
      SlotDesc sd = sd_at(vb);
      if (a == 0 && T.n == 0) {
        // probe: when the first rows hold only a few groups, T starts with
        // exactly those keys (identity states) and the absorb kernel takes
        // every row from here on, the probed ones included
        probe_chunk(kd, sd, a - base, (u32)std::min<int64_t>(probe_rows(), std::min(n, wend) - a));
      }
      int64_t len = chunk_len(std::min(n, wend) - a, last_len, last_flushed, last_cycle, a - cycle_start);
      int64_t b = a + len;
      rows_left = n - a;
      expect_flush = last_flushed;
      int64_t nxt = process_chunk(kd, sd, base, a, b);
      expect_flush = false;
      last_flushed = nxt < b;
      if (last_flushed) {
        last_cycle = nxt - cycle_start;
        cycles.push_back(last_cycle);
        cycle_start = nxt;
        // auto: the hash-image absorb is exact but measured no faster than
        // sorting every row on config 3 (run generation 170 vs 162 ms: the
        // cold hits' atomics miss L2 and the per-cycle table merge doubles,
        // profiles/r2_ab_hot.txt), so auto keeps the sort path; "always"
        // turns it on
        if (hot_mode < 0) hot_mode = 0;
      }
      last_len = nxt - a;
      if (last_len == 0) last_len = 1;
      a = nxt;
    }
    // residue becomes the last run if anything spilled (sortagg.py:353-374);
    // with host-tier runs it stays where it is (HBM): the wide merge reads it
    // next, so a PCIe round trip would buy nothing (the ledger counts it as
    // written like every run)
    if (!runs.empty() && !seq && T.n > 0) {
      if ((cfg.run_tier == ISA_TIER_HOST || cfg.run_tier == ISA_TIER_AUTO) && T.n > 0) {
        Run r;
        r.dir = make_dir();
        r.rows = T.n;
        r.host = false;
        r.lo = T.plo();
        r.hi = KW == 2 ? T.phi() : nullptr;
        r.st = S ? T.pst() : nullptr;
        runs.push_back(r);
        account_written(r);
      } else {
        spill_T();
      }
    }
    led.runs_after_generation = (int64_t)runs.size();
    CK(cudaEventRecord(rg1, st));
    sync();
    auto t1 = std::chrono::steady_clock::now();
    led.ms_run_generation = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (runs.empty()) {
      std::swap(result, T);
      T.n = 0;
    } else {
      wide_merge();
      CK(cudaEventRecord(wm1, st));
      sync();
      led.ms_wide_merge = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, rg1, wm1));
      phases[ISA_PH_WIDE_MERGE].ms += ms;
      phases[ISA_PH_WIDE_MERGE].calls += 1;
    }
    {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, rg0, rg1));
      phases[ISA_PH_RUN_GEN].ms += ms;
      phases[ISA_PH_RUN_GEN].calls += 1;
      phases[ISA_PH_RUN_GEN].rows += n;
    }
    ev_pool.push_back(rg0); ev_pool.push_back(rg1); ev_pool.push_back(wm1);
    ph_collect();
    led.n_groups = result.n;
    // output allocator, nothing streamed (device input, no spill, or the
    // streamed columns were too small and none were handed out): the caller's
    // columns are allocated now, at the exact group count, and filled directly
    if (out_alloc && !streamed_ok && !stream_alloc_called && result.n > 0) {
      void* kptr[ISA_MAX_KEY_COLS] = {nullptr};
      void* sptr[ISA_MAX_SLOTS] = {nullptr};
      if (out_alloc(out_user, (int64_t)result.n, kptr, sptr) == 0) {
        result_copy(kptr, sptr, in_on_host, st);
        streamed_ok = true;
        streamed_during_merge = false;
      }
    }
    led.kernel_launches = g_launches.load() - launch0;
    CK(cudaGetLastError());
    return result.n;
  }

  // Device outputs: one fused export kernel on the caller's stream, no host
  // synchronization (stream order makes the columns ready for the caller).
  // Host outputs: export into a device staging area, then one D2H copy per
  // column and a single synchronization.
  void result_copy(void* const* key_out, void* const* slot_out, bool out_on_host, cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    if (result_in_caller)
      throw IsaError(ISA_ERR_CONTRACT, "the result of the last execute was written to the output allocator's columns");
    const u32 n = result.n;
    if (n == 0) return;
    ExportDesc ed;
    memset(&ed, 0, sizeof(ed));
    ed.ncols = kd0.ncols;
    ed.nslots = S;
    size_t off = 0;
    std::vector<size_t> koff(kd0.ncols), soff(S);
    for (int c = 0; c < kd0.ncols; ++c) {
      ed.shift[c] = kd0.shift[c];
      ed.width[c] = kd0.width[c];
      ed.is_signed[c] = dtype_signed(kd0.dtype[c]) ? 1 : 0;
      koff[c] = off;
      if (key_out[c]) off += (((size_t)n * key_elem(c)) + 255) & ~(size_t)255;
    }
    for (int s = 0; s < S; ++s) {
      soff[s] = off;
      if (slot_out[s]) off += (((size_t)n * 8) + 255) & ~(size_t)255;
    }
    if (out_on_host) out_tmp.ensure(off + 256);
    for (int c = 0; c < kd0.ncols; ++c)
      ed.key_dst[c] = !key_out[c] ? nullptr : (out_on_host ? (void*)(out_tmp.as<char>() + koff[c]) : key_out[c]);
    for (int s = 0; s < S; ++s)
      ed.slot_dst[s] = !slot_out[s] ? nullptr : (out_on_host ? (void*)(out_tmp.as<char>() + soff[s]) : slot_out[s]);
    kt_begin(KF_EXPORT, st);
    export_all(result.plo(), KW == 2 ? result.phi() : nullptr, result.pst(), n, ed, st);
    kt_end(KF_EXPORT, (int64_t)n * 2 * (8 * KW + 8 * S), st);
    if (!out_on_host) return;
    for (int c = 0; c < kd0.ncols; ++c)
      if (key_out[c])
        CK(cudaMemcpyAsync(key_out[c], out_tmp.as<char>() + koff[c], (size_t)n * key_elem(c), cudaMemcpyDeviceToHost, st));
    for (int s = 0; s < S; ++s)
      if (slot_out[s])
        CK(cudaMemcpyAsync(slot_out[s], out_tmp.as<char>() + soff[s], (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    sync();
  }

  // ------------------------------------------------ downstream consumers --
  // Device copies of host columns (pinned or pageable) for the one-shot entry points.
  void to_device_cols(int64_t n, const void* const* key_cols, const void* const* val_cols, int nval,
                      std::vector<const void*>& kb, std::vector<const void*>& vb) {
    Window& w = win[0];
    CK(cudaStreamSynchronize(h2d));
    w.staged = false;
    stage_window(w, key_cols, val_cols, 0, n);
    CK(cudaStreamWaitEvent(st, w.ready, 0));
    kb.assign(sch.n_key_cols, nullptr);
    vb.assign(std::max(nval, 1), nullptr);
    for (int c = 0; c < sch.n_key_cols; ++c) kb[c] = w.keys[c].p;
    for (int j = 0; j < nval; ++j) vb[j] = w.vals[j].p;
    w.staged = false;
  }

  // bench.in_stream_aggregate (bench.py:199-212): rows already sorted on the
  // key -> one group per run of equal consecutive keys (no sort, no budget);
  // the result is read with isa_result_copy.
  int64_t in_stream(int64_t n, const void* const* key_cols, const void* const* val_cols, bool on_host,
                    cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    streaming = streamed_ok = false;
    result_in_caller = false;
    memset(&led, 0, sizeof(led));
    memset(phases, 0, sizeof(phases));
    runs.clear();
    cycles.clear();
    steps.clear();
    result.n = 0;
    if (n < 0) throw IsaError(ISA_ERR_INVALID_INPUT, "negative row count");
    if (n > 0x7FFFFFFFll) throw IsaError(ISA_ERR_INVALID_INPUT, "in-stream aggregation of more than 2^31 rows");
    led.rows_seen = n;
    if (n == 0) return 0;
    const u32 m = (u32)n;
    std::vector<const void*> kb, vb;
    if (on_host) to_device_cols(n, key_cols, val_cols, sch.n_val_cols, kb, vb);
    const KeyDesc kd = kd_at(on_host ? kb.data() : key_cols);
    const SlotDesc sd = sd_at(on_host ? vb.data() : val_cols);
    ensure_sort(m);
    CK(cudaMemsetAsync(dvary(), 0, 2 * sizeof(u64), st));
    build_keys(KW, kd, 0, nullptr, m, s_lo[0].as<u64>(), s_hi[0].as<u64>(), s_val[0].as<u32>(), dvary(), st);
    collapse_chunk(0, m, 0xFFFFFFFFu, sd, 0, nullptr, result, (size_t)m + 1);
    led.n_groups = result.n;
    ph_collect();
    return result.n;
  }

  // HashAggregate baseline (hashagg.py:73-198): one hash table of every
  // group in HBM, rows -> slots, states absorbed (k_hot_absorb), groups in
  // first-arrival order (the reference's in-memory table order).  The
  // result is read with isa_result_copy.
  DevBuf ha_lo, ha_hi, ha_st, ha_occ, ha_first, ha_slot;
  int64_t hash_aggregate(int64_t n, const void* const* key_cols, const void* const* val_cols, bool on_host,
                         cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    streaming = streamed_ok = false;
    result_in_caller = false;
    memset(&led, 0, sizeof(led));
    memset(phases, 0, sizeof(phases));
    runs.clear();
    cycles.clear();
    steps.clear();
    result.n = 0;
    if (n < 0) throw IsaError(ISA_ERR_INVALID_INPUT, "negative row count");
    if (n > ((int64_t)1 << 30)) throw IsaError(ISA_ERR_INVALID_INPUT, "hash aggregation of more than 2^30 rows");
    led.rows_seen = n;
    if (n == 0) return 0;
    std::vector<const void*> kb, vb;
    if (on_host) to_device_cols(n, key_cols, val_cols, sch.n_val_cols, kb, vb);
    const KeyDesc kd = kd_at(on_host ? kb.data() : key_cols);
    const SlotDesc sd = sd_at(on_host ? vb.data() : val_cols);
    u32 cap = 1024;
    while ((int64_t)cap < 2 * n) cap <<= 1;
    ha_lo.ensure((size_t)cap * 8);
    if (KW == 2) ha_hi.ensure((size_t)cap * 8);
    if (S) ha_st.ensure((size_t)cap * 8 * S);
    ha_occ.ensure((size_t)cap * 4);
    ha_first.ensure((size_t)cap * 4);
    ha_slot.ensure((size_t)n * 4 + 64);
    HashAggTable t{ha_lo.as<u64>(), ha_hi.as<u64>(), ha_st.as<u64>(), ha_occ.as<u32>(), ha_first.as<u32>(), cap - 1,
                   dscal32(23)};
    ph_begin(ISA_PH_HOT);
    ha_insert(KW, kd, (u32)n, t, ha_slot.as<u32>(), st);
    ha_init_states(t, sd, st);
    hot_absorb(sd, 0, (u32)n, ha_slot.as<u32>(), t.st, num_sms, st);
    cl_flags.ensure(((size_t)cap + 1) * 4);
    scan_tmp.ensure((scan_tmp_words(cap + 1) + 64) * 4);
    ha_flags(t, cl_flags.as<u32>(), st);
    scan_exclusive_u32(cl_flags.as<u32>(), cap, scan_tmp.as<u32>(), dscal32(24), st);
    ph_end(ISA_PH_HOT, n, 0);
    const u32 g = read_u32(dscal32(24));
    ensure_sort(g);
    ha_compact(t, cl_flags.as<u32>(), s_lo[0].as<u64>(), s_val[0].as<u32>(), st);
    // first-arrival order: sort the groups by their first row
    SortBufs b;
    for (int i = 0; i < 2; ++i) { b.lo[i] = s_lo[i].as<u64>(); b.hi[i] = nullptr; b.val[i] = s_val[i].as<u32>(); }
    b.aux = tile_hist.p;
    b.map_dev = d_hist_mapped;
    b.map_host = h_hist;
    b.pack_ok = true;
    int bits = 1;
    while (bits < 32 && ((int64_t)1 << bits) < n) ++bits;
    const int cur = radix_sort_pairs(1, b, g, 0, bits, st, nullptr);
    result.reserve(std::max<u32>(g, 1), KW, S);
    ha_emit(t, s_val[cur].as<u32>(), g, KW, S, result.plo(), result.phi(), result.pst(), st);
    result.n = g;
    // hashagg.py accounting of an in-memory table: one hash + one access per
    // key column per row, two accesses per key column per match
    led.hash_computations = n;
    led.column_value_accesses = n * sch.n_key_cols + 2 * (int64_t)sch.n_key_cols * (n - (int64_t)g);
    led.n_groups = g;
    sync();
    ph_collect();
    return g;
  }

  // bench.merge_intersect (bench.py:536-550): keys present in both inputs,
  // each strictly ascending (SortAggregate outputs); binary-search ranks of
  // a in b, then a compaction.  Output keys in the input dtypes.
  int64_t merge_intersect(int64_t na, const void* const* a_keys, int64_t nb, const void* const* b_keys,
                          void* const* out_keys, bool on_host, cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    if (na < 0 || nb < 0) throw IsaError(ISA_ERR_INVALID_INPUT, "negative row count");
    if (na > 0x7FFFFFFFll || nb > 0x7FFFFFFFll) throw IsaError(ISA_ERR_INVALID_INPUT, "inputs of more than 2^31 keys");
    if (na == 0 || nb == 0) return 0;
    const u32 ma = (u32)na, mb = (u32)nb;
    ensure_sort(std::max(ma, mb));
    ensure_merge(ma, mb);
    std::vector<const void*> kb, vb;
    if (on_host) to_device_cols(nb, b_keys, nullptr, 0, kb, vb);
    build_keys(KW, kd_at(on_host ? kb.data() : b_keys), 0, nullptr, mb, s_lo[1].as<u64>(), s_hi[1].as<u64>(),
               s_val[1].as<u32>(), dvary(), st);
    if (on_host) {
      // the window's buffers are reused for a: b's keys are already normalized
      CK(cudaStreamSynchronize(st));
      to_device_cols(na, a_keys, nullptr, 0, kb, vb);
    }
    build_keys(KW, kd_at(on_host ? kb.data() : a_keys), 0, nullptr, ma, s_lo[0].as<u64>(), s_hi[0].as<u64>(),
               s_val[0].as<u32>(), dvary(), st);
    rank_match(KW, s_lo[0].as<u64>(), s_hi[0].as<u64>(), ma, s_lo[1].as<u64>(), s_hi[1].as<u64>(), mb,
               mg_rank_a.as<u32>(), mg_match_a.as<u32>(), st);
    u32* pre = mg_match_a.as<u32>() + ma + 1;
    CK(cudaMemcpyAsync(pre, mg_match_a.p, (size_t)ma * 4, cudaMemcpyDeviceToDevice, st));
    scan_exclusive_u32(pre, ma, scan_tmp.as<u32>(), dscal32(8), st);
    const u32 k = read_u32(dscal32(8));
    U.reserve(std::max<u32>(k, 1), KW, S);
    compact_keys(KW, s_lo[0].as<u64>(), s_hi[0].as<u64>(), mg_match_a.as<u32>(), pre, ma, U.plo(), U.phi(), st);
    for (int c = 0; c < kd0.ncols; ++c) {
      if (!out_keys[c] || !k) continue;
      if (on_host) {
        out_tmp.ensure((size_t)k * 8 + 256);
        export_key_col(U.plo(), KW == 2 ? U.phi() : nullptr, k, kd0.dtype[c], kd0.shift[c], kd0.width[c],
                       out_tmp.p, st);
        CK(cudaMemcpyAsync(out_keys[c], out_tmp.p, (size_t)k * key_elem(c), cudaMemcpyDeviceToHost, st));
        sync();
      } else {
        export_key_col(U.plo(), KW == 2 ? U.phi() : nullptr, k, kd0.dtype[c], kd0.shift[c], kd0.width[c],
                       out_keys[c], st);
      }
    }
    U.n = 0;
    return k;
  }

  // ------------------------------------------- fused range exchange --
  // Phase 1: destinations + the destination-sorted permutation (kept in the
  // handle) and per-destination counts.  Phase 2: one kernel gathers every
  // column in that order and stores it into the destination ranks' receive
  // columns (peer pointers), so the data crosses NVLink inside the kernel.
  int pc_cur = 0;
  u32 pc_m = 0;
  int pc_ndest = 0;
  DevBuf pc_tab, pc_off, pc_seg;
  void partition_counts(int64_t n, const void* const* key_cols, const u64* sp_lo, const u64* sp_hi, int ns,
                        int64_t* counts, cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    if (ns < 0 || ns > 255) throw IsaError(ISA_ERR_INVALID_INPUT, "at most 255 splitters");
    if (n > 0x7FFFFFFFll) throw IsaError(ISA_ERR_INVALID_INPUT, "partition of more than 2^31 rows per call");
    const u32 m = (u32)n;
    pc_m = m;
    pc_ndest = ns + 1;
    if (m == 0) { for (int d = 0; d <= ns; ++d) counts[d] = 0; return; }
    ensure_sort(m);
    KeyDesc kd = kd_at(key_cols);
    partition_dest(KW, kd, m, sp_lo, sp_hi, ns, s_lo_buf(0), s_val[0].as<u32>(), st);
    SortBufs b;
    for (int i = 0; i < 2; ++i) { b.lo[i] = s_lo[i].as<u64>(); b.hi[i] = nullptr; b.val[i] = s_val[i].as<u32>(); }
    b.aux = tile_hist.p;
    pc_cur = radix_sort_pairs(1, b, m, 0, 8, st, nullptr);
    word_tmp.ensure(4 * 256);
    count_dest(s_lo[pc_cur].as<u64>(), m, ns + 1, word_tmp.as<u32>(), st);
    std::vector<u32> ub(ns + 1);
    CK(cudaMemcpyAsync(ub.data(), word_tmp.p, 4 * (ns + 1), cudaMemcpyDeviceToHost, st));
    sync();
    u32 prev = 0;
    std::vector<u32> seg(ns + 1);
    for (int d = 0; d <= ns; ++d) { counts[d] = ub[d] - prev; seg[d] = prev; prev = ub[d]; }
    pc_seg.ensure(4 * 256);
    CK(cudaMemcpyAsync(pc_seg.p, seg.data(), 4 * (ns + 1), cudaMemcpyHostToDevice, st));
    sync();
  }
  void scatter_to_peers(int64_t n, const void* const* key_cols, const void* const* val_cols,
                        void* const* peer_cols, const int64_t* peer_off, cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    if ((u32)n != pc_m) throw IsaError(ISA_ERR_CONTRACT, "scatter_to_peers without a matching partition_counts");
    if (n == 0) return;
    PeerScatter ps;
    memset(&ps, 0, sizeof(ps));
    for (int c = 0; c < sch.n_key_cols; ++c) { ps.src[ps.ncols] = key_cols[c]; ps.elem[ps.ncols++] = (int)key_elem(c); }
    for (int j = 0; j < sch.n_val_cols; ++j) { ps.src[ps.ncols] = val_cols[j]; ps.elem[ps.ncols++] = (int)val_elem(j); }
    const size_t ntab = (size_t)pc_ndest * ps.ncols;
    pc_tab.ensure(ntab * sizeof(void*) + 16);
    pc_off.ensure((size_t)pc_ndest * 8 + 16);
    std::vector<u64> offs(pc_ndest);
    for (int d = 0; d < pc_ndest; ++d) offs[d] = (u64)peer_off[d];
    CK(cudaMemcpyAsync(pc_tab.p, peer_cols, ntab * sizeof(void*), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(pc_off.p, offs.data(), (size_t)pc_ndest * 8, cudaMemcpyHostToDevice, st));
    scatter_peers(ps, s_val[pc_cur].as<u32>(), s_lo[pc_cur].as<u64>(), (u32)n, (void* const*)pc_tab.p,
                  pc_off.as<u64>(), pc_seg.as<u32>(), st);
    sync();   // the host buffers above, and the peers may read once every rank returned
  }

  // --------------------------------------------------------- partition --
  void partition(int64_t n, const void* const* key_cols, const void* const* val_cols, const u64* sp_lo,
                 const u64* sp_hi, int ns, void* const* key_out, void* const* val_out, int64_t* counts,
                 cudaStream_t stream) {
    CK(cudaSetDevice(dev));
    st = stream;
    if (ns < 0 || ns > 255) throw IsaError(ISA_ERR_INVALID_INPUT, "at most 255 splitters");
    if (n > 0x7FFFFFFFll) throw IsaError(ISA_ERR_INVALID_INPUT, "partition of more than 2^31 rows per call");
    const u32 m = (u32)n;
    if (m == 0) { for (int d = 0; d <= ns; ++d) counts[d] = 0; return; }
    ensure_sort(m);
    KeyDesc kd = kd_at(key_cols);
    partition_dest(KW, kd, m, sp_lo, sp_hi, ns, s_lo_buf(0), s_val[0].as<u32>(), st);
    SortBufs b;
    for (int i = 0; i < 2; ++i) { b.lo[i] = s_lo[i].as<u64>(); b.hi[i] = nullptr; b.val[i] = s_val[i].as<u32>(); }
    b.aux = tile_hist.p;
    int cur = radix_sort_pairs(1, b, m, 0, 8, st, nullptr);
    const u32* perm = s_val[cur].as<u32>();
    for (int c = 0; c < sch.n_key_cols; ++c) gather_column(key_cols[c], (int)key_elem(c), perm, m, key_out[c], st);
    for (int j = 0; j < sch.n_val_cols; ++j) gather_column(val_cols[j], (int)val_elem(j), perm, m, val_out[j], st);
    word_tmp.ensure(4 * 256);
    count_dest(s_lo[cur].as<u64>(), m, ns + 1, word_tmp.as<u32>(), st);
    std::vector<u32> ub(ns + 1);
    CK(cudaMemcpyAsync(ub.data(), word_tmp.p, 4 * (ns + 1), cudaMemcpyDeviceToHost, st));
    sync();
    u32 prev = 0;
    for (int d = 0; d <= ns; ++d) { counts[d] = ub[d] - prev; prev = ub[d]; }
  }
  u64* s_lo_buf(int i) { return s_lo[i].as<u64>(); }
};

int fail(isa_handle* h, const std::exception& e);

}  // namespace

struct isa_handle {
  Engine* eng;
};

namespace {
int fail(isa_handle* h, const std::exception& e) {
  const IsaError* ie = dynamic_cast<const IsaError*>(&e);
  int code = ie ? ie->code : ISA_ERR_RESOURCE;
  if (h && h->eng) h->eng->err = e.what();
  else g_create_error = e.what();
  return code;
}
}  // namespace

extern "C" {

const char* isa_version(void) { return "insortagg_b200 0.1.0 (sm_100a)"; }

isa_handle* isa_create(const isa_config* config, const isa_schema* schema) {
  if (!config || !schema) {
    g_create_error = "null config or schema";
    return nullptr;
  }
  try {
    isa_handle* h = new isa_handle;
    h->eng = new Engine(*config, *schema);
    g_create_error.clear();
    return h;
  } catch (const std::exception& e) {
    fail(nullptr, e);
    return nullptr;
  }
}

void isa_destroy(isa_handle* h) {
  if (!h) return;
  delete h->eng;
  delete h;
}

int isa_execute(isa_handle* h, int64_t n_rows, const void* const* key_cols, const void* const* val_cols,
                int32_t input_on_host, void* stream, int64_t* n_groups_out) {
  if (!h) return ISA_ERR_CONTRACT;
  (void)cudaGetLastError();   // a failed call before this one must not fail this one
  try {
    int64_t g = h->eng->execute(n_rows, key_cols, val_cols, input_on_host != 0, (cudaStream_t)stream);
    if (n_groups_out) *n_groups_out = g;
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

int isa_in_stream_aggregate(isa_handle* h, int64_t n_rows, const void* const* key_cols, const void* const* val_cols,
                            int32_t input_on_host, void* stream, int64_t* n_groups_out) {
  if (!h) return ISA_ERR_CONTRACT;
  try {
    int64_t g = h->eng->in_stream(n_rows, key_cols, val_cols, input_on_host != 0, (cudaStream_t)stream);
    if (n_groups_out) *n_groups_out = g;
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

int isa_hash_aggregate(isa_handle* h, int64_t n_rows, const void* const* key_cols, const void* const* val_cols,
                       int32_t input_on_host, void* stream, int64_t* n_groups_out) {
  if (!h) return ISA_ERR_CONTRACT;
  try {
    int64_t g = h->eng->hash_aggregate(n_rows, key_cols, val_cols, input_on_host != 0, (cudaStream_t)stream);
    if (n_groups_out) *n_groups_out = g;
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

int isa_merge_intersect(isa_handle* h, int64_t n_a, const void* const* a_keys, int64_t n_b,
                        const void* const* b_keys, void* const* out_keys, int32_t on_host, void* stream,
                        int64_t* n_out) {
  if (!h) return ISA_ERR_CONTRACT;
  try {
    int64_t k = h->eng->merge_intersect(n_a, a_keys, n_b, b_keys, out_keys, on_host != 0, (cudaStream_t)stream);
    if (n_out) *n_out = k;
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

int isa_partition_counts(isa_handle* h, int64_t n_rows, const void* const* key_cols, const uint64_t* split_lo,
                         const uint64_t* split_hi, int32_t n_split, int64_t* counts, void* stream) {
  if (!h || !counts) return ISA_ERR_CONTRACT;
  try {
    h->eng->partition_counts(n_rows, key_cols, (const u64*)split_lo, (const u64*)split_hi, n_split, counts,
                             (cudaStream_t)stream);
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

int isa_scatter_to_peers(isa_handle* h, int64_t n_rows, const void* const* key_cols, const void* const* val_cols,
                         void* const* peer_cols, const int64_t* peer_offsets, void* stream) {
  if (!h || !peer_cols || !peer_offsets) return ISA_ERR_CONTRACT;
  try {
    h->eng->scatter_to_peers(n_rows, key_cols, val_cols, peer_cols, peer_offsets, (cudaStream_t)stream);
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

// Multi-GPU execute in one process: handles[g] lives
// on its own device (isa_config.device) and holds shard g of the input in
// device memory.  Sampled splitters cut the key space into n_devices ranges
// of about equal row counts; every device partitions its shard by range and
// the fused scatter kernel stores the rows straight into the destination
// devices' receive columns over NVLink peer access (one process: plain
// device pointers, no IPC); then every device runs its operator on its range,
// one host thread per device.  Range g's result is held by handles[g].
int isa_execute_multi(isa_handle* const* handles, int32_t n_devices, const int64_t* n_rows,
                      const void* const* const* key_cols, const void* const* const* val_cols, void* const* streams,
                      int64_t* n_groups_out) {
  if (!handles || n_devices < 1 || n_devices > 256 || !n_rows || !key_cols || !val_cols) return ISA_ERR_CONTRACT;
  const int G = n_devices;
  for (int g = 0; g < G; ++g)
    if (!handles[g] || !handles[g]->eng) return ISA_ERR_CONTRACT;
  isa_handle* h0 = handles[0];
  std::vector<std::vector<void*>> recv(G);   // receive columns of every device (freed on every path)
  auto free_recv = [&]() {
    for (int d = 0; d < G; ++d) {
      cudaSetDevice(handles[d]->eng->dev);
      for (void* p : recv[d]) if (p) cudaFree(p);
      recv[d].clear();
    }
  };
  try {
    Engine* e0 = h0->eng;
    const int nk = e0->sch.n_key_cols, nv = e0->sch.n_val_cols, ncol = nk + nv;
    auto stream_of = [&](int g) { return streams ? (cudaStream_t)streams[g] : (cudaStream_t) nullptr; };
    if (G == 1) {
      int64_t ng = e0->execute(n_rows[0], key_cols[0], val_cols[0], false, stream_of(0));
      if (n_groups_out) n_groups_out[0] = ng;
      return ISA_OK;
    }
    // peer access between every pair of distinct devices
    for (int a = 0; a < G; ++a)
      for (int b = 0; b < G; ++b) {
        const int da = handles[a]->eng->dev, db = handles[b]->eng->dev;
        if (da == db) continue;
        int can = 0;
        CK(cudaDeviceCanAccessPeer(&can, da, db));
        if (!can) throw IsaError(ISA_ERR_RESOURCE, "isa_execute_multi needs peer access between the devices");
        CK(cudaSetDevice(da));
        const cudaError_t pe = cudaDeviceEnablePeerAccess(db, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
        (void)cudaGetLastError();
      }
    // 1. sampled normalized keys of every shard -> G - 1 splitters at equal-count quantiles
    const int64_t per = 1 << 16;
    std::vector<std::pair<u64, u64>> samples;   // (hi, lo)
    for (int g = 0; g < G; ++g) {
      Engine* e = handles[g]->eng;
      if (n_rows[g] <= 0) continue;
      CK(cudaSetDevice(e->dev));
      const int64_t stride = std::max<int64_t>(1, n_rows[g] / per), ns = (n_rows[g] + stride - 1) / stride;
      u64 *dlo = nullptr, *dhi = nullptr;
      CK(cudaMalloc(&dlo, 8 * (size_t)ns));
      CK(cudaMalloc(&dhi, 8 * (size_t)ns));
      isa::sample_keys(e->kd_at(key_cols[g]), n_rows[g], stride, dlo, dhi, stream_of(g));
      std::vector<u64> lo(ns), hi(ns);
      CK(cudaMemcpyAsync(lo.data(), dlo, 8 * (size_t)ns, cudaMemcpyDeviceToHost, stream_of(g)));
      CK(cudaMemcpyAsync(hi.data(), dhi, 8 * (size_t)ns, cudaMemcpyDeviceToHost, stream_of(g)));
      CK(cudaStreamSynchronize(stream_of(g)));
      cudaFree(dlo);
      cudaFree(dhi);
      for (int64_t i = 0; i < ns; ++i) samples.push_back({hi[i], lo[i]});
    }
    std::sort(samples.begin(), samples.end());
    std::vector<u64> sp_lo(G - 1, ~0ull), sp_hi(G - 1, ~0ull);
    if (!samples.empty())
      for (int r = 0; r + 1 < G; ++r) {
        const size_t pos = std::min(samples.size() - 1, samples.size() * (size_t)(r + 1) / (size_t)G);
        sp_hi[r] = samples[pos].first;
        sp_lo[r] = samples[pos].second;
      }
    // 2. every shard: destinations by splitter + per-destination counts (the permutation stays in the handle)
    std::vector<std::vector<int64_t>> counts(G, std::vector<int64_t>(G, 0));
    for (int g = 0; g < G; ++g) {
      Engine* e = handles[g]->eng;
      CK(cudaSetDevice(e->dev));
      u64 *dlo = nullptr, *dhi = nullptr;
      CK(cudaMalloc(&dlo, 8 * (size_t)G));
      CK(cudaMalloc(&dhi, 8 * (size_t)G));
      CK(cudaMemcpy(dlo, sp_lo.data(), 8 * (size_t)(G - 1), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dhi, sp_hi.data(), 8 * (size_t)(G - 1), cudaMemcpyHostToDevice));
      e->partition_counts(n_rows[g], key_cols[g], dlo, dhi, G - 1, counts[g].data(), stream_of(g));
      cudaFree(dlo);
      cudaFree(dhi);
    }
    // 3. receive columns on every destination; source g's block lands at sum of counts[q][d], q < g
    std::vector<int64_t> recv_n(G, 0);
    for (int d = 0; d < G; ++d) {
      for (int g = 0; g < G; ++g) recv_n[d] += counts[g][d];
      Engine* e = handles[d]->eng;
      CK(cudaSetDevice(e->dev));
      recv[d].assign(ncol, nullptr);
      for (int c = 0; c < ncol; ++c) {
        const size_t el = c < nk ? e->key_elem(c) : e->val_elem(c - nk);
        CK(cudaMalloc(&recv[d][c], std::max<size_t>((size_t)recv_n[d] * el, 256)));
      }
    }
    std::vector<void*> table((size_t)G * ncol);
    for (int d = 0; d < G; ++d)
      for (int c = 0; c < ncol; ++c) table[(size_t)d * ncol + c] = recv[d][c];
    for (int g = 0; g < G; ++g) {
      std::vector<int64_t> offs(G, 0);
      for (int d = 0; d < G; ++d)
        for (int q = 0; q < g; ++q) offs[d] += counts[q][d];
      handles[g]->eng->scatter_to_peers(n_rows[g], key_cols[g], val_cols[g], table.data(), offs.data(), stream_of(g));
    }
    for (int g = 0; g < G; ++g) {   // every store landed before anyone reads
      CK(cudaSetDevice(handles[g]->eng->dev));
      CK(cudaDeviceSynchronize());
    }
    // 4. the local operator on every range, one host thread per device
    std::vector<int> rc(G, ISA_OK);
    std::vector<int64_t> ng(G, 0);
    std::vector<std::thread> th;
    for (int d = 0; d < G; ++d)
      th.emplace_back([&, d]() {
        std::vector<const void*> kc(recv[d].begin(), recv[d].begin() + nk), vc(recv[d].begin() + nk, recv[d].end());
        if (vc.empty()) vc.push_back(nullptr);
        rc[d] = isa_execute(handles[d], recv_n[d], kc.data(), vc.data(), 0, streams ? streams[d] : nullptr, &ng[d]);
      });
    for (auto& t : th) t.join();
    free_recv();
    for (int d = 0; d < G; ++d) {
      if (rc[d] != ISA_OK) {
        if (d) h0->eng->err = handles[d]->eng->err;
        return rc[d];
      }
      if (n_groups_out) n_groups_out[d] = ng[d];
    }
    return ISA_OK;
  } catch (const std::exception& e) {
    free_recv();
    return fail(h0, e);
  }
}

// An IPC handle names a whole allocation (a caching allocator hands out
// pointers inside larger segments): the 72-byte handle carries the
// allocation's handle plus the pointer's offset inside it (base from the
// driver's cuMemGetAddressRange, reached through the runtime's entry-point
// query so the library does not link libcuda).
typedef int (*GetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);
static GetAddressRangeFn address_range_fn() {
  static GetAddressRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (GetAddressRangeFn)p;
  }
  return fn;
}

int isa_ipc_handle(void* dev_ptr, void* handle_out /* 72 bytes */) {
  if (!dev_ptr || !handle_out) return ISA_ERR_CONTRACT;
  GetAddressRangeFn fn = address_range_fn();
  if (!fn) return ISA_ERR_CUDA;
  unsigned long long base = 0;
  size_t size = 0;
  if (fn(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0) return ISA_ERR_CUDA;
  cudaIpcMemHandle_t hnd;
  if (cudaIpcGetMemHandle(&hnd, (void*)(uintptr_t)base) != cudaSuccess) return ISA_ERR_CUDA;
  const uint64_t off = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  memcpy(handle_out, &hnd, sizeof(hnd));
  memcpy((char*)handle_out + 64, &off, 8);
  return ISA_OK;
}

int isa_ipc_open(const void* handle, void** base_out, void** dev_ptr_out) {
  if (!handle || !base_out || !dev_ptr_out) return ISA_ERR_CONTRACT;
  cudaIpcMemHandle_t hnd;
  uint64_t off = 0;
  memcpy(&hnd, handle, sizeof(hnd));
  memcpy(&off, (const char*)handle + 64, 8);
  if (cudaIpcOpenMemHandle(base_out, hnd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return ISA_ERR_CUDA;
  *dev_ptr_out = (char*)*base_out + off;
  return ISA_OK;
}

int isa_ipc_close(void* base) {
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? ISA_OK : ISA_ERR_CUDA;
}

int isa_set_spill_dir(isa_handle* h, const char* dir, int64_t first_run_id) {
  if (!h || !dir) return ISA_ERR_CONTRACT;
  h->eng->spill_dir = dir;
  h->eng->next_run_id = first_run_id;
  return ISA_OK;
}

int isa_result_copy(isa_handle* h, void* const* key_out, void* const* slot_out, int32_t out_on_host, void* stream) {
  if (!h) return ISA_ERR_CONTRACT;
  try {
    h->eng->result_copy(key_out, slot_out, out_on_host != 0, (cudaStream_t)stream);
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

int isa_set_output_allocator(isa_handle* h, isa_alloc_fn fn, void* user) {
  if (!h) return ISA_ERR_CONTRACT;
  h->eng->out_alloc = fn;
  h->eng->out_user = user;
  return ISA_OK;
}

int isa_result_streamed(isa_handle* h) {
  if (!h) return 0;
  return h->eng->streamed_ok ? (h->eng->streamed_during_merge ? 2 : 1) : 0;
}

int isa_metrics(isa_handle* h, isa_ledger* out) {
  if (!h || !out) return ISA_ERR_CONTRACT;
  *out = h->eng->led;
  return ISA_OK;
}

int64_t isa_cycles(isa_handle* h, int64_t* out, int64_t cap) {
  if (!h) return -1;
  auto& c = h->eng->cycles;
  for (int64_t i = 0; i < (int64_t)c.size() && i < cap; ++i) out[i] = c[i];
  return (int64_t)c.size();
}

int64_t isa_steps(isa_handle* h, isa_step* out, int64_t cap) {
  if (!h) return -1;
  auto& s = h->eng->steps;
  for (int64_t i = 0; i < (int64_t)s.size() && i < cap; ++i) out[i] = s[i];
  return (int64_t)s.size();
}

int isa_phase_stats(isa_handle* h, isa_phase* out, int cap) {
  if (!h) return -1;
  for (int i = 0; i < ISA_PH_COUNT && i < cap; ++i) out[i] = h->eng->phases[i];
  return ISA_PH_COUNT;
}

int64_t isa_launch_count(void) { return (int64_t)isa::g_launches.load(); }

void isa_set_kernel_timing(int32_t on) { isa::kt_set(on != 0); }
void isa_kernel_timing_reserve(int64_t events) { isa::kt_reserve(events); }

int isa_kernel_stats(isa_kstat* out, int cap) {
  double ms[isa::KF_COUNT];
  int64_t la[isa::KF_COUNT], by[isa::KF_COUNT];
  isa::kt_collect(ms, la, by);
  for (int f = 0; f < isa::KF_COUNT && f < cap; ++f) out[f] = isa_kstat{ms[f], la[f], by[f]};
  return isa::KF_COUNT;
}

int64_t isa_run_rows(isa_handle* h, int64_t* out, int64_t cap) {
  if (!h) return -1;
  auto& r = h->eng->runs;
  for (int64_t i = 0; i < (int64_t)r.size() && i < cap; ++i) out[i] = r[i].rows;
  return (int64_t)r.size();
}

const char* isa_last_error(isa_handle* h) {
  if (!h) return g_create_error.c_str();
  return h->eng->err.c_str();
}

int isa_sample_keys(isa_handle* h, int64_t n_rows, const void* const* key_cols, int64_t stride, uint64_t* out_lo,
                    uint64_t* out_hi, void* stream) {
  if (!h) return ISA_ERR_CONTRACT;
  try {
    if (stride < 1) throw IsaError(ISA_ERR_INVALID_INPUT, "stride must be positive");
    CK(cudaSetDevice(h->eng->dev));
    (void)cudaGetLastError();
    KeyDesc kd = h->eng->kd_at(key_cols);
    isa::sample_keys(kd, n_rows, stride, out_lo, out_hi, (cudaStream_t)stream);
    CK(cudaGetLastError());
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

int isa_partition(isa_handle* h, int64_t n_rows, const void* const* key_cols, const void* const* val_cols,
                  const uint64_t* split_lo, const uint64_t* split_hi, int32_t n_splitters, void* const* key_out,
                  void* const* val_out, int64_t* counts_out, void* stream) {
  if (!h) return ISA_ERR_CONTRACT;
  try {
    h->eng->partition(n_rows, key_cols, val_cols, split_lo, split_hi, n_splitters, key_out, val_out, counts_out,
                      (cudaStream_t)stream);
    return ISA_OK;
  } catch (const std::exception& e) {
    return fail(h, e);
  }
}

}  // extern "C"
