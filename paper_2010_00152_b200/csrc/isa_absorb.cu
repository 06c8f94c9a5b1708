// Tiny-table absorb kernel (early aggregation against a register-resident index).
#include "isa_kernels.h"

#include <algorithm>

namespace isa {

// ======================================================= tiny absorb ====
// The early-aggregation probe (OrderedIndex.insert_or_aggregate ABSORBED
// branch, memindex.py:197-236) for a resident table of nt <= 8 groups: the
// table keys are kernel parameters (constant bank), every row is compared
// against all of them, and hits are combined one slot at a time: for a batch
// of AB_ROWS rows per thread the slot's values are loaded (AB_ROWS loads in
// flight per thread), reduced per table row in registers (one-hot,
// predicated), and folded into a per-thread shared-memory accumulator.  Rows
// whose key is not resident are appended, in row order, to a per-CTA miss
// list.  One CTA processes one contiguous row range; the per-CTA partial
// states are folded into the table afterwards, so a discarded pass (a flush
// inside the chunk) costs nothing.
#define AB_THREADS 256
#define AB_ROWS 16
#define AB_MAX_CELLS 54   // (nt + 1) * S accumulators per thread (shared memory)

enum { CLS_ADD_I = 0, CLS_ADD_F = 1, CLS_MIN_I = 2, CLS_MAX_I = 3, CLS_MIN_F = 4, CLS_MAX_F = 5 };

// Load one column for the AB_ROWS rows of this thread's batch: one dtype
// switch per (batch, column), then an unrolled, coalesced load per row.
// FULL: every row of the batch is valid (no per-row bounds predicate).
template <bool FULL, typename T>
__device__ __forceinline__ void ab_load_col(const void* p, i64 base, u32 lim, T (&out)[AB_ROWS]) {
  const T* q = (const T*)p + base;
#pragma unroll
  for (int k = 0; k < AB_ROWS; ++k)
    out[k] = (FULL || (u32)(k * AB_THREADS) < lim) ? __ldg(q + k * AB_THREADS) : T(0);
}

// Key field (order-preserving unsigned image) of every row of the batch.
template <bool FULL>
__device__ __forceinline__ void ab_key_field(int dt, const void* p, i64 base, u32 lim, u64 (&f)[AB_ROWS]) {
  switch (dt) {
    case DT_U8: case DT_I8: {
      unsigned char t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
      const u64 x = dt == DT_I8 ? 0x80ull : 0;
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) f[k] = (u64)t[k] ^ x;
    } break;
    case DT_U16: case DT_I16: {
      unsigned short t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
      const u64 x = dt == DT_I16 ? 0x8000ull : 0;
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) f[k] = (u64)t[k] ^ x;
    } break;
    case DT_U32: case DT_I32: {
      unsigned int t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
      const u64 x = dt == DT_I32 ? 0x80000000ull : 0;
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) f[k] = (u64)t[k] ^ x;
    } break;
    default: {
      unsigned long long t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
      const u64 x = dt == DT_I64 ? 0x8000000000000000ull : 0;
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) f[k] = (u64)t[k] ^ x;
    } break;
  }
}

// make_state value of every row of the batch as 8-byte slot bits.
template <bool FULL>
__device__ __forceinline__ void ab_slot_values(int ty, int dt, const void* p, i64 base, u32 lim, u64 (&v)[AB_ROWS]) {
  switch (dt) {
    case DT_F64: { unsigned long long t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) v[k] = t[k]; } break;
    case DT_F32: { float t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) v[k] = d2u((double)t[k]); } break;
    case DT_I64: case DT_U64: { unsigned long long t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) v[k] = ty == ST_F64 ? d2u(dt == DT_I64 ? (double)(long long)t[k] : (double)t[k]) : t[k]; } break;
    case DT_I32: { int t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) v[k] = ty == ST_F64 ? d2u((double)t[k]) : (u64)(i64)t[k]; } break;
    case DT_U32: { unsigned int t[AB_ROWS]; ab_load_col<FULL>(p, base, lim, t);
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k) v[k] = ty == ST_F64 ? d2u((double)t[k]) : (u64)t[k]; } break;
    default: {   // 8/16-bit integer value columns: rare, per-row generic path
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k)
        v[k] = (FULL || (u32)(k * AB_THREADS) < lim) ? load_slot_value(SRC_COL, ty, dt, p, base + k * AB_THREADS) : 0;
    } break;
  }
}

// One batch (AB_ROWS rows per thread, row k*AB_THREADS + tid).  KW = 0:
// keys of <= 32 bits compared as u32; 1/2: one/two 64-bit words.
__device__ __forceinline__ bool ab_is_count(const SlotDesc& sd, int s) {
  return sd.src[s] == SRC_ONE && sd.op[s] == OP_ADD && sd.type[s] == ST_I64;
}

template <int KW, int NT, bool FULL>
__device__ __forceinline__ u32 ab_batch(const KeyDesc& kd, const SlotDesc& sd, const TinyTable& tt, i64 row_abs,
                                        u32 lim, u64* __restrict__ sacc_t, u32* __restrict__ missbits_out,
                                        u32 (&cnt)[NT]) {
  u64 kl[AB_ROWS], kh[AB_ROWS];
#pragma unroll
  for (int k = 0; k < AB_ROWS; ++k) { kl[k] = 0; kh[k] = 0; }
  for (int col = 0; col < kd.ncols; ++col) {
    u64 f[AB_ROWS];
    ab_key_field<FULL>(kd.dtype[col], kd.ptr[col], row_abs, lim, f);
    const int s = kd.shift[col], wdt = kd.width[col];
#pragma unroll
    for (int k = 0; k < AB_ROWS; ++k) {
      if (KW == 0) {
        kl[k] = (u32)kl[k] | ((u32)f[k] << s);
      } else if (s < 64) {
        kl[k] |= f[k] << s;
        if (KW == 2 && s > 0 && s + wdt > 64) kh[k] |= f[k] >> (64 - s);
      } else if (KW == 2) {
        kh[k] |= f[k] << (s - 64);
      }
    }
  }
  // probe: table row, or NT (the trash cell) for misses and rows past the end
  u32 hoff[AB_ROWS];
  u32 missbits = 0;
  u64 pc = 0;   // per-table-row 8-bit hit counters (COUNT slots)
#pragma unroll
  for (int k = 0; k < AB_ROWS; ++k) {
    u32 hk = NT;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      bool eq;
      if (KW == 0) eq = (u32)kl[k] == (u32)tt.lo[j];
      else eq = key_eq<KW == 2 ? 2 : 1>(kh[k], kl[k], tt.hi[j], tt.lo[j]);
      hk = eq ? (u32)j : hk;
    }
    const bool valid = FULL || (u32)(k * AB_THREADS) < lim;
    if (!valid) hk = NT;
    if (valid && hk == (u32)NT) missbits |= 1u << k;
    if (hk < (u32)NT) pc += 1ull << (8 * hk);
    hoff[k] = hk * (AB_THREADS * 8);
  }
  const int S = sd.nslots;
  // clean batch: every row valid and resident -> branch-free accumulation
  const bool clean = FULL && missbits == 0;
#pragma unroll
  for (int j = 0; j < NT; ++j) cnt[j] += (u32)(pc >> (8 * j)) & 0xFFu;   // COUNT slots: registers
#define AB_LOOP(STMT)                                                      \
  if (clean) {                                                             \
    _Pragma("unroll") for (int k = 0; k < AB_ROWS; ++k) {                  \
      u64* a = (u64*)(acc + hoff[k]);                                      \
      STMT;                                                                \
    }                                                                      \
  } else {                                                                 \
    _Pragma("unroll") for (int k = 0; k < AB_ROWS; ++k) {                  \
      if (hoff[k] < (u32)(NT * AB_THREADS * 8)) {                          \
        u64* a = (u64*)(acc + hoff[k]);                                    \
        STMT;                                                              \
      }                                                                    \
    }                                                                      \
  }
  int cell = 0;
  for (int s = 0; s < S; ++s) {
    const int op = sd.op[s], ty = sd.type[s];
    if (ab_is_count(sd, s)) continue;
    char* acc = (char*)(sacc_t + (size_t)(cell++) * NT * AB_THREADS);
    if (sd.src[s] == SRC_ONE) {
      {
        const u64 one = ty == ST_F64 ? 0x3FF0000000000000ull : 1ull;
        AB_LOOP(*a = combine_slot(op, ty, *a, one))
      }
      continue;
    }
    u64 v[AB_ROWS];
    ab_slot_values<FULL>(ty, sd.dtype[s], sd.ptr[s], row_abs, lim, v);
    if (op == OP_ADD) {
      if (ty == ST_F64) AB_LOOP(*a = d2u(u2d(*a) + u2d(v[k])))
      else AB_LOOP(*a = *a + v[k])
    } else if (ty == ST_F64) {
      if (op == OP_MIN) AB_LOOP(*a = combine_slot(OP_MIN, ST_F64, *a, v[k]))
      else AB_LOOP(*a = combine_slot(OP_MAX, ST_F64, *a, v[k]))
    } else {
      if (op == OP_MIN) AB_LOOP(*a = combine_slot(OP_MIN, ST_I64, *a, v[k]))
      else AB_LOOP(*a = combine_slot(OP_MAX, ST_I64, *a, v[k]))
    }
  }
#undef AB_LOOP
  *missbits_out = missbits;
  return missbits;
}

template <int KW, int NT>
__global__ void __launch_bounds__(AB_THREADS, 3) k_absorb_tiny(KeyDesc kd, SlotDesc sd, i64 row0, u32 n,
                                                           TinyTable tt, u32 rows_per_cta,
                                                           u64* __restrict__ partials, u32* __restrict__ miss_buf,
                                                           u32* __restrict__ miss_cnt) {
  // Per-thread accumulators sacc[c][j][tid] for every non-COUNT slot c
  // (COUNT slots are per-thread register counters): the address of (cell
  // slot c, table row j) for thread tid is ((c*NT + j) * AB_THREADS + tid) * 8
  // bytes, so a warp's 32 accesses hit 32 consecutive 8-byte words whatever
  // rows its lanes matched (conflict-free), and the cost per row does not
  // grow with NT.  Batches in which every row is resident accumulate
  // branch-free; the few others skip misses with a predicate.  Keeping the
  // shared-memory footprint small leaves L1 for in-flight global loads
  // (measured: 70 -> 56 KB per CTA took the kernel from 4.8 to 5.9 TB/s).
  extern __shared__ __align__(16) u64 sacc[];
  __shared__ u32 sw[8];
  __shared__ u32 scnt[AB_THREADS / 32][NT];
  const int S = sd.nslots;
  const int tid = threadIdx.x;
  const u32 c = blockIdx.x;
  const u32 r0 = c * rows_per_cta;
  const u32 r1 = min(r0 + rows_per_cta, n);
  {
    int cell = 0;
    for (int s = 0; s < S; ++s) {
      if (ab_is_count(sd, s)) continue;
      for (int j = 0; j < NT; ++j) sacc[(cell * NT + j) * AB_THREADS + tid] = identity_slot(sd.op[s], sd.type[s]);
      ++cell;
    }
  }
  u32 cnt[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) cnt[j] = 0;

  u32 nmiss = 0;
  for (u32 base = r0; base < r1; base += AB_THREADS * AB_ROWS) {
    const u32 row_t = base + tid;                       // this thread's first row of the batch
    const u32 lim = r1 > row_t ? r1 - row_t : 0;        // rows k*AB_THREADS < lim are valid
    u32 missbits;
    if (base + AB_THREADS * AB_ROWS <= r1)
      ab_batch<KW, NT, true>(kd, sd, tt, row0 + row_t, lim, sacc + tid, &missbits, cnt);
    else
      ab_batch<KW, NT, false>(kd, sd, tt, row0 + row_t, lim, sacc + tid, &missbits, cnt);
    // ordered miss compaction (row order = (k, tid) within this step)
    if (__syncthreads_or(missbits != 0)) {
      for (int k = 0; k < AB_ROWS; ++k) {
        u32 f = (missbits >> k) & 1u;
        u32 tot;
        u32 pre = block_excl_scan256(f, sw, &tot);
        if (f) miss_buf[(size_t)c * rows_per_cta + nmiss + pre] = base + k * AB_THREADS + tid;
        nmiss += tot;
      }
    }
  }
  __syncthreads();
  // COUNT totals: warp sums, then across warps
  const int lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    u32 x = cnt[j];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) scnt[w][j] = x;
  }
  __syncthreads();
  if (tid < NT) {
    u64 x = 0;
    for (int ww = 0; ww < AB_THREADS / 32; ++ww) x += scnt[ww][tid];
    for (int s = 0; s < S; ++s)
      if (ab_is_count(sd, s)) partials[((size_t)c * NT + tid) * S + s] = x;
  }
  // block reduction of the per-thread accumulators: one warp per (cell slot, row)
  int ncell = 0;
  for (int s = 0; s < S; ++s) ncell += ab_is_count(sd, s) ? 0 : 1;
  for (int q = w; q < ncell * NT; q += AB_THREADS / 32) {
    const int ci = q / NT, j = q % NT;
    int s = 0;
    for (int cc = -1;; ++s) { if (!ab_is_count(sd, s)) ++cc; if (cc == ci) break; }
    const int op = sd.op[s], ty = sd.type[s];
    const u64* row = sacc + (size_t)(ci * NT + j) * AB_THREADS;
    u64 x = row[lane];
    for (int i = lane + 32; i < AB_THREADS; i += 32) x = combine_slot(op, ty, x, row[i]);
    for (int o = 16; o; o >>= 1) x = combine_slot(op, ty, x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) partials[((size_t)c * NT + j) * S + s] = x;
  }
  if (tid == 0) miss_cnt[c] = nmiss;
}

bool absorb_supported(int nt, int nslots) { return nt >= 1 && nt <= 8 && (nt + 1) * nslots <= AB_MAX_CELLS; }

void absorb_geometry(u32 n, int num_sms, u32* grid, u32* rows_per_cta) {
  const u32 step = AB_THREADS * AB_ROWS;
  u32 max_grid = (u32)num_sms * 3;
  u32 rpc = (n + max_grid - 1) / max_grid;
  rpc = ((rpc + step - 1) / step) * step;
  if (rpc == 0) rpc = step;
  *rows_per_cta = rpc;
  *grid = (n + rpc - 1) / rpc;
  if (*grid == 0) *grid = 1;
}

template <int KW, int NT>
static void absorb_launch(const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, const TinyTable& tt, u32 grid,
                          u32 rpc, u64* partials, u32* miss_buf, u32* miss_cnt, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  int ncell = 0;
  for (int s = 0; s < sd.nslots; ++s) ncell += (sd.src[s] == SRC_ONE && sd.op[s] == OP_ADD && sd.type[s] == ST_I64) ? 0 : 1;
  const size_t smem = (size_t)std::max(ncell, 1) * NT * AB_THREADS * 8;
  if (first_on_device(attr))
    cudaFuncSetAttribute(k_absorb_tiny<KW, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         AB_MAX_CELLS * AB_THREADS * 8);
  klaunch(k_absorb_tiny<KW, NT>, grid, AB_THREADS, smem, st, kd, sd, row0, n, tt, rpc, partials, miss_buf, miss_cnt);
}

template <int KW>
static void absorb_dispatch(int nt, const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, const TinyTable& tt,
                            u32 grid, u32 rpc, u64* partials, u32* miss_buf, u32* miss_cnt, cudaStream_t st) {
#define AB_CASE(N) case N: absorb_launch<KW, N>(kd, sd, row0, n, tt, grid, rpc, partials, miss_buf, miss_cnt, st); break;
  switch (nt) {
    AB_CASE(1) AB_CASE(2) AB_CASE(3) AB_CASE(4) AB_CASE(5) AB_CASE(6) AB_CASE(7) AB_CASE(8)
    default: break;
  }
#undef AB_CASE
}

void absorb_tiny(int KW, int nt, const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, const TinyTable& tt,
                 u32 grid, u32 rows_per_cta, u64* partials, u32* miss_buf, u32* miss_cnt, cudaStream_t st) {
  if (KW == 1 && kd.total_bits <= 32) {   // narrow keys: 32-bit compares
    absorb_dispatch<0>(nt, kd, sd, row0, n, tt, grid, rows_per_cta, partials, miss_buf, miss_cnt, st);
    return;
  }
  if (KW == 2) absorb_dispatch<2>(nt, kd, sd, row0, n, tt, grid, rows_per_cta, partials, miss_buf, miss_cnt, st);
  else absorb_dispatch<1>(nt, kd, sd, row0, n, tt, grid, rows_per_cta, partials, miss_buf, miss_cnt, st);
}

// ============================================================= probe ====
// First chunk of an execute (T empty, <= PR_THREADS * PR_RPT rows): find the
// distinct keys (OrderedIndex.insert_or_aggregate inserting into an empty
// index, memindex.py:197-236): every warp dedupes its rows with
// warp-synchronous rounds, then warp 0 dedupes the per-warp lists.  If there are at most max_nt of them no flush can
// happen before the chunk ends (max_nt <= M), and a table holding exactly
// these keys from the start is equivalent (every row of the chunk hits it):
// the kernel writes the sorted keys into T with identity states and
// publishes them to mapped host memory for the absorb kernel, which then
// aggregates the chunk's rows with the rest.  Otherwise it only reports
// failure and the host runs the general sort path on the chunk.  out (mapped, u64 words):
// [0] = nt or ~0 on failure, [8 + j] = lo, [16 + j] = hi of sorted row j.
#define PR_THREADS 1024
#define PR_RPT 4
// Distinct keys of `nrow` candidates held by the 32 lanes (row bits in
// `pending`, keys selectable by index): warp-synchronous rounds, each picks
// the first pending candidate, broadcasts its key and clears every equal
// one.  Appends to (tlo, thi)[*cnt ..]; returns false past `cap` keys.
template <int KW, int R>
__device__ __forceinline__ bool warp_distinct(const u64 (&klo)[R], const u64 (&khi)[R], u32 pending, u32 cap,
                                              u64* tlo, u64* thi, u32* cnt) {
  const u32 full = 0xffffffffu;
  const u32 lane = threadIdx.x & 31;
  for (;;) {
    const u32 ball = __ballot_sync(full, pending != 0);
    if (!ball) return true;
    if (*cnt == cap) return false;
    const int src = __ffs(ball) - 1;
    const int kk = __ffs(__shfl_sync(full, pending, src)) - 1;
    u64 blo = 0, bhi = 0;
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (k == kk) { blo = klo[k]; bhi = khi[k]; }
    blo = __shfl_sync(full, blo, src);
    bhi = __shfl_sync(full, bhi, src);
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (((pending >> k) & 1u) && key_eq<KW>(khi[k], klo[k], bhi, blo)) pending &= ~(1u << k);
    if (lane == 0) { tlo[*cnt] = blo; thi[*cnt] = bhi; }
    __syncwarp();
    ++*cnt;
  }
}

template <int KW>
__global__ void __launch_bounds__(PR_THREADS) k_probe_tiny(KeyDesc kd, SlotDesc sd, i64 row0, u32 n, u32 max_nt,
                                                         u64* __restrict__ T_lo, u64* __restrict__ T_hi,
                                                         u64* __restrict__ T_st, u64* out) {
  constexpr int NW = PR_THREADS / 32;
  __shared__ u64 wlo[NW][8], whi[NW][8];
  __shared__ u32 wn[NW];
  __shared__ u64 tlo[8], thi[8];
  const u32 tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  u64 klo[PR_RPT], khi[PR_RPT];
  u32 pending = 0;
#pragma unroll
  for (int k = 0; k < PR_RPT; ++k) {
    const u32 q = k * PR_THREADS + tid;
    klo[k] = khi[k] = 0;
    if (q < n) {
      load_key(kd, row0 + q, khi[k], klo[k]);
      pending |= 1u << k;
    }
  }
  // 1. every warp: the distinct keys of its rows (at most max_nt)
  u32 cnt = 0;
  const bool fits = warp_distinct<KW, PR_RPT>(klo, khi, pending, max_nt, wlo[w], whi[w], &cnt);
  if (lane == 0) wn[w] = fits ? cnt : 0xFFFFFFFFu;
  __syncthreads();
  if (w != 0) return;
  // 2. warp 0: the distinct keys over every warp's list
  const u32 mine = wn[lane < NW ? lane : 0];
  const bool over = __any_sync(0xffffffffu, lane < NW && mine == 0xFFFFFFFFu);
  u32 nt = 0;
  bool ok = !over;
  if (ok) {
    u64 clo[8], chi[8];
    u32 cp = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      clo[j] = chi[j] = 0;
      if (lane < NW && (u32)j < mine) { clo[j] = wlo[lane][j]; chi[j] = whi[lane][j]; cp |= 1u << j; }
    }
    ok = warp_distinct<KW, 8>(clo, chi, cp, max_nt, tlo, thi, &nt);
  }
  if (!ok) {
    if (lane == 0) *(volatile u64*)out = ~0ull;
    return;
  }
  // table row -> its sorted position; states start at the identity (the
  // absorb pass that follows covers these rows too)
  if (lane < nt) {
    u32 r = 0;
    for (u32 j = 0; j < nt; ++j) r += key_less<KW>(thi[j], tlo[j], thi[lane], tlo[lane]) ? 1u : 0u;
    T_lo[r] = tlo[lane];
    if (KW == 2) T_hi[r] = thi[lane];
    ((volatile u64*)out)[8 + r] = tlo[lane];
    ((volatile u64*)out)[16 + r] = thi[lane];
  }
  const int S = sd.nslots;
  for (int i = lane; i < (int)nt * S; i += 32) T_st[i] = identity_slot(sd.op[i % S], sd.type[i % S]);
  if (lane == 0) *(volatile u64*)out = nt;
}

u32 probe_rows() { return PR_THREADS * PR_RPT; }

void probe_tiny(int KW, const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, u32 max_nt, u64* T_lo,
                u64* T_hi, u64* T_st, u64* out_mapped, cudaStream_t st) {
  if (KW == 2) klaunch(k_probe_tiny<2>, 1, PR_THREADS, 0, st, kd, sd, (i64)row0, n, max_nt, T_lo, T_hi, T_st, out_mapped);
  else klaunch(k_probe_tiny<1>, 1, PR_THREADS, 0, st, kd, sd, (i64)row0, n, max_nt, T_lo, T_hi, T_st, out_mapped);
}

}  // namespace isa
