// Tiny-table absorb kernel (early aggregation against a register-resident index).
#include "isa_kernels.h"

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
#define AB_MAX_CELLS 48   // nt * S accumulators per thread (shared memory)

enum { CLS_ADD_I = 0, CLS_ADD_F = 1, CLS_MIN_I = 2, CLS_MAX_I = 3, CLS_MIN_F = 4, CLS_MAX_F = 5 };

template <int NT, typename T, typename F>
__device__ __forceinline__ void ab_reduce_rows(const u32 (&hit)[AB_ROWS], const u64 (&v)[AB_ROWS], T ident, F f,
                                               T (&t)[NT]) {
#pragma unroll
  for (int j = 0; j < NT; ++j) t[j] = ident;
#pragma unroll
  for (int k = 0; k < AB_ROWS; ++k) {
    const T x = *reinterpret_cast<const T*>(&v[k]);
#pragma unroll
    for (int j = 0; j < NT; ++j)
      if (hit[k] == (u32)j) t[j] = f(t[j], x);
  }
}

template <int KW, int NT>
__global__ void __launch_bounds__(AB_THREADS) k_absorb_tiny(KeyDesc kd, SlotDesc sd, i64 row0, u32 n,
                                                           TinyTable tt, u32 rows_per_cta,
                                                           u64* __restrict__ partials, u32* __restrict__ miss_buf,
                                                           u32* __restrict__ miss_cnt) {
  extern __shared__ __align__(16) u64 sacc[];   // [S][NT][AB_THREADS]
  __shared__ u32 sw[8];
  const int S = sd.nslots;
  const int tid = threadIdx.x;
  const u32 c = blockIdx.x;
  const u32 r0 = c * rows_per_cta;
  const u32 r1 = min(r0 + rows_per_cta, n);
  int cls[ISA_MAX_SLOTS];
  for (int s = 0; s < S; ++s) {
    const int op = sd.op[s], ty = sd.type[s];
    cls[s] = op == OP_ADD ? (ty == ST_F64 ? CLS_ADD_F : CLS_ADD_I)
                          : (op == OP_MIN ? (ty == ST_F64 ? CLS_MIN_F : CLS_MIN_I) : (ty == ST_F64 ? CLS_MAX_F : CLS_MAX_I));
    for (int j = 0; j < NT; ++j) sacc[(s * NT + j) * AB_THREADS + tid] = identity_slot(op, ty);
  }

  u32 nmiss = 0;
  for (u32 base = r0; base < r1; base += AB_THREADS * AB_ROWS) {
    u32 hit[AB_ROWS];   // table row, NT = miss, 0xFF = past the end
    bool anymiss = false;
#pragma unroll
    for (int k = 0; k < AB_ROWS; ++k) {
      const u32 row = base + k * AB_THREADS + tid;
      hit[k] = 0xFFu;
      if (row < r1) {
        u64 h, l;
        load_key(kd, row0 + row, h, l);
        u32 hk = NT;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          if (key_eq<KW>(h, l, tt.hi[j], tt.lo[j])) hk = j;
        hit[k] = hk;
        anymiss |= (hk == NT);
      }
    }
    for (int s = 0; s < S; ++s) {
      const int src = sd.src[s], ty = sd.type[s], dt = sd.dtype[s];
      const void* p = sd.ptr[s];
      u64 v[AB_ROWS];
#pragma unroll
      for (int k = 0; k < AB_ROWS; ++k)
        v[k] = (hit[k] < (u32)NT) ? load_slot_value(src, ty, dt, p, row0 + base + k * AB_THREADS + tid) : 0;
      u64* acc = sacc + (size_t)s * NT * AB_THREADS + tid;
      switch (cls[s]) {
        case CLS_ADD_F: {
          double t[NT];
          ab_reduce_rows<NT>(hit, v, 0.0, [](double a, double b) { return a + b; }, t);
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[j * AB_THREADS] = d2u(u2d(acc[j * AB_THREADS]) + t[j]);
        } break;
        case CLS_ADD_I: {
          long long t[NT];
          ab_reduce_rows<NT>(hit, v, 0ll, [](long long a, long long b) { return (long long)((u64)a + (u64)b); }, t);
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[j * AB_THREADS] = acc[j * AB_THREADS] + (u64)t[j];
        } break;
        case CLS_MIN_I: {
          long long t[NT];
          ab_reduce_rows<NT>(hit, v, 0x7FFFFFFFFFFFFFFFll, [](long long a, long long b) { return a <= b ? a : b; }, t);
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[j * AB_THREADS] = combine_slot(OP_MIN, ST_I64, acc[j * AB_THREADS], (u64)t[j]);
        } break;
        case CLS_MAX_I: {
          long long t[NT];
          ab_reduce_rows<NT>(hit, v, (long long)0x8000000000000000ull, [](long long a, long long b) { return a >= b ? a : b; }, t);
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[j * AB_THREADS] = combine_slot(OP_MAX, ST_I64, acc[j * AB_THREADS], (u64)t[j]);
        } break;
        case CLS_MIN_F: {
          double t[NT];
          ab_reduce_rows<NT>(hit, v, __longlong_as_double(0x7FF0000000000000ll), [](double a, double b) { return a <= b ? a : b; }, t);
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[j * AB_THREADS] = combine_slot(OP_MIN, ST_F64, acc[j * AB_THREADS], d2u(t[j]));
        } break;
        default: {
          double t[NT];
          ab_reduce_rows<NT>(hit, v, __longlong_as_double((long long)0xFFF0000000000000ull), [](double a, double b) { return a >= b ? a : b; }, t);
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[j * AB_THREADS] = combine_slot(OP_MAX, ST_F64, acc[j * AB_THREADS], d2u(t[j]));
        } break;
      }
    }
    // ordered miss compaction (row order = (k, tid) within this step)
    if (__syncthreads_or(anymiss)) {
      for (int k = 0; k < AB_ROWS; ++k) {
        u32 f = (hit[k] == (u32)NT) ? 1u : 0u;
        u32 tot;
        u32 pre = block_excl_scan256(f, sw, &tot);
        if (f) miss_buf[(size_t)c * rows_per_cta + nmiss + pre] = base + k * AB_THREADS + tid;
        nmiss += tot;
      }
    }
  }
  __syncthreads();
  // block reduction of the per-thread accumulators: one warp per cell
  const int lane = tid & 31, w = tid >> 5;
  for (int q = w; q < S * NT; q += AB_THREADS / 32) {
    const int s = q / NT, j = q % NT;
    const int op = sd.op[s], ty = sd.type[s];
    const u64* row = sacc + (size_t)q * AB_THREADS;
    u64 x = row[lane];
    for (int i = lane + 32; i < AB_THREADS; i += 32) x = combine_slot(op, ty, x, row[i]);
    for (int o = 16; o; o >>= 1) x = combine_slot(op, ty, x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) partials[((size_t)c * NT + j) * S + s] = x;
  }
  if (tid == 0) miss_cnt[c] = nmiss;
}

bool absorb_supported(int nt, int nslots) { return nt >= 1 && nt <= 8 && nt * nslots <= AB_MAX_CELLS; }

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
  static bool attr = false;
  const size_t smem = (size_t)sd.nslots * NT * AB_THREADS * 8;
  if (!attr) {
    cudaFuncSetAttribute(k_absorb_tiny<KW, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         AB_MAX_CELLS * AB_THREADS * 8);
    attr = true;
  }
  k_absorb_tiny<KW, NT><<<grid, AB_THREADS, smem, st>>>(kd, sd, row0, n, tt, rpc, partials, miss_buf, miss_cnt);
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
  if (KW == 2) absorb_dispatch<2>(nt, kd, sd, row0, n, tt, grid, rows_per_cta, partials, miss_buf, miss_cnt, st);
  else absorb_dispatch<1>(nt, kd, sd, row0, n, tt, grid, rows_per_cta, partials, miss_buf, miss_cnt, st);
}

}  // namespace isa
