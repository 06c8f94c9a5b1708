// sm_100a kernels of the B200 sort-based aggregation operator.
//
// Every kernel here is HBM-bound integer/byte work (sort, scan, segmented
// reduce, merge): no tensor cores.  Design rules followed: coalesced global
// access, shared-memory staging of tiles, warp-synchronous ranking with
// match.any, grids sized from the SM count for streaming kernels.
#include <type_traits>
#include "isa_kernels.h"
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <stdexcept>
#include <vector>

namespace isa {

std::atomic<long long> g_launches{0};

// ------------------------------------------------------- kernel timer ---
namespace {
struct KtRec { int fam; cudaEvent_t a, b; int64_t bytes; };
struct KTimer {
  bool on = false;
  std::vector<KtRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t open[KF_COUNT] = {};
  double ms[KF_COUNT] = {};
  int64_t launches[KF_COUNT] = {}, bytes[KF_COUNT] = {};
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
thread_local KTimer g_kt;
}  // namespace

bool kt_enabled() { return g_kt.on; }
void kt_set(bool on) { g_kt.on = on; }
void kt_reserve(int64_t events) {   // create the timing events ahead of a timed region
  while ((int64_t)g_kt.pool.size() < events) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    g_kt.pool.push_back(e);
  }
}
void kt_begin(int fam, cudaStream_t st) {
  if (!g_kt.on) return;
  cudaEvent_t e = g_kt.get();
  cudaEventRecord(e, st);
  g_kt.open[fam] = e;
}
void kt_end(int fam, int64_t alg_bytes, cudaStream_t st) {
  if (!g_kt.on || !g_kt.open[fam]) return;
  cudaEvent_t e = g_kt.get();
  cudaEventRecord(e, st);
  g_kt.recs.push_back({fam, g_kt.open[fam], e, alg_bytes});
  g_kt.open[fam] = nullptr;
}
void kt_add_bytes(int fam, int64_t alg_bytes) {
  if (!g_kt.on) return;
  for (size_t i = g_kt.recs.size(); i-- > 0;)
    if (g_kt.recs[i].fam == fam) { g_kt.recs[i].bytes += alg_bytes; return; }
}
void kt_collect(double* ms, int64_t* launches, int64_t* bytes) {
  for (auto& r : g_kt.recs) {
    float t = 0;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
      g_kt.ms[r.fam] += t;
      g_kt.launches[r.fam] += 1;
      g_kt.bytes[r.fam] += r.bytes;
    }
    g_kt.pool.push_back(r.a);
    g_kt.pool.push_back(r.b);
  }
  g_kt.recs.clear();
  for (int f = 0; f < KF_COUNT; ++f) {
    if (ms) ms[f] = g_kt.ms[f];
    if (launches) launches[f] = g_kt.launches[f];
    if (bytes) bytes[f] = g_kt.bytes[f];
    g_kt.ms[f] = 0;
    g_kt.launches[f] = 0;
    g_kt.bytes[f] = 0;
  }
}

// ============================================================== scan ====
#define SC_THREADS 256
#define SC_ITEMS 16
#define SC_TILE (SC_THREADS * SC_ITEMS)

__global__ void __launch_bounds__(SC_THREADS) k_scan_reduce(const u32* __restrict__ d, u32 n, u32* __restrict__ bsum) {
  __shared__ u32 sw[8];
  u32 base = blockIdx.x * SC_TILE;
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    u32 idx = base + i * SC_THREADS + threadIdx.x;
    if (idx < n) s += d[idx];
  }
  u32 tot;
  block_excl_scan256(s, sw, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_single(u32* __restrict__ bsum, u32 nb, u32* __restrict__ total,
                                                           bool write_total_slot) {
  __shared__ u32 sw[8];
  u32 carry = 0;
  for (u32 base = 0; base < nb; base += SC_TILE) {
    u32 v[SC_ITEMS];
    u32 s = 0;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
      u32 idx = base + threadIdx.x * SC_ITEMS + i;
      v[i] = idx < nb ? bsum[idx] : 0;
      s += v[i];
    }
    u32 tot;
    u32 pre = block_excl_scan256(s, sw, &tot) + carry;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
      u32 idx = base + threadIdx.x * SC_ITEMS + i;
      if (idx < nb) bsum[idx] = pre;
      pre += v[i];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    if (write_total_slot) bsum[nb] = carry;
    if (total) *total = carry;
  }
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_apply(u32* __restrict__ d, u32 n, const u32* __restrict__ bsum) {
  __shared__ u32 sw[8];
  __shared__ u32 tile[SC_TILE];
  u32 base = blockIdx.x * SC_TILE;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    u32 idx = base + i * SC_THREADS + threadIdx.x;
    tile[i * SC_THREADS + threadIdx.x] = idx < n ? d[idx] : 0;
  }
  __syncthreads();
  u32 v[SC_ITEMS];
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) { v[i] = tile[threadIdx.x * SC_ITEMS + i]; s += v[i]; }
  u32 tot;
  u32 pre = block_excl_scan256(s, sw, &tot) + bsum[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) { tile[threadIdx.x * SC_ITEMS + i] = pre; pre += v[i]; }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    u32 idx = base + i * SC_THREADS + threadIdx.x;
    if (idx < n) d[idx] = tile[i * SC_THREADS + threadIdx.x];
  }
}

size_t scan_tmp_words(u32 n) { return (size_t)(n + SC_TILE - 1) / SC_TILE + 2; }

void scan_exclusive_u32(u32* data, u32 n, u32* tmp, u32* total, cudaStream_t st) {
  u32 nb = (n + SC_TILE - 1) / SC_TILE;
  if (n == 0) {
    if (total) cudaMemsetAsync(total, 0, sizeof(u32), st);
    return;
  }
  if (n <= 16 * SC_TILE) {   // small: one CTA scans in place (1 launch instead of 3)
    klaunch(k_scan_single, 1, SC_THREADS, 0, st, data, n, total, false);
    return;
  }
  klaunch(k_scan_reduce, nb, SC_THREADS, 0, st, data, n, tmp);
  klaunch(k_scan_single, 1, SC_THREADS, 0, st, tmp, nb, total, true);
  klaunch(k_scan_apply, nb, SC_THREADS, 0, st, data, n, tmp);
}

// ======================================================== radix sort ====
#define RS_THREADS 256   // x 16 rows per thread (512 x 8 measured no faster: config 5 scatter 113 = 113 ms, config 3
                         // 81 -> 89, config 4 54 -> 67)
#ifndef RS_PK_THREADS
#define RS_PK_THREADS 512   // packed passes: 512 x 16 rows per tile
#endif
#define RS_ITEMS 16
#define RS_TILE (RS_THREADS * RS_ITEMS)
#define RS_WARPS (RS_THREADS / 32)
#define RS_WARP_ITEMS (RS_TILE / RS_WARPS)
// Packed passes (one 8-byte word per row) run 512-thread tiles of 8,192 rows
// at 2 CTAs/SM -- the same 32 warps/SM as 4 tiles of 4,096, but the per-tile
// work (digit scan, publish, look-back: a third of the pass's instructions)
// is paid half as often; the other passes' tiles (12-20 bytes of shared
// memory per row) stay at 256 threads.
__host__ __device__ constexpr int rs_threads(int PK) { return (PK >= 1 && PK <= 3) ? RS_PK_THREADS : RS_THREADS; }
__host__ __device__ constexpr int rs_min_ctas(int KW, int PK) {
  return (PK >= 1 && PK <= 3) ? (RS_PK_THREADS == 512 ? 2 : 4) : (KW == 2 ? 2 : 3);
}
__host__ __device__ constexpr int rs_tile(int PK) { return rs_threads(PK) * RS_ITEMS; }

__device__ __forceinline__ u32 digit_of(u64 hi, u64 lo, int shift) {
  u64 v;
  if (shift >= 64) v = hi >> (shift - 64);
  else if (shift > 56) v = (lo >> shift) | (hi << (64 - shift));
  else v = lo >> shift;
  return (u32)(v & 0xFFu);
}

// peers & (lanes whose digit bit `m` equals mine): the bit test feeds the
// ballot as a predicate and the same predicate selects the replicated mask,
// so the select folds into one LOP3 (4 instructions per bit instead of 6)
__device__ __forceinline__ u32 ballot_same_bit(u32 peers, u32 d, u32 m) {
  u32 r;
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t, rep;\n\t"
      "and.b32 t, %2, %3;\n\t"
      "setp.ne.u32 p, t, 0;\n\t"
      "vote.sync.ballot.b32 t, p, 0xffffffff;\n\t"
      "selp.b32 rep, 0xffffffff, 0, p;\n\t"
      "xor.b32 t, t, rep;\n\t"
      "not.b32 t, t;\n\t"
      "and.b32 %0, %1, t;\n\t}"
      : "=r"(r) : "r"(peers), "r"(d), "r"(m));
  return r;
}

// one key word: no cross-word digit (the hot loops of k_rs_scatter)
template <int KW>
__device__ __forceinline__ u32 digit_kw(u64 hi, u64 lo, int shift) {
  if (KW == 1) return (u32)(lo >> shift) & 0xFFu;
  return digit_of(hi, lo, shift);
}

#ifndef RS_WUNROLL
#define RS_WUNROLL 16   // write-out loop unroll (shared-memory loads in flight per thread; 4: -1 to -3% sort)
#endif
static constexpr int kRsWriteUnroll = RS_WUNROLL;
#ifndef RS_LB
#define RS_LB 4   // look-back window (predecessor status words per round trip)
#endif
__device__ __forceinline__ u64 ld_relaxed_gpu(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One LSD pass over 8 bits.  Single tile (status == nullptr): the in-tile
// digit scan is the global offset.  Otherwise onesweep: tiles are taken in
// order from a counter, every tile publishes its per-digit count and looks
// back over its predecessors (decoupled look-back) for the exclusive prefix;
// the digit's global start comes from the all-pass histogram (ghist).
// Status word per (tile, digit): count | flag << 32 (1 aggregate, 2
// inclusive prefix) | epoch << 34; words of other passes carry another epoch
// and read as "not published yet", so the array is never cleared.
//
// Packed mode (PK > 0, KW == 1 only; the caller guarantees that key bits
// outside [pk_lo, pk_lo + 32) are the same in every key): a pass moves one
// 8-byte word per row, (key bits [pk_lo, +32) << 32) | row id, instead of
// 8 + 4 bytes.  PK 1 packs on the way in (and records the constant key bits
// in *pk_const), PK 2 moves packed words, PK 3 unpacks on the way out to
// the usual (key, row id) columns.  `shift` is then the digit's position
// in the packed word.
//
// Carried values (PK 4 / 5, with plain PK 0 passes over the packed words in
// between): the payload column holds a 4-byte value per row instead of the
// row id, which sits in the packed word's low half.  PK 4 packs like PK 1
// (row ids 0..n-1) and takes the payload from v_in = the values in row order;
// PK 5 unpacks like PK 3 and also writes the payload, now in sorted order, to
// carry_out -- the collapse then reads every row's value at its sorted
// position instead of gathering it by row id.
template <int KW, bool BALLOT, int PK = 0>
__global__ void __launch_bounds__(rs_threads(PK), rs_min_ctas(KW, PK)) k_rs_scatter(const u64* __restrict__ lo_in, const u64* __restrict__ hi_in,
                                                         const u32* __restrict__ v_in, u64* __restrict__ lo_out,
                                                         u64* __restrict__ hi_out, u32* __restrict__ v_out, u32 n,
                                                         int shift, u64* __restrict__ status,
                                                         const u32* __restrict__ ghist, u32* __restrict__ tile_ctr,
                                                         u32 epoch, int pk_lo, u64* __restrict__ pk_const,
                                                         int lb_sleep, u32* __restrict__ carry_out) {
  static_assert(PK == 0 || KW == 1, "packed passes carry one key word");
  constexpr bool HASV = PK == 0 || PK >= 4;   // a payload column moves with the key words
  constexpr int THREADS = rs_threads(PK), ITEMS = RS_ITEMS, TILE = THREADS * ITEMS, WARPS = THREADS / 32,
                WARP_ITEMS = TILE / WARPS;
  extern __shared__ __align__(16) unsigned char smem[];
  u32* wcnt = (u32*)smem;               // [WARPS][256]
  u32* dstart = wcnt + WARPS * 256;  // [256]
  u32* gbase = dstart + 256;            // [256]
  u32* sw = gbase + 256;                // [WARPS]
  u64* s_lo = (u64*)(sw + WARPS);    // [TILE]
  u64* s_hi = s_lo + TILE;           // [TILE] (KW == 2)
  u32* s_v = (u32*)(s_lo + KW * TILE);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (status && tid == 0) sw[0] = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const u32 tile = status ? sw[0] : blockIdx.x, base = tile * TILE;
  const u32 tile_n = min((u32)TILE, n - base);
  for (int i = tid; i < WARPS * 256; i += THREADS) wcnt[i] = 0;
  __syncthreads();

  u64 lo[ITEMS], hi[ITEMS];
  u32 v[ITEMS], off[ITEMS];
  const u32 lt = lanemask_lt();
  // load + rank; full tiles (all but the last) drop every bounds test
  auto load_rank = [&](auto full_tag) {
  constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    u32 li = w * WARP_ITEMS + it * 32 + lane;
    const bool valid = FULL || li < tile_n;
    u32 gi = base + li;
    lo[it] = valid ? lo_in[gi] : 0;
    hi[it] = (KW == 2 && valid) ? hi_in[gi] : 0;
    v[it] = ((PK <= 1 || PK >= 4) && valid) ? ((PK == 1 && !v_in) ? gi : v_in[gi]) : 0;   // PK 1, null v_in: row ids 0..n-1
    if (PK == 1 || PK == 4) {
      if (gi == 0 && valid) *pk_const = lo[it] & ~(0xFFFFFFFFull << pk_lo);
      lo[it] = (((lo[it] >> pk_lo) & 0xFFFFFFFFull) << 32) | (PK == 4 ? gi : v[it]);
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    u32 li = w * WARP_ITEMS + it * 32 + lane;
    const bool valid = FULL || li < tile_n;
    u32 d = valid ? digit_kw<KW>(hi[it], lo[it], shift) : 256 + lane;
    // lanes holding the same digit: MATCH.ANY, or (BALLOT: chosen by the
    // host for large passes whose digits are not skewed) eight independent
    // ballots -- data-independent cost, measured faster on uniform digits
    u32 peers;
    if (!BALLOT) {
      peers = __match_any_sync(0xffffffffu, d);
    } else {
      peers = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int b = 0; b < 8; ++b) peers = ballot_same_bit(peers, d, 1u << b);
      if (!FULL && !valid) peers = 1u << lane;
    }
    int leader = __ffs(peers) - 1;
    u32 cnt = 0;
    if (valid && lane == leader) {
      cnt = wcnt[w * 256 + d];
      wcnt[w * 256 + d] = cnt + __popc(peers);
    }
    cnt = __shfl_sync(0xffffffffu, cnt, leader);
    off[it] = (cnt + __popc(peers & lt)) | (d << 16);   // digit kept for the staging loop
    __syncwarp();
  }
  };
  if (tile_n == TILE) load_rank(std::true_type{});
  else load_rank(std::false_type{});
  __syncthreads();
  // per-digit exclusive prefix over warps, then over digits; the tile's
  // aggregate is published now, but the look-back for its exclusive prefix
  // waits until the rows are staged, so predecessors have had that long to
  // publish (fewer spinning reloads)
  const int dg = tid;  // threads 0..255 own one digit each
  const bool isd = dg < 256;
  u32 run = 0, ds, gs = 0;
  {
    if (isd) {
#pragma unroll
      for (int ww = 0; ww < WARPS; ++ww) {
        u32 c = wcnt[ww * 256 + dg];
        wcnt[ww * 256 + dg] = run;
        run += c;
      }
    }
    u32 tot;
    ds = block_excl_scan_nw<WARPS>(run, sw, &tot);
    if (isd) dstart[dg] = ds;
    if (status) {
      gs = block_excl_scan_nw<WARPS>(isd ? ghist[dg] : 0u, sw, &tot);   // global start of digit dg
      const u64 E = (u64)epoch << 34;
      if (isd) st_relaxed_gpu(status + (size_t)tile * 256 + dg, E | ((tile == 0 ? 2ull : 1ull) << 32) | run);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    u32 li = w * WARP_ITEMS + it * 32 + lane;
    if (li < tile_n) {
      const u32 d = off[it] >> 16;
      u32 p = dstart[d] + wcnt[w * 256 + d] + (off[it] & 0xFFFFu);
      s_lo[p] = lo[it];
      if (KW == 2) s_hi[p] = hi[it];
      if (HASV) s_v[p] = v[it];
    }
  }
  if (!isd) {
    // no digit of its own
  } else if (!status) {
    gbase[dg] = 0u;   // one tile: in-tile offsets are global
  } else {
    const u64 E = (u64)epoch << 34;
    u32 excl = 0;
    if (tile != 0) {
      // look back RS_LB predecessors per round trip
      int j = (int)tile - 1;
      bool done = false;
      while (!done) {
        u64 x[RS_LB];
#pragma unroll
        for (int i = 0; i < RS_LB; ++i)
          x[i] = j - i >= 0 ? ld_relaxed_gpu(status + (size_t)(j - i) * 256 + dg) : (E | (2ull << 32));
#pragma unroll
        for (int i = 0; i < RS_LB; ++i) {
          if ((x[i] >> 34) != (u64)epoch) {   // not published yet: reload from tile j
            if (lb_sleep) __nanosleep(lb_sleep);
            break;
          }
          excl += (u32)x[i];
          --j;
          if (((x[i] >> 32) & 3u) == 2u) { done = true; break; }
        }
      }
      st_relaxed_gpu(status + (size_t)tile * 256 + dg, E | (2ull << 32) | (excl + run));
    }
    gbase[dg] = gs + excl - ds;
  }
  const u64 kc = (PK == 3 || PK == 5) ? *pk_const : 0;
  __syncthreads();
#pragma unroll kRsWriteUnroll
  for (int it = 0; it < ITEMS; ++it) {
    u32 p = it * THREADS + tid;
    if (p < tile_n) {
      u64 l = s_lo[p];
      u64 h = KW == 2 ? s_hi[p] : 0;
      u32 d = digit_kw<KW>(h, l, shift);
      u32 dst = gbase[d] + p;
      if (PK == 3 || PK == 5) {
        lo_out[dst] = kc | ((l >> 32) << pk_lo);
        v_out[dst] = (u32)l;
        if (PK == 5) carry_out[dst] = s_v[p];
      } else {
        lo_out[dst] = l;
        if (KW == 2) hi_out[dst] = h;
        if (HASV) v_out[dst] = s_v[p];
      }
    }
  }
}

// Histograms of every pass's digit in one read of the keys (onesweep
// upsweep): ghist[p][d] += count of digit d at bits [bit_lo + 8p, +8).
#define RS_MAX_PASS 16
template <int KW>
__global__ void __launch_bounds__(256) k_rs_hist_all(const u64* __restrict__ klo, const u64* __restrict__ khi, u32 n,
                                                     int bit_lo, int npass, u32* __restrict__ ghist) {
  __shared__ u32 h[RS_MAX_PASS * 256];
  for (int i = threadIdx.x; i < npass * 256; i += 256) h[i] = 0;
  __syncthreads();
  for (u32 i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
    const u64 lo = klo[i], hi = KW == 2 ? khi[i] : 0;
    for (int p = 0; p < npass; ++p) atomicAdd(&h[p * 256 + digit_kw<KW>(hi, lo, bit_lo + 8 * p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += 256)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
}

// ---------------------------------------------------------------------------
// Hybrid sort for wide keys: LSD passes over the top 16 bits of the sort
// field only (two onesweep passes), then every run of equal top-16 bits (a
// "bucket", ~n / 65536 rows for spread keys) is finished inside one CTA's
// shared memory -- an LSD sort of the bucket rows over the field bits that
// vary inside the CTA's range, keys read through a u16 row index.  Replaces
// npass - 2 global passes (config 3's 64-bit keys: 8 -> 2 + 1 local) with
// one read + write.  Stable: every pass is stable and the top-16 passes keep
// equal keys in input order.  A bucket larger than a CTA's capacity
// (clustered keys) sets *overflow; the caller then finishes with the plain
// LSD passes from the top-16-sorted array (stable from any stable order).
#define RL_THREADS 256
#define RL_WARPS (RL_THREADS / 32)
// rows one CTA sorts (template CAP: 4096 or 1024, ISA_RL_CAP); nominal rows
// per CTA = CAP / 2 (ranges snap to bucket starts)

// top-16 bucket of row i: field bits [bit_hi - 16, bit_hi) of the 128-bit key
// (packed words: key bits [pk_lo, pk_lo + 32) sit in word bits 32..63)
template <int KW, int PKIN>
__device__ __forceinline__ u32 rl_top(const u64* __restrict__ lo, const u64* __restrict__ hi, u32 i, int bit_hi,
                                      int pk_lo) {
  if (PKIN) return (u32)(lo[i] >> (32 + bit_hi - 16 - pk_lo)) & 0xFFFFu;
  const u64 h = KW == 2 ? hi[i] : 0, l = lo[i];
  const int sft = bit_hi - 16;
  u64 v;
  if (sft >= 64) v = h >> (sft - 64);
  else if (sft == 0) v = l;
  else v = (l >> sft) | (sft > 48 ? (h << (64 - sft)) : 0ull);
  return (u32)v & 0xFFFFu;
}

// CTA range starts: bnd[c] = first row of the bucket holding row c * RL_SPAN
template <int KW, int PKIN>
__global__ void k_rs_bounds(const u64* __restrict__ lo, const u64* __restrict__ hi, u32 n, u32 nctas, int bit_hi,
                            int pk_lo, u32* __restrict__ bnd, u32* __restrict__ overflow, u32 RL_SPAN) {
  const u32 c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nctas) return;
  if (c == 0) { bnd[0] = 0; return; }
  if (c == nctas) { bnd[c] = n; return; }
  const u32 x = c * RL_SPAN;
  const u32 t = rl_top<KW, PKIN>(lo, hi, x, bit_hi, pk_lo);
  u32 l = x > RL_SPAN ? x - RL_SPAN : 0, h = x;   // smallest j in [l, x] with top(j) == t
  if (l > 0 && rl_top<KW, PKIN>(lo, hi, l, bit_hi, pk_lo) == t) atomicExch(overflow, 1u);   // bucket > RL_SPAN
  while (l < h) {
    const u32 m = (l + h) >> 1;
    if (rl_top<KW, PKIN>(lo, hi, m, bit_hi, pk_lo) < t) l = m + 1; else h = m;
  }
  bnd[c] = l;
}

template <int KW, int PKIN, int RL_CAP>
__global__ void __launch_bounds__(RL_THREADS, RL_CAP <= 1024 ? 6 : 2) k_rs_local(const u64* __restrict__ lo_in, const u64* __restrict__ hi_in,
                                                             const u32* __restrict__ v_in, u64* __restrict__ lo_out,
                                                             u64* __restrict__ hi_out, u32* __restrict__ v_out,
                                                             const u32* __restrict__ bnd, int bit_lo, int bit_hi,
                                                             int pk_lo, const u64* __restrict__ pk_const,
                                                             u32* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  u64* k_lo = (u64*)smem;                         // [RL_CAP]
  u64* k_hi = k_lo + RL_CAP;                      // [RL_CAP] (KW == 2)
  u32* vv = (u32*)(k_lo + (size_t)KW * RL_CAP);   // [RL_CAP]
  unsigned short* o0 = (unsigned short*)(vv + RL_CAP);
  unsigned short* o1 = o0 + RL_CAP;
  u32* scratch = (u32*)(o1 + RL_CAP);             // [RL_CAP] (digit, rank) per row
  u32* wcnt = scratch + RL_CAP;                   // [RL_WARPS][256]
  u32* dstart = wcnt + RL_WARPS * 256;            // [256]
  __shared__ u32 sw[RL_WARPS];
  __shared__ u64 s_or_lo[RL_WARPS], s_or_hi[RL_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const u32 r0 = bnd[blockIdx.x], r1 = bnd[blockIdx.x + 1];
  if (r1 <= r0) return;
  const u32 n = r1 - r0;
  if (n > RL_CAP) {   // a bucket too large for one CTA: the caller falls back
    if (tid == 0) atomicExch(overflow, 1u);
    return;
  }
  const u64 kc = PKIN ? *pk_const : 0;
  // load (coalesced); packed words unpack here
  u64 orl = 0, orh = 0;
  for (u32 i = tid; i < n; i += RL_THREADS) {
    u64 l, h = 0;
    u32 v;
    if (PKIN) {
      const u64 wd = lo_in[r0 + i];
      l = kc | ((wd >> 32) << pk_lo);
      v = (u32)wd;
    } else {
      l = lo_in[r0 + i];
      if (KW == 2) h = hi_in[r0 + i];
      v = v_in[r0 + i];
    }
    k_lo[i] = l;
    if (KW == 2) k_hi[i] = h;
    vv[i] = v;
    o0[i] = (unsigned short)i;
  }
  __syncthreads();
  // field bits that vary inside the range (relative to its first row)
  {
    const u64 f_lo = k_lo[0], f_hi = KW == 2 ? k_hi[0] : 0;
    for (u32 i = tid; i < n; i += RL_THREADS) {
      orl |= k_lo[i] ^ f_lo;
      if (KW == 2) orh |= k_hi[i] ^ f_hi;
    }
    for (int o = 16; o; o >>= 1) {
      orl |= __shfl_xor_sync(0xffffffffu, orl, o);
      orh |= __shfl_xor_sync(0xffffffffu, orh, o);
    }
    if (lane == 0) { s_or_lo[w] = orl; s_or_hi[w] = orh; }
    __syncthreads();
    orl = 0; orh = 0;
    for (int q = 0; q < RL_WARPS; ++q) { orl |= s_or_lo[q]; orh |= s_or_hi[q]; }
  }
  // highest varying bit below bit_hi
  int msb = -1;
  {
    u64 mh = orh, ml = orl;
    if (bit_hi < 128) {
      if (bit_hi >= 64) mh &= bit_hi == 64 ? 0ull : ((1ull << (bit_hi - 64)) - 1);
      else { mh = 0; ml &= (1ull << bit_hi) - 1; }
    }
    if (mh) msb = 127 - __clzll((long long)mh);
    else if (ml) msb = 63 - __clzll((long long)ml);
  }
  const int npass = msb < bit_lo ? 0 : (msb - bit_lo) / 8 + 1;
  // LSD passes over [bit_lo, bit_lo + 8 npass): warp-contiguous rows in order
  const u32 WI = (((n + RL_WARPS - 1) / RL_WARPS) + 31) & ~31u;
  const u32 lt = lanemask_lt();
  unsigned short* cur = o0;
  unsigned short* nxt = o1;
  for (int p = 0; p < npass; ++p) {
    const int sft = bit_lo + 8 * p;
    for (int q = lane; q < 256; q += 32) wcnt[w * 256 + q] = 0;
    __syncwarp();
    const u32 a0 = w * WI, a1 = min(n, a0 + WI);
    for (u32 i = a0 + lane; i < ((a1 + 31) & ~31u) && a0 < a1; i += 32) {
      const bool valid = i < a1;
      u32 d = 256 + lane;
      if (valid) {
        const u32 x = cur[i];
        d = digit_of(KW == 2 ? k_hi[x] : 0, k_lo[x], sft);
      }
      const u32 peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      u32 c = 0;
      if (valid && lane == leader) {
        c = wcnt[w * 256 + d];
        wcnt[w * 256 + d] = c + __popc(peers);
      }
      c = __shfl_sync(0xffffffffu, c, leader);
      if (valid) scratch[i] = (d << 16) | (c + __popc(peers & lt));
      __syncwarp();
    }
    __syncthreads();
    {
      const int dg = tid;
      u32 run = 0;
#pragma unroll
      for (int ww = 0; ww < RL_WARPS; ++ww) {
        const u32 c = wcnt[ww * 256 + dg];
        wcnt[ww * 256 + dg] = run;
        run += c;
      }
      u32 tot;
      dstart[dg] = block_excl_scan256(run, sw, &tot);
    }
    __syncthreads();
    for (u32 i = a0 + lane; i < a1; i += 32) {
      const u32 v = scratch[i], d = v >> 16;
      nxt[dstart[d] + wcnt[w * 256 + d] + (v & 0xFFFFu)] = cur[i];
    }
    __syncthreads();
    unsigned short* t = cur; cur = nxt; nxt = t;
  }
  // write in sorted order (coalesced)
  for (u32 i = tid; i < n; i += RL_THREADS) {
    const u32 x = cur[i];
    lo_out[r0 + i] = k_lo[x];
    if (KW == 2) hi_out[r0 + i] = k_hi[x];
    v_out[r0 + i] = vv[x];
  }
}

static size_t rl_smem(int KW, int cap) {
  return (size_t)cap * (8 * KW + 4 + 2 + 2 + 4) + (RL_WARPS * 256 + 256) * 4 + 64;
}

static size_t rs_scatter_smem(int KW, bool packed = false) {
  const int threads = packed ? RS_PK_THREADS : RS_THREADS, warps = threads / 32;
  return (warps * 256 + 256 + 256 + warps) * sizeof(u32) + (size_t)threads * RS_ITEMS * (packed ? 8 : 8 * KW + 4);
}

// aux layout: [ghist: RS_MAX_PASS * 256 u32][tile counters: RS_MAX_PASS u32][pad][status: 256 * ntiles u64].
// The status words sit at a fixed offset and are only ever written as
// status words (or zero), so no stale counter can alias a live epoch.
#define RS_AUX_HDR 16640
size_t sort_aux_bytes(u32 n) {
  return RS_AUX_HDR + (size_t)256 * ((n + RS_TILE - 1) / RS_TILE) * 8 + ((size_t)n / 512 + 4) * 4 + 64;
}
static std::atomic<u32> g_rs_epoch{0};

// LSD onesweep passes over [bit_lo, bit_hi).  pack_lo >= 0: pack (key bits
// [pack_lo, pack_lo + 32) << 32 | row id) on the first pass whatever the
// range; pack_lo == -2: never pack; -1: pack when the range fits 32 bits.
// leave_packed: the last pass keeps the packed words (the local sort of the
// hybrid path unpacks them).
static int radix_lsd(int KW, SortBufs& b, u32 n, int bit_lo, int bit_hi, cudaStream_t st, int64_t* launches, int start,
                     int pack_lo, bool leave_packed) {
  int cur = start;
  if (n <= 1 || bit_hi <= bit_lo) return cur;
  static std::atomic<unsigned long long> attr_set[3];
  if (first_on_device(attr_set[KW])) {
    if (KW == 1) {
      const int ps = (int)rs_scatter_smem(1, true);
      cudaFuncSetAttribute(k_rs_scatter<1, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ps);
      cudaFuncSetAttribute(k_rs_scatter<1, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ps);
      cudaFuncSetAttribute(k_rs_scatter<1, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ps);
      cudaFuncSetAttribute(k_rs_scatter<1, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ps);
      cudaFuncSetAttribute(k_rs_scatter<1, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, ps);
      cudaFuncSetAttribute(k_rs_scatter<1, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, ps);
      const int fs = (int)rs_scatter_smem(1);
      cudaFuncSetAttribute(k_rs_scatter<1, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
      cudaFuncSetAttribute(k_rs_scatter<1, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
      cudaFuncSetAttribute(k_rs_scatter<1, false, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
      cudaFuncSetAttribute(k_rs_scatter<1, true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
    }
    if (KW == 2) {
      cudaFuncSetAttribute(k_rs_scatter<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_scatter_smem(2));
      cudaFuncSetAttribute(k_rs_scatter<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_scatter_smem(2));
    } else {
      cudaFuncSetAttribute(k_rs_scatter<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_scatter_smem(1));
      cudaFuncSetAttribute(k_rs_scatter<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_scatter_smem(1));
    }
  }
  const u32 ntiles = (n + RS_TILE - 1) / RS_TILE;
  const u32 pk_tiles = (n + rs_tile(1) - 1) / rs_tile(1);   // packed passes run larger tiles
  const size_t smem = rs_scatter_smem(KW);
  const int npass = (bit_hi - bit_lo + 7) / 8;
  u32* ghist = (u32*)b.aux;
  u32* tctr = ghist + RS_MAX_PASS * 256;
  u64* status = (u64*)((char*)b.aux + RS_AUX_HDR);
  u64* pk_const = (u64*)((char*)b.aux + RS_AUX_HDR - 64);   // header pad, after the tile counters
  // packed passes: one 8-byte word per row when the varying key bits fit 32
  static int pk_env = -1;
  if (pk_env < 0) { const char* e = getenv("ISA_PACKED"); pk_env = e && e[0] == '0' ? 0 : 1; }
  const bool packed = pack_lo >= 0 ? true
                                   : (pack_lo == -1 && pk_env && KW == 1 && b.pack_ok && ntiles > 1 && npass >= 2 &&
                                      bit_hi - bit_lo <= 32);
  const int pk_lo = pack_lo >= 0 ? pack_lo : bit_lo;
  // values carried through the sort as the payload (see k_rs_scatter, PK 4 / 5): opt-in (ISA_CARRY=1, read
  // per sort) -- measured on config 5 at 4e9 rows the collapse without the gather saves 19 ms and the
  // 12-byte passes at 3 CTAs/SM cost 24 ms (sort 154 -> 177 ms, collapse 98 -> 80 ms)
  const char* ce = getenv("ISA_CARRY");
  const int carry_env = ce && ce[0] == '1' ? 1 : 0;
  const bool carry = carry_env && packed && pack_lo == -1 && !leave_packed && b.val_iota && b.carry_in && b.carry_out &&
                     npass >= 2;
  b.carried = carry;
  const size_t psmem = rs_scatter_smem(1, true);
  static int lb_sleep = -1;   // look-back back-off (ns) while a predecessor has not published
  if (lb_sleep < 0) { const char* e = getenv("ISA_LB_SLEEP"); lb_sleep = e ? atoi(e) : 0; }
  const bool hist_ready = b.hist_npass == npass && b.hist_bit_lo == bit_lo && start == 0;
  b.hist_npass = 0;   // consumed (a second sort on these buffers counts for itself)
  if (ntiles > 1) {
    if (npass > RS_MAX_PASS) throw std::runtime_error("radix sort: too many passes");
    if (hist_ready) {
      // counted by the key-building pass: only the tile counters are reset
      cudaMemsetAsync(tctr, 0, RS_MAX_PASS * 4, st);
    } else {
      cudaMemsetAsync(ghist, 0, (RS_MAX_PASS * 256 + RS_MAX_PASS) * 4, st);
      const u32 g = std::min<u32>(ntiles, 148u * 8u);
      kt_begin(KF_HIST, st);
      if (KW == 2) klaunch(k_rs_hist_all<2>, g, 256, 0, st, b.lo[cur], b.hi[cur], n, bit_lo, npass, ghist);
      else klaunch(k_rs_hist_all<1>, g, 256, 0, st, b.lo[cur], (const u64*)nullptr, n, bit_lo, npass, ghist);
      kt_end(KF_HIST, (int64_t)n * 8 * KW, st);
    }
  }
  // ranking per pass: ballots for large passes without heavy digits (one
  // small read-back of the histograms; MATCH.ANY otherwise)
  bool ballot[RS_MAX_PASS] = {};
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("ISA_RANK");
    mode = !e ? -1 : (e[0] == 'm' ? 0 : (e[0] == 'b' ? 1 : -1));
  }
  if (mode >= 0) {
    for (int p = 0; p < npass; ++p) ballot[p] = mode == 1 && ntiles > 1;
  }
  const bool hinted = mode >= 0 || (b.hint && b.hint[0] >= 0 && b.hint_bit_lo == bit_lo && b.hint_npass == npass);
  if (hinted) {
    if (mode < 0)
      for (int p = 0; p < npass; ++p) ballot[p] = b.hint[p] != 0;
  } else if (ntiles >= 64 && b.map_dev) {
    // through mapped host memory by a kernel: a copy-engine read would queue
    // behind the spill copies on the D2H engine
    read_words(b.map_dev, ghist, (u32)npass * 256, st);
    cudaStreamSynchronize(st);
    const volatile u32* hh = b.map_host;
    for (int p = 0; p < npass; ++p) {
      u32 mx = 0;
      for (int d = 0; d < 256; ++d) mx = std::max(mx, (u32)hh[(size_t)p * 256 + d]);
      ballot[p] = (u64)mx * 32 <= (u64)n;   // no digit holds more than 1/32 of the keys
    }
    if (b.hint) {   // later sorts of the same kind reuse the choice (no read-back)
      for (int p = 0; p < npass; ++p) b.hint[p] = ballot[p] ? 1 : 0;
      b.hint_bit_lo = bit_lo;
      b.hint_npass = npass;
    }
  }
  for (int p = 0; p < npass; ++p) {
    const int shift = bit_lo + 8 * p;
    const int nxt = cur ^ 1;
    const bool one = ntiles == 1;
    u64* stt = one ? nullptr : status;
    const u32* gh = one ? nullptr : ghist + p * 256;
    u32* tc = one ? nullptr : tctr + p;
    const u32 ep = one ? 0u : ((g_rs_epoch.fetch_add(1) % 0x3FFFFFFEu) + 1u);
#define RS_GO(K, BL, HI_IN, HI_OUT)                                                                          \
  klaunch(k_rs_scatter<K, BL>, ntiles, RS_THREADS, smem, st, b.lo[cur], HI_IN, b.val[cur], b.lo[nxt], HI_OUT, \
          b.val[nxt], n, shift, stt, gh, tc, ep, 0, (u64*)nullptr, lb_sleep, (u32*)nullptr)
#define RS_PK(PK)                                                                                            \
  do {                                                                                                       \
    if (ballot[p])                                                                                           \
      klaunch(k_rs_scatter<1, true, PK>, pk_tiles, RS_PK_THREADS, psmem, st, b.lo[cur], (const u64*)nullptr, \
              b.val[cur], b.lo[nxt], (u64*)nullptr, b.val[nxt], n, 32 + shift - pk_lo, stt, gh, tc, ep, pk_lo,   \
              pk_const, lb_sleep, (u32*)nullptr);                                                                      \
    else                                                                                                     \
      klaunch(k_rs_scatter<1, false, PK>, pk_tiles, RS_PK_THREADS, psmem, st, b.lo[cur], (const u64*)nullptr, \
              b.val[cur], b.lo[nxt], (u64*)nullptr, b.val[nxt], n, 32 + shift - pk_lo, stt, gh, tc, ep, pk_lo,   \
              pk_const, lb_sleep, (u32*)nullptr);                                                                      \
  } while (0)
    // algorithmic bytes of the pass: every row's key words + row id read and written once
    // (packed passes: 8-byte words in the middle, 12 -> 8 / 8 -> 12 at the ends)
    const int64_t pass_bytes =
        (int64_t)n * (carry ? (p == npass - 1 ? 28 : 24)
                            : packed ? (p == 0 || (p == npass - 1 && !leave_packed) ? 20 : 16) : 2 * (8 * KW + 4));
    kt_begin(KF_SCATTER, st);
    if (carry) {
      // (packed word, value) pairs: PK 4 in, plain passes over the word's key half, PK 5 out
      const int wshift = 32 + shift - pk_lo;
      const u32* vin = p == 0 ? b.carry_in : b.val[cur];
#define RS_CARRY(BL, PKM)                                                                                       \
  klaunch(k_rs_scatter<1, BL, PKM>, ntiles, RS_THREADS, smem, st, b.lo[cur], (const u64*)nullptr, vin, b.lo[nxt], \
          (u64*)nullptr, b.val[nxt], n, wshift, stt, gh, tc, ep, pk_lo, pk_const, lb_sleep, b.carry_out)
      if (p == 0) { if (ballot[p]) RS_CARRY(true, 4); else RS_CARRY(false, 4); }
      else if (p == npass - 1) { if (ballot[p]) RS_CARRY(true, 5); else RS_CARRY(false, 5); }
      else { if (ballot[p]) RS_CARRY(true, 0); else RS_CARRY(false, 0); }
#undef RS_CARRY
    } else if (packed) {
      if (p == 0 && b.val_iota) {   // row ids 0..n-1: the pass numbers the rows itself (no row-id read)
        if (ballot[p])
          klaunch(k_rs_scatter<1, true, 1>, pk_tiles, RS_PK_THREADS, psmem, st, b.lo[cur], (const u64*)nullptr,
                  (const u32*)nullptr, b.lo[nxt], (u64*)nullptr, b.val[nxt], n, 32 + shift - pk_lo, stt, gh, tc, ep, pk_lo,
                  pk_const, lb_sleep, (u32*)nullptr);
        else
          klaunch(k_rs_scatter<1, false, 1>, pk_tiles, RS_PK_THREADS, psmem, st, b.lo[cur], (const u64*)nullptr,
                  (const u32*)nullptr, b.lo[nxt], (u64*)nullptr, b.val[nxt], n, 32 + shift - pk_lo, stt, gh, tc, ep, pk_lo,
                  pk_const, lb_sleep, (u32*)nullptr);
      } else if (p == 0) RS_PK(1);
      else if (p == npass - 1 && !leave_packed) RS_PK(3);
      else RS_PK(2);
    } else if (KW == 2) {
      if (ballot[p]) RS_GO(2, true, b.hi[cur], b.hi[nxt]);
      else RS_GO(2, false, b.hi[cur], b.hi[nxt]);
    } else {
      if (ballot[p]) RS_GO(1, true, (const u64*)nullptr, (u64*)nullptr);
      else RS_GO(1, false, (const u64*)nullptr, (u64*)nullptr);
    }
    kt_end(KF_SCATTER, pass_bytes, st);
#undef RS_GO
#undef RS_PK
    if (launches) *launches += 1;
    cur = nxt;
  }
  return cur;
}

// unpack packed words (key bits << 32 | row id) into key / row-id columns
__global__ void k_rs_unpack(const u64* __restrict__ w, u32 n, int pk_lo, const u64* __restrict__ pk_const,
                            u64* __restrict__ lo, u32* __restrict__ val) {
  const u64 kc = *pk_const;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 x = w[i];
    lo[i] = kc | ((x >> 32) << pk_lo);
    val[i] = (u32)x;
  }
}

int radix_sort_pairs(int KW, SortBufs& b, u32 n, int bit_lo, int bit_hi, cudaStream_t st, int64_t* launches,
                     int start) {
  // opt-in (ISA_HYBRID=1, read per sort): measured slower than plain
  // onesweep LSD (config 5 sort 42 -> 58 ms, config 3 92 -> 143 ms per 1e9
  // rows, profiles/r2_ab_hybrid.txt)
  const char* he = getenv("ISA_HYBRID");
  const int hyb_env = he && he[0] == '1' ? 1 : 0;
  const int npass = (bit_hi - bit_lo + 7) / 8;
  if (!(hyb_env && b.map_dev && npass >= 3 && n >= (1u << 16) && n <= 0x7FFFFFFFu))
    return radix_lsd(KW, b, n, bit_lo, bit_hi, st, launches, start, -1, false);
  const char* ce = getenv("ISA_RL_CAP");
  const int cap_env = ce && atoi(ce) <= 1024 ? 1024 : 4096;
  const u32 RL_CAP = (u32)cap_env, RL_SPAN = RL_CAP / 2;
  static std::atomic<unsigned long long> attr_set[3];
  if (first_on_device(attr_set[KW])) {
    const int s4 = (int)rl_smem(KW, 4096), s1 = (int)rl_smem(KW, 1024);
    if (KW == 2) {
      cudaFuncSetAttribute(k_rs_local<2, 0, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, s4);
      cudaFuncSetAttribute(k_rs_local<2, 0, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
    } else {
      cudaFuncSetAttribute(k_rs_local<1, 0, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, s4);
      cudaFuncSetAttribute(k_rs_local<1, 1, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, s4);
      cudaFuncSetAttribute(k_rs_local<1, 0, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
      cudaFuncSetAttribute(k_rs_local<1, 1, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
    }
  }
  static int pk_env = -1;
  if (pk_env < 0) { const char* e = getenv("ISA_PACKED"); pk_env = e && e[0] == '0' ? 0 : 1; }
  const bool packed = pk_env && KW == 1 && b.pack_ok && bit_hi - bit_lo <= 32;
  // 1. the top 16 bits of the field
  int cur = radix_lsd(KW, b, n, bit_hi - 16, bit_hi, st, launches, start, packed ? bit_lo : -2, packed);
  const int nxt = cur ^ 1;
  u64* pk_const = (u64*)((char*)b.aux + RS_AUX_HDR - 64);
  u32* overflow = (u32*)((char*)b.aux + RS_AUX_HDR - 32);
  const u32 ntiles = (n + RS_TILE - 1) / RS_TILE;
  u32* bnd = (u32*)((char*)b.aux + RS_AUX_HDR + (size_t)256 * ntiles * 8);
  const u32 nctas = (n + RL_SPAN - 1) / RL_SPAN;
  cudaMemsetAsync(overflow, 0, sizeof(u32), st);
  // 2. CTA ranges snapped to bucket starts, 3. local sort of every range
  kt_begin(KF_SCATTER, st);
  const int bg = (int)((nctas + 256) / 256);
  if (KW == 2) klaunch(k_rs_bounds<2, 0>, bg, 256, 0, st, b.lo[cur], b.hi[cur], n, nctas, bit_hi, bit_lo, bnd, overflow, RL_SPAN);
  else if (packed) klaunch(k_rs_bounds<1, 1>, bg, 256, 0, st, b.lo[cur], (const u64*)nullptr, n, nctas, bit_hi, bit_lo, bnd, overflow, RL_SPAN);
  else klaunch(k_rs_bounds<1, 0>, bg, 256, 0, st, b.lo[cur], (const u64*)nullptr, n, nctas, bit_hi, bit_lo, bnd, overflow, RL_SPAN);
  const size_t sm = rl_smem(KW, RL_CAP);
#define RL_GO(K, P, C, HI_IN, HI_OUT)                                                                             \
  klaunch(k_rs_local<K, P, C>, nctas, RL_THREADS, sm, st, b.lo[cur], HI_IN, b.val[cur], b.lo[nxt], HI_OUT, b.val[nxt], \
          bnd, bit_lo, bit_hi, bit_lo, pk_const, overflow)
#define RL_CAPS(K, P, HI_IN, HI_OUT) \
  { if (RL_CAP == 1024) RL_GO(K, P, 1024, HI_IN, HI_OUT); else RL_GO(K, P, 4096, HI_IN, HI_OUT); }
  if (KW == 2) RL_CAPS(2, 0, b.hi[cur], b.hi[nxt])
  else if (packed) RL_CAPS(1, 1, (const u64*)nullptr, (u64*)nullptr)
  else RL_CAPS(1, 0, (const u64*)nullptr, (u64*)nullptr)
#undef RL_CAPS
#undef RL_GO
  kt_end(KF_SCATTER, (int64_t)n * (packed ? 20 : 2 * (8 * KW + 4)), st);
  if (launches) *launches += 3;
  // 4. a bucket too large for a CTA: plain LSD over every bit from the
  //    top-16-sorted rows (stable from any stable order)
  read_words(b.map_dev + 16 * 256 - 1, overflow, 1, st);
  cudaStreamSynchronize(st);
  if (((const volatile u32*)b.map_host)[16 * 256 - 1] == 0) return nxt;
  if (packed) {
    klaunch(k_rs_unpack, (int)std::min<u32>((n + 255) / 256, 148u * 16u), 256, 0, st, (const u64*)b.lo[cur], n, bit_lo, (const u64*)pk_const, b.lo[nxt],
            b.val[nxt]);
    cur = nxt;
  }
  return radix_lsd(KW, b, n, bit_lo, bit_hi, st, launches, cur, -2, false);
}

static int grid_for(u64 n, int threads, int cap = 148 * 16);

// 128-bit keys sorted on the high word only: finish every run of equal
// high words (usually exact duplicates or rare collisions) with a stable
// insertion sort on the low word.  A run longer than maxlen sets *too_long
// (the caller then completes the sort with full LSD passes).
__global__ void k_sort_small_segments(u64* __restrict__ lo, u64* __restrict__ hi, u32* __restrict__ val, u32 n,
                                      u32 maxlen, int shift, u32* __restrict__ too_long) {
  // shift > 0: the rows were sorted on hi >> shift only; a run = equal
  // hi >> shift, ordered by (hi, lo)
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 h = hi[i] >> shift;
    if (i > 0 && (hi[i - 1] >> shift) == h) continue;   // not the first element of a run
    u32 j = i + 1;
    while (j < n && (hi[j] >> shift) == h) {
      ++j;
      if (j - i > maxlen) break;
    }
    if (j - i > maxlen) { *too_long = 1u; continue; }
    for (u32 a = i + 1; a < j; ++a) {
      const u64 kl = lo[a], kh = hi[a];
      const u32 kv = val[a];
      u32 p = a;
      while (p > i && (hi[p - 1] > kh || (hi[p - 1] == kh && lo[p - 1] > kl))) {
        lo[p] = lo[p - 1];
        if (shift) hi[p] = hi[p - 1];
        val[p] = val[p - 1];
        --p;
      }
      lo[p] = kl;
      if (shift) hi[p] = kh;
      val[p] = kv;
    }
  }
}

void sort_small_segments(u64* lo, u64* hi, u32* val, u32 n, u32 maxlen, int shift, u32* too_long, cudaStream_t st) {
  if (n) klaunch(k_sort_small_segments, grid_for(n, 256), 256, 0, st, lo, hi, val, n, maxlen, shift, too_long);
}

// one-word keys sorted on their top bits only: is the full key order
// non-decreasing?  (*bad_mapped: mapped host word, zeroed by the host, set on
// an inversion -- two distinct keys that share the sorted bits, out of order)
__global__ void __launch_bounds__(256) k_check_sorted(const u64* __restrict__ lo, u32 n, u32* __restrict__ bad_mapped) {
  bool bad = false;
  for (u32 i = blockIdx.x * 256 + threadIdx.x + 1; i < n; i += gridDim.x * 256) bad |= lo[i] < lo[i - 1];
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *bad_mapped = 1u;
}
void check_sorted(const u64* lo, u32 n, u32* bad_mapped, cudaStream_t st) {
  if (n > 1) klaunch(k_check_sorted, grid_for(n, 256), 256, 0, st, lo, n, bad_mapped);
}

// ======================================================= key building ====
template <int KW>
__global__ void k_build_keys(KeyDesc kd, i64 row0, const u32* __restrict__ pos, u32 n, u64* __restrict__ lo,
                             u64* __restrict__ hi, u32* __restrict__ val, u64* __restrict__ varying,
                             u32* __restrict__ ghist, int h_bit_lo, int h_npass) {
  // ghist != nullptr (fast path only): the all-pass digit histograms of the
  // sort that follows (bits [h_bit_lo, h_bit_lo + 8 * h_npass)) are counted
  // here, while the keys are in registers, instead of a pass of their own
  __shared__ u32 hsm[KW == 1 ? RS_MAX_PASS * 256 : 1];
  if (KW == 1 && ghist) {
    for (int i = threadIdx.x; i < h_npass * 256; i += blockDim.x) hsm[i] = 0;
    __syncthreads();
  }
  u64 r_hi, r_lo;
  load_key(kd, row0 + (pos ? pos[0] : 0), r_hi, r_lo);
  u64 acc_lo = 0, acc_hi = 0;
  if (KW == 1 && !pos && kd.ncols == 1 && kd.shift[0] == 0 && (kd.dtype[0] == DT_I64 || kd.dtype[0] == DT_U64)) {
    // one 64-bit key column, rows in order (configs 3 and 5): no per-row
    // dtype dispatch, four independent loads in flight per thread
    const u64* col = (const u64*)kd.ptr[0] + row0;
    const u64 flip = kd.dtype[0] == DT_I64 ? 0x8000000000000000ull : 0ull;
    const u32 stride = gridDim.x * blockDim.x;
    u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * (u64)stride < n; i += 4 * stride) {
      u64 l[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) l[j] = __ldg(col + i + j * stride) ^ flip;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lo[i + j * stride] = l[j];
        val[i + j * stride] = i + j * stride;
        acc_lo |= l[j] ^ r_lo;
        if (ghist)
          for (int p = 0; p < h_npass; ++p) atomicAdd(&hsm[p * 256 + ((u32)(l[j] >> (h_bit_lo + 8 * p)) & 0xFFu)], 1u);
      }
    }
    for (; i < n; i += stride) {
      const u64 l = __ldg(col + i) ^ flip;
      lo[i] = l;
      val[i] = i;
      acc_lo |= l ^ r_lo;
      if (ghist)
        for (int p = 0; p < h_npass; ++p) atomicAdd(&hsm[p * 256 + ((u32)(l >> (h_bit_lo + 8 * p)) & 0xFFu)], 1u);
    }
    if (ghist) {
      __syncthreads();
      for (int q = threadIdx.x; q < h_npass * 256; q += blockDim.x)
        if (hsm[q]) atomicAdd(&ghist[q], hsm[q]);
    }
  } else
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u32 r = pos ? pos[i] : i;
    u64 h, l;
    load_key(kd, row0 + r, h, l);
    lo[i] = l;
    if (KW == 2) hi[i] = h;
    val[i] = r;
    acc_lo |= l ^ r_lo;
    acc_hi |= h ^ r_hi;
  }
  // warp OR-reduce, one atomic per warp
  for (int o = 16; o; o >>= 1) {
    acc_lo |= __shfl_xor_sync(0xffffffffu, acc_lo, o);
    acc_hi |= __shfl_xor_sync(0xffffffffu, acc_hi, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (acc_lo) atomicOr((unsigned long long*)&varying[0], (unsigned long long)acc_lo);
    if (acc_hi) atomicOr((unsigned long long*)&varying[1], (unsigned long long)acc_hi);
  }
}

static int grid_for(u64 n, int threads, int cap) {
  u64 g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > (u64)cap) g = cap;
  return (int)g;
}

// the kernel's fast path (one 64-bit key column in row order): it can count the sort's histograms on the way
bool build_keys_counts_histograms(int KW, const KeyDesc& kd, const u32* pos) {
  return KW == 1 && !pos && kd.ncols == 1 && kd.shift[0] == 0 && (kd.dtype[0] == DT_I64 || kd.dtype[0] == DT_U64);
}
void build_keys(int KW, const KeyDesc& kd, int64_t row0, const u32* pos, u32 n, u64* lo, u64* hi, u32* val,
                u64* varying, cudaStream_t st, u32* ghist, int h_bit_lo, int h_npass) {
  if (n == 0) return;
  int g = grid_for(n, 256);
  if (!build_keys_counts_histograms(KW, kd, pos) || h_npass < 1 || h_npass > RS_MAX_PASS) ghist = nullptr;
  if (KW == 2) klaunch(k_build_keys<2>, g, 256, 0, st, kd, row0, pos, n, lo, hi, val, varying, (u32*)nullptr, 0, 0);
  else klaunch(k_build_keys<1>, g, 256, 0, st, kd, row0, pos, n, lo, hi, val, varying, ghist, h_bit_lo, h_npass);
}
// the histogram area of a sort's aux buffer (zeroed by whoever counts into it)
u32* sort_aux_hist(void* aux) { return (u32*)aux; }
size_t sort_aux_hist_bytes() { return (size_t)RS_MAX_PASS * 256 * 4; }

template <int KW>
__global__ void k_keys_varying(const u64* __restrict__ lo, const u64* __restrict__ hi, u32 n, u64* varying) {
  u64 r_lo = lo[0], r_hi = KW == 2 ? hi[0] : 0;
  u64 acc_lo = 0, acc_hi = 0;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    acc_lo |= lo[i] ^ r_lo;
    if (KW == 2) acc_hi |= hi[i] ^ r_hi;
  }
  for (int o = 16; o; o >>= 1) {
    acc_lo |= __shfl_xor_sync(0xffffffffu, acc_lo, o);
    acc_hi |= __shfl_xor_sync(0xffffffffu, acc_hi, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (acc_lo) atomicOr((unsigned long long*)&varying[0], (unsigned long long)acc_lo);
    if (acc_hi) atomicOr((unsigned long long*)&varying[1], (unsigned long long)acc_hi);
  }
}

void keys_varying(int KW, const u64* lo, const u64* hi, u32 n, u64* varying, cudaStream_t st) {
  if (n == 0) return;
  int g = grid_for(n, 256);
  if (KW == 2) klaunch(k_keys_varying<2>, g, 256, 0, st, lo, hi, n, varying);
  else klaunch(k_keys_varying<1>, g, 256, 0, st, lo, hi, n, varying);
}

// Small device -> host reads through mapped pinned memory: the copy engines
// stay free for bulk spill/readback copies (a 4-byte cudaMemcpyAsync would
// queue behind a 200 MB spill on the same engine).
__global__ void k_read_words(u32* __restrict__ dst_mapped, const u32* __restrict__ src, u32 nwords) {
  for (u32 i = threadIdx.x; i < nwords; i += blockDim.x) dst_mapped[i] = src[i];
}
void read_words(u32* dst_mapped, const u32* src, u32 nwords, cudaStream_t st) {
  klaunch(k_read_words, 1, 64, 0, st, dst_mapped, src, nwords);
}

// wide-merge window keys relative to the window's low bound (fewer varying
// bits, exact pass count without a read-back) + the staged-row payload
template <int KW>
__global__ void k_window_keys(const u64* __restrict__ slo, const u64* __restrict__ shi, u32 m, u64 llo, u64 lhi,
                              u64* __restrict__ dlo, u64* __restrict__ dhi, u32* __restrict__ val) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const u64 l = slo[i];
    dlo[i] = l - llo;
    if (KW == 2) dhi[i] = shi[i] - lhi - (l < llo ? 1ull : 0ull);
    val[i] = i;
  }
}
void window_keys(int KW, const u64* slo, const u64* shi, u32 m, u64 llo, u64 lhi, u64* dlo, u64* dhi, u32* val,
                 cudaStream_t st) {
  if (!m) return;
  const int g = (int)std::min<u32>((m + 255) / 256, 148u * 16u);
  if (KW == 2) klaunch(k_window_keys<2>, g, 256, 0, st, slo, shi, m, llo, lhi, dlo, dhi, val);
  else klaunch(k_window_keys<1>, g, 256, 0, st, slo, (const u64*)nullptr, m, llo, lhi, dlo, (u64*)nullptr, val);
}

__global__ void k_iota(u32* v, u32 n) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}
void iota_u32(u32* v, u32 n, cudaStream_t st) {
  if (n) klaunch(k_iota, grid_for(n, 256), 256, 0, st, v, n);
}

// ==================================================== flush analysis ====
template <int KW>
__global__ void k_new_heads(const u64* __restrict__ lo, const u64* __restrict__ hi, const u32* __restrict__ val,
                            u32 m, const u64* __restrict__ T_lo, const u64* __restrict__ T_hi, u32 t,
                            u32* __restrict__ bitmap, u32* __restrict__ n_new, const u32* __restrict__ firstpos,
                            int invert) {
  // invert (val[] is a permutation of the bitmap's positions): the rows that
  // are NOT first occurrences of a new key set their bit instead -- the few
  // duplicates of a chunk of mostly new keys rather than every row
  u32 cnt = 0;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    u64 l = lo[i], h = KW == 2 ? hi[i] : 0;
    bool head = (i == 0) || !key_eq<KW>(h, l, KW == 2 ? hi[i - 1] : 0, lo[i - 1]);
    bool is_new = head;
    if (head && t) {
      u32 p = lower_bound_key<KW>(T_lo, T_hi, t, h, l);
      is_new = !(p < t && key_eq<KW>(KW == 2 ? T_hi[p] : 0, T_lo[p], h, l));
    }
    if (is_new) ++cnt;
    if (is_new != (invert != 0)) {
      u32 pos = firstpos ? firstpos[val[i]] : val[i];
      atomicOr(&bitmap[pos >> 5], 1u << (pos & 31));
    }
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_new, cnt);
}

// Small chunks (span <= FS_MAX_BITS): the whole flush analysis in one CTA --
// new heads into a shared-memory bitmap, their count, and the k-th set bit
// (the flush row) -- written straight to mapped host memory: out[0] = new
// keys, out[1] = flush row (span when fewer than k).
#define FS_THREADS 1024
#define FS_MAX_BITS 32768
template <int KW>
__global__ void __launch_bounds__(FS_THREADS) k_flush_small(const u64* __restrict__ lo, const u64* __restrict__ hi,
                                                          const u32* __restrict__ val, u32 m,
                                                          const u64* __restrict__ T_lo, const u64* __restrict__ T_hi,
                                                          u32 t, u32 span, u32 k, u32* out) {
  __shared__ u32 bm[FS_MAX_BITS / 32];
  __shared__ u32 sw[FS_THREADS / 32];
  const u32 nw = (span + 31) / 32;
  for (u32 i = threadIdx.x; i < nw; i += FS_THREADS) bm[i] = 0;
  __syncthreads();
  for (u32 i = threadIdx.x; i < m; i += FS_THREADS) {
    const u64 l = lo[i], h = KW == 2 ? hi[i] : 0;
    if (i > 0 && key_eq<KW>(h, l, KW == 2 ? hi[i - 1] : 0, lo[i - 1])) continue;
    bool in_t = false;
    if (t) {
      const u32 p = lower_bound_key<KW>(T_lo, T_hi, t, h, l);
      in_t = p < t && key_eq<KW>(KW == 2 ? T_hi[p] : 0, T_lo[p], h, l);
    }
    if (!in_t) {
      const u32 pos = val[i];
      atomicOr(&bm[pos >> 5], 1u << (pos & 31));
    }
  }
  __syncthreads();
  // words per thread: contiguous ranges so the prefix follows bit order
  const u32 per = (nw + FS_THREADS - 1) / FS_THREADS;
  const u32 w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
  u32 c = 0;
  for (u32 w = w0; w < w1; ++w) c += __popc(bm[w]);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u32 x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sw[wid] = x;
  __syncthreads();
  if (wid == 0) {
    u32 v = sw[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    sw[lane] = v;
  }
  __syncthreads();
  const u32 total = sw[FS_THREADS / 32 - 1];
  u32 pre = (wid ? sw[wid - 1] : 0) + x - c;   // exclusive prefix of this thread's words
  if (threadIdx.x == 0) {
    ((volatile u32*)out)[0] = total;
    if (total < k) ((volatile u32*)out)[1] = span;
  }
  if (k >= 1 && pre < k && pre + c >= k) {
    for (u32 w = w0; w < w1; ++w) {
      const u32 word = bm[w], pc = __popc(word);
      if (pre + pc >= k) {
        u32 need = k - pre, bits = word;
        for (;;) {
          const int b = __ffs(bits) - 1;
          if (--need == 0) { ((volatile u32*)out)[1] = w * 32 + b; break; }
          bits &= bits - 1;
        }
        break;
      }
      pre += pc;
    }
  }
}

bool flush_small_ok(u32 span) { return span <= FS_MAX_BITS; }

void flush_small(int KW, const u64* lo, const u64* hi, const u32* val, u32 m, const u64* T_lo, const u64* T_hi, u32 t,
                 u32 span, u32 k, u32* out_mapped, cudaStream_t st) {
  if (KW == 2) klaunch(k_flush_small<2>, 1, FS_THREADS, 0, st, lo, hi, val, m, T_lo, T_hi, t, span, k, out_mapped);
  else klaunch(k_flush_small<1>, 1, FS_THREADS, 0, st, lo, hi, val, m, T_lo, T_hi, t, span, k, out_mapped);
}

void new_heads(int KW, const u64* lo, const u64* hi, const u32* val, u32 m, const u64* T_lo, const u64* T_hi,
               u32 t, u32* bitmap, u32* n_new, cudaStream_t st, const u32* firstpos, bool invert) {
  if (m == 0) return;
  int g = grid_for(m, 256);
  const int inv = invert ? 1 : 0;
  if (KW == 2) klaunch(k_new_heads<2>, g, 256, 0, st, lo, hi, val, m, T_lo, T_hi, t, bitmap, n_new, firstpos, inv);
  else klaunch(k_new_heads<1>, g, 256, 0, st, lo, hi, val, m, T_lo, T_hi, t, bitmap, n_new, firstpos, inv);
}

// word w of the bitmap as the selection sees it: complemented (bits beyond
// nbits cleared) when the bitmap marks the rows that are not new heads
__device__ __forceinline__ u32 sel_word(const u32* __restrict__ bm, u32 w, u32 nw, u32 nbits, int invert) {
  u32 x = bm[w];
  if (invert) {
    x = ~x;
    if (w == nw - 1 && (nbits & 31)) x &= (1u << (nbits & 31)) - 1;
  }
  return x;
}
__global__ void k_popc_words(const u32* __restrict__ bm, u32 nw, u32 nbits, int invert, u32* __restrict__ cnt) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x)
    cnt[i] = __popc(sel_word(bm, i, nw, nbits, invert));
}
__global__ void k_find_kth(const u32* __restrict__ bm, const u32* __restrict__ pre, u32 nw, u32 nbits, int invert, u32 k,
                           u32* __restrict__ out) {
  for (u32 w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    u32 word = sel_word(bm, w, nw, nbits, invert);
    u32 p = pre[w], c = __popc(word);
    if (p < k && p + c >= k) {
      u32 need = k - p;  // 1-based within word
      for (int b = 0; b < 32; ++b) {
        if (word & (1u << b)) {
          if (--need == 0) { *out = w * 32 + b; break; }
        }
      }
    }
  }
}

void select_kth_bit(const u32* bitmap, u32 nbits, u32 k, u32* word_tmp, u32* scan_tmp, u32* out, cudaStream_t st,
                    bool invert) {
  u32 nw = (nbits + 31) / 32;
  int g = grid_for(nw, 256);
  const int inv = invert ? 1 : 0;
  klaunch(k_popc_words, g, 256, 0, st, bitmap, nw, nbits, inv, word_tmp);
  scan_exclusive_u32(word_tmp, nw, scan_tmp, nullptr, st);
  klaunch(k_find_kth, g, 256, 0, st, bitmap, word_tmp, nw, nbits, inv, k, out);
}

// ====================================================== row records ====
// The chunk's value columns interleaved into one record per row (rows <
// n): the segmented reduce then gathers one record (one sector) per row
// instead of one sector per column.
__global__ void k_row_pack(RowPack rp, i64 row0, u32 n, char* __restrict__ out) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    char* rec = out + (size_t)i * rp.R;
    for (int c = 0; c < rp.nc; ++c) {
      const char* src = (const char*)rp.src[c];
      switch (rp.elem[c]) {
        case 1: *(unsigned char*)(rec + rp.off[c]) = ((const unsigned char*)src)[row0 + i]; break;
        case 2: *(unsigned short*)(rec + rp.off[c]) = ((const unsigned short*)src)[row0 + i]; break;
        case 4: *(unsigned int*)(rec + rp.off[c]) = ((const unsigned int*)src)[row0 + i]; break;
        default: *(u64*)(rec + rp.off[c]) = ((const u64*)src)[row0 + i]; break;
      }
    }
  }
}

void row_pack(const RowPack& rp, int64_t row0, u32 n, char* out, cudaStream_t st) {
  if (n) klaunch(k_row_pack, grid_for(n, 256), 256, 0, st, rp, (i64)row0, n, out);
}

// One int64 value column narrowed to int32 for rows [row0, row0 + n): the
// collapse gathers values by pre-sort row position (random reads), and a
// 4-byte record per row of a fill cycle mostly stays in the 126 MB L2 where
// the 8-byte column does not.  *bad_mapped (mapped host memory, zeroed by the
// host) is set when a value does not fit int32: the caller then keeps the
// column.
__global__ void __launch_bounds__(256) k_narrow_i64(const i64* __restrict__ src, u32 n, int* __restrict__ out,
                                                    u32* __restrict__ bad_mapped) {
  bool bad = false;
  for (u32 i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
    const i64 v = src[i];
    const int x = (int)v;
    out[i] = x;
    bad |= (i64)x != v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *bad_mapped = 1u;
}

void narrow_i64(const void* src, int64_t row0, u32 n, int* out, u32* bad_mapped, cudaStream_t st) {
  if (n) klaunch(k_narrow_i64, grid_for(n, 256), 256, 0, st, (const i64*)src + row0, n, out, bad_mapped);
}

// ========================================================== collapse ====
// Consecutive sorted items per segmented-reduce thread: 4 for states of
// <= 2 slots (measured: config 5's collapse 51 -> 35 ms; more threads keep
// more random gathers in flight), 8 for wider states (config 3's 5 slots:
// 4 was 7% slower).
__host__ __device__ constexpr int cl_items(int MS) { return MS <= 2 ? 4 : 8; }
u32 collapse_threads(u32 m, int S) {
  const u32 c = (u32)cl_items(S <= 1 ? 1 : (S <= 2 ? 2 : (S <= 4 ? 4 : (S <= 5 ? 5 : 8))));
  return (m + c - 1) / c;
}

template <int KW>
__global__ void k_head_flags(const u64* __restrict__ lo, const u64* __restrict__ hi, const u32* __restrict__ val,
                             u32 m, u32 limit, u32* __restrict__ flags) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    bool inc = val[i] < limit;
    bool head = inc && ((i == 0) || !key_eq<KW>(KW == 2 ? hi[i] : 0, lo[i], KW == 2 ? hi[i - 1] : 0, lo[i - 1]));
    flags[i] = head ? 1u : 0u;
  }
}

// ---- collapse with block head counts (default): per 128-thread block of
// the segmented reduce, the included heads are counted (keys + row ids read
// once), the block counts scanned (one tiny kernel), and the reduce kernel
// numbers its groups itself (block base + in-block prefix) -- instead of a
// per-row head-flag array, a 3-kernel scan over it and a per-row read of the
// scanned positions.
#define CB_THREADS 128
template <int KW, int MS>
__global__ void __launch_bounds__(CB_THREADS) k_cl_count(const u64* __restrict__ lo, const u64* __restrict__ hi,
                                                         const u32* __restrict__ val, u32 m, u32 limit,
                                                         u32* __restrict__ counts) {
  constexpr u32 CLI = (u32)cl_items(MS);
  const u32 t = blockIdx.x * CB_THREADS + threadIdx.x;
  const u32 i0 = t * CLI, i1 = min(i0 + CLI, m);
  u32 c = 0;
  if (i0 < m) {
    u64 pl = i0 > 0 ? lo[i0 - 1] : 0, ph = (KW == 2 && i0 > 0) ? hi[i0 - 1] : 0;
    for (u32 i = i0; i < i1; ++i) {
      const u64 l = lo[i], h = KW == 2 ? hi[i] : 0;
      c += (val[i] < limit && (i == 0 || !key_eq<KW>(h, l, ph, pl))) ? 1u : 0u;
      pl = l; ph = h;
    }
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ u32 ws[CB_THREADS / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 tot = 0;
    for (int q = 0; q < CB_THREADS / 32; ++q) tot += ws[q];
    counts[blockIdx.x] = tot;
  }
}

// exclusive scan of nb block counts in one CTA (1024 threads, sequential per
// thread chunk); *total = sum
// base != nullptr: group numbers continue after *base (device-resident
// output count, the wide merge appending window after window without a host
// round trip); *total = *base + groups then
__global__ void __launch_bounds__(1024) k_cl_scan(u32* __restrict__ counts, u32 nb, u32* __restrict__ total,
                                                  const u32* __restrict__ base) {
  const u32 b0v = base ? *base : 0u;
  __shared__ u32 ws[32];
  const u32 per = (nb + 1023) / 1024;
  const u32 b0 = min(nb, threadIdx.x * per), b1 = min(nb, b0 + per);
  u32 s = 0;
  for (u32 b = b0; b < b1; ++b) s += counts[b];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32 x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    u32 v = ws[lane];
    u32 y = v;
    for (int o = 1; o < 32; o <<= 1) {
      const u32 z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    ws[lane] = y - v;
    if (lane == 31) *total = b0v + y;
  }
  __syncthreads();
  u32 run = b0v + ws[w] + x - s;
  for (u32 b = b0; b < b1; ++b) {
    const u32 c = counts[b];
    counts[b] = run;
    run += c;
  }
}

void block_counts_scan(u32* counts, u32 nb, u32* total, const u32* base, cudaStream_t st) {
  klaunch(k_cl_scan, 1, 1024, 0, st, counts, nb, total, base);
}

template <int KW, int MS>
__global__ void __launch_bounds__(CB_THREADS) k_seg_reduce_b(const u64* __restrict__ lo, const u64* __restrict__ hi,
                                                             const u32* __restrict__ val, u32 m, u32 limit, SlotDesc sd,
                                                             i64 row0, const u64* __restrict__ st_in,
                                                             const u32* __restrict__ bbase, u64* __restrict__ out_lo,
                                                             u64* __restrict__ out_hi, u64* __restrict__ out_st,
                                                             u64* __restrict__ partial, u32* __restrict__ partial_slot,
                                                             u64 add_lo, u64 add_hi, int by_pos) {
  const int S = sd.nslots;
  constexpr u32 CLI = (u32)cl_items(MS);
  const u32 t = blockIdx.x * CB_THREADS + threadIdx.x;
  const u32 i0 = t * CLI, i1 = min(i0 + CLI, m);
  // States of <= 2 slots: the thread's items are read once into registers and
  // every item's state row is requested before any is combined (CLI random
  // gathers in flight per thread instead of one).
  constexpr bool PF = MS <= 2;
  constexpr u32 NPF = PF ? CLI : 1;
  u64 L[NPF], Hh[NPF], C[NPF][MS];
  u32 V[NPF];
  if (PF && i0 < m) {
#pragma unroll
    for (u32 j = 0; j < NPF; ++j) {
      const u32 i = i0 + j;
      const bool ok = i < i1;
      L[j] = ok ? lo[i] : 0;
      Hh[j] = (KW == 2 && ok) ? hi[i] : 0;
      V[j] = ok ? val[i] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (u32 j = 0; j < NPF; ++j) {
#pragma unroll
      for (int k = 0; k < MS; ++k) C[j][k] = 0;
      if (S && i0 + j < i1 && V[j] < limit)
        load_state_row<MS>(sd, by_pos ? (i64)0 : row0, st_in, by_pos ? i0 + j : V[j], C[j]);
    }
  }
  // this thread's included heads -> its first group index (block scan)
  u32 c = 0;
  if (i0 < m) {
    u64 pl = i0 > 0 ? lo[i0 - 1] : 0, ph = (KW == 2 && i0 > 0) ? hi[i0 - 1] : 0;
#pragma unroll(PF ? CLI : 1)
    for (u32 jj = 0; jj < CLI; ++jj) {
      const u32 i = i0 + jj;
      if (i >= i1) break;
      const u32 pj = PF ? jj : 0;
      const u64 l = PF ? L[pj] : lo[i], h = KW == 2 ? (PF ? Hh[pj] : hi[i]) : 0;
      const u32 vv = PF ? V[pj] : val[i];
      c += (vv < limit && (i == 0 || !key_eq<KW>(h, l, ph, pl))) ? 1u : 0u;
      pl = l; ph = h;
    }
  }
  __shared__ u32 ws[CB_THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32 x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  u32 wpre = 0;
  for (int q = 0; q < w; ++q) wpre += ws[q];
  u32 hp = bbase[blockIdx.x] + wpre + x - c;   // group index of this thread's first head
  if (i0 >= m) return;
  u64 acc[MS];
  u64 cur[MS];
#pragma unroll
  for (int k = 0; k < MS; ++k) acc[k] = cur[k] = 0;
  bool have = false, lead = true;
  u32 slot = 0;
  u64 prev_lo = 0, prev_hi = 0;
  if (i0 > 0) { prev_lo = lo[i0 - 1]; prev_hi = KW == 2 ? hi[i0 - 1] : 0; }
  partial_slot[t] = 0xFFFFFFFFu;
  const u32 lead_slot = hp - 1;
  auto flush = [&]() {
    if (lead) {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) partial[(size_t)t * S + k] = acc[k];
      partial_slot[t] = lead_slot;
    } else {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) out_st[(size_t)slot * S + k] = acc[k];
    }
  };
#pragma unroll(PF ? CLI : 1)
  for (u32 jj = 0; jj < CLI; ++jj) {
    const u32 i = i0 + jj;
    if (i >= i1) break;
    const u32 pj = PF ? jj : 0;
    u64 l = PF ? L[pj] : lo[i], h = KW == 2 ? (PF ? Hh[pj] : hi[i]) : 0;
    u32 v = PF ? V[pj] : val[i];
    bool head = (i == 0) || !key_eq<KW>(h, l, prev_hi, prev_lo);
    prev_lo = l; prev_hi = h;
    if (v >= limit) continue;
    if (PF) {
#pragma unroll
      for (int k = 0; k < MS; ++k) cur[k] = C[pj][k];
    } else if (S) {
      load_state_row<MS>(sd, by_pos ? (i64)0 : row0, st_in, by_pos ? i : v, cur);   // by_pos: values in sorted order
    }
    if (head) {
      if (have) flush();
      have = true; lead = false;
      slot = hp++;
      const u64 ol = l + add_lo;   // keys were sorted relative to the window's low bound
      out_lo[slot] = ol;
      if (KW == 2) out_hi[slot] = h + add_hi + (ol < l ? 1ull : 0ull);
#pragma unroll
      for (int k = 0; k < MS; ++k) acc[k] = cur[k];
    } else if (!have) {
      have = true;
#pragma unroll
      for (int k = 0; k < MS; ++k) acc[k] = cur[k];
    } else {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) acc[k] = combine_slot(sd.op[k], sd.type[k], acc[k], cur[k]);
    }
  }
  if (have) flush();
}

template <int KW, int MS>
__global__ void k_seg_reduce(const u64* __restrict__ lo, const u64* __restrict__ hi, const u32* __restrict__ val,
                             u32 m, u32 limit, SlotDesc sd, i64 row0, const u64* __restrict__ st_in,
                             const u32* __restrict__ hpos, u64* __restrict__ out_lo, u64* __restrict__ out_hi,
                             u64* __restrict__ out_st, u64* __restrict__ partial, u32* __restrict__ partial_slot) {
  const int S = sd.nslots;
  const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
  constexpr u32 CLI = (u32)cl_items(MS);
  const u32 i0 = t * CLI;
  if (i0 >= m) return;
  const u32 i1 = min(i0 + CLI, m);
  u64 acc[MS];
  u64 cur[MS];
#pragma unroll
  for (int k = 0; k < MS; ++k) acc[k] = cur[k] = 0;
  bool have = false, lead = true;
  u32 slot = 0;
  u64 prev_lo = 0, prev_hi = 0;
  if (i0 > 0) { prev_lo = lo[i0 - 1]; prev_hi = KW == 2 ? hi[i0 - 1] : 0; }
  partial_slot[t] = 0xFFFFFFFFu;
  auto flush = [&]() {
    if (lead) {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) partial[(size_t)t * S + k] = acc[k];
      partial_slot[t] = hpos[i0] - 1;
    } else {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) out_st[(size_t)slot * S + k] = acc[k];
    }
  };
  for (u32 i = i0; i < i1; ++i) {
    u64 l = lo[i], h = KW == 2 ? hi[i] : 0;
    u32 v = val[i];
    bool head = (i == 0) || !key_eq<KW>(h, l, prev_hi, prev_lo);
    prev_lo = l; prev_hi = h;
    if (v >= limit) continue;
    if (S) load_state_row<MS>(sd, row0, st_in, v, cur);
    if (head) {
      if (have) flush();
      have = true; lead = false;
      slot = hpos[i];
      out_lo[slot] = l;
      if (KW == 2) out_hi[slot] = h;
#pragma unroll
      for (int k = 0; k < MS; ++k) acc[k] = cur[k];
    } else if (!have) {
      have = true;
#pragma unroll
      for (int k = 0; k < MS; ++k) acc[k] = cur[k];
    } else {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) acc[k] = combine_slot(sd.op[k], sd.type[k], acc[k], cur[k]);
    }
  }
  if (have) flush();
}

// Carries of segments that span several threads: consecutive threads that
// carry into the same output slot are first combined inside the warp (a
// segmented shuffle reduction toward the first lane of each run), then one
// atomic per (warp, slot) — heavy keys (Zipf) would otherwise serialize
// hundreds of thousands of same-address atomics.
template <int MS>
__global__ void k_seg_fixup(u32 nthreads, SlotDesc sd, const u64* __restrict__ partial,
                            const u32* __restrict__ partial_slot, u64* __restrict__ out_st) {
  const int S = sd.nslots;
  const int lane = threadIdx.x & 31;
  for (u32 base = blockIdx.x * blockDim.x; base < nthreads; base += gridDim.x * blockDim.x) {
    const u32 t = base + threadIdx.x;
    u32 slot = t < nthreads ? partial_slot[t] : 0xFFFFFFFFu;
    u64 x[MS];
#pragma unroll
    for (int k = 0; k < MS; ++k) x[k] = (k < S && slot != 0xFFFFFFFFu) ? partial[(size_t)t * S + k] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const u32 ys = __shfl_down_sync(0xffffffffu, slot, off);
      const bool take = lane + off < 32 && ys == slot && slot != 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < MS; ++k) {
        const u64 y = __shfl_down_sync(0xffffffffu, x[k], off);
        if (k < S && take) x[k] = combine_slot(sd.op[k], sd.type[k], x[k], y);
      }
    }
    const u32 prev = __shfl_up_sync(0xffffffffu, slot, 1);
    const bool head = (lane == 0 || prev != slot) && slot != 0xFFFFFFFFu;
    if (head) {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) atomic_combine(out_st + (size_t)slot * S + k, sd.op[k], sd.type[k], x[k]);
    }
  }
}

// ---------------------------------------------------------------------------
// Fused collapse: head flags, group numbering and the segmented reduce in one
// kernel over tiles of CF_THREADS * CF_IT sorted rows (Schema.merge_states
// over runs of equal keys, core.py:184-208; evict_all's sorted unique
// output, memindex.py:275-285).  Tiles take their index from a counter and
// chain through a decoupled look-back whose payload is (groups so far, state
// of the group still open at the tile's end): a tile learns both its first
// output index and the carry-in state of a group that started in an earlier
// tile.  Inside a tile every thread reduces its consecutive rows; a
// segmented scan over the threads gives each thread the state of the group
// open at its first row.  A group is written by the thread that holds the
// next group's head (or by the very last thread), so every output row is
// written once, without atomics.  The keys and row ids are read once
// (striped, coalesced, transposed through shared memory), each included
// row's state gathered once.
#define CF_THREADS 256
__host__ __device__ constexpr int cf_items(int MS) { return MS <= 2 ? 8 : (MS <= 8 ? 4 : 2); }

__device__ __forceinline__ u64 ld_acquire_gpu(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MS>
__device__ __forceinline__ void cf_identity(const SlotDesc& sd, u64 (&x)[MS]) {
#pragma unroll
  for (int k = 0; k < MS; ++k) x[k] = k < sd.nslots ? identity_slot(sd.op[k], sd.type[k]) : 0;
}
// a <- a (+) b, a before b in row order
template <int MS>
__device__ __forceinline__ void cf_combine(const SlotDesc& sd, u64 (&a)[MS], const u64 (&b)[MS]) {
#pragma unroll
  for (int k = 0; k < MS; ++k)
    if (k < sd.nslots) a[k] = combine_slot(sd.op[k], sd.type[k], a[k], b[k]);
}

template <int KW, int MS>
__global__ void __launch_bounds__(CF_THREADS) k_collapse_fused(
    const u64* __restrict__ lo, const u64* __restrict__ hi, const u32* __restrict__ val, u32 m, u32 limit, SlotDesc sd,
    i64 row0, const u64* __restrict__ st_in, u64* __restrict__ out_lo, u64* __restrict__ out_hi,
    u64* __restrict__ out_st, u64* __restrict__ status, u64* __restrict__ pay, u32* __restrict__ ticket, u32 epoch,
    u32 ntiles, u32* __restrict__ total) {
  constexpr int IT = cf_items(MS);
  constexpr u32 TILE = CF_THREADS * IT;
  constexpr u32 PADN = TILE + TILE / IT;
  __shared__ u64 s_lo[PADN];
  __shared__ u64 s_hi[KW == 2 ? PADN : 1];
  __shared__ u32 s_v[PADN];
  __shared__ u32 s_tile, s_hx, sw[8];
  __shared__ u64 s_prev_lo, s_prev_hi;
  __shared__ u64 s_wv[8][MS];
  __shared__ unsigned char s_wf[8];
  __shared__ u64 s_carry[MS];
  const int S = sd.nslots;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 base = tile * TILE;
  const u32 tn = min(TILE, m - base);
  auto P = [](u32 i) { return i + i / IT; };
  // ---- striped, coalesced loads -> shared memory
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const u32 q = it * CF_THREADS + tid;
    if (q < tn) {
      s_lo[P(q)] = lo[base + q];
      if (KW == 2) s_hi[P(q)] = hi[base + q];
      s_v[P(q)] = val[base + q];
    }
  }
  if (tid == 0 && base > 0) {
    s_prev_lo = lo[base - 1];
    s_prev_hi = KW == 2 ? hi[base - 1] : 0;
  }
  __syncthreads();
  // ---- blocked: heads, included rows, gathered states
  const u32 i0 = tid * IT;
  u64 kl[IT], kh[IT];
  u32 hmask = 0, imask = 0;
  u64 pl = 0, ph = 0;
  bool have_prev = false;
  if (i0 > 0 && i0 <= tn) { pl = s_lo[P(i0 - 1)]; ph = KW == 2 ? s_hi[P(i0 - 1)] : 0; have_prev = true; }
  else if (i0 == 0 && base > 0) { pl = s_prev_lo; ph = s_prev_hi; have_prev = true; }
  u64 cur[IT][MS];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const u32 i = i0 + it;
    kl[it] = 0; kh[it] = 0;
    if (i < tn) {
      kl[it] = s_lo[P(i)];
      kh[it] = KW == 2 ? s_hi[P(i)] : 0;
      const u32 v = s_v[P(i)];
      const bool inc = v < limit;
      const bool head = inc && (!have_prev || !key_eq<KW>(kh[it], kl[it], ph, pl));
      pl = kl[it]; ph = kh[it]; have_prev = true;
      if (inc) {
        imask |= 1u << it;
        if (S) load_state_row<MS>(sd, row0, st_in, v, cur[it]);
      }
      if (head) hmask |= 1u << it;
    }
  }
  // ---- thread summary: lead (rows before the first head) or trail (from the last head)
  u64 sv[MS];
  cf_identity<MS>(sd, sv);
  const u32 nh = __popc(hmask);
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    if (!((imask >> it) & 1u)) continue;
    if ((hmask >> it) & 1u) {
#pragma unroll
      for (int k = 0; k < MS; ++k) sv[k] = cur[it][k];
    } else {
      cf_combine<MS>(sd, sv, cur[it]);
    }
  }
  // after this loop: nh > 0 -> sv = trail; nh == 0 -> sv = lead (all rows)
  u32 htot;
  const u32 hx = block_excl_scan256(nh, sw, &htot);
  // ---- segmented scan over threads of (has head, sv): exclusive -> (fx, cx)
  bool f = nh > 0;
  u64 v[MS];
#pragma unroll
  for (int k = 0; k < MS; ++k) v[k] = sv[k];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const bool fu = __shfl_up_sync(0xffffffffu, f, o);
    u64 vu[MS];
#pragma unroll
    for (int k = 0; k < MS; ++k) vu[k] = __shfl_up_sync(0xffffffffu, v[k], o);
    if (lane >= o) {
      if (!f) {
        cf_combine<MS>(sd, vu, v);
#pragma unroll
        for (int k = 0; k < MS; ++k) v[k] = vu[k];
      }
      f = f || fu;
    }
  }
  if (lane == 31) {
    s_wf[wid] = f ? 1 : 0;
#pragma unroll
    for (int k = 0; k < MS; ++k) s_wv[wid][k] = v[k];
  }
  // exclusive within the warp
  bool fx = __shfl_up_sync(0xffffffffu, f, 1);
  u64 cx[MS];
#pragma unroll
  for (int k = 0; k < MS; ++k) cx[k] = __shfl_up_sync(0xffffffffu, v[k], 1);
  if (lane == 0) { fx = false; cf_identity<MS>(sd, cx); }
  __syncthreads();
  // warp prefixes (thread 0, in order) + the tile's inclusive summary
  __shared__ unsigned char s_pf[8];
  __shared__ u64 s_pv[8][MS];
  __shared__ u64 s_tv[MS];
  __shared__ unsigned char s_tf;
  if (tid == 0) {
    bool pf = false;
    u64 pv[MS];
    cf_identity<MS>(sd, pv);
    for (int q = 0; q < 8; ++q) {
      s_pf[q] = pf ? 1 : 0;
#pragma unroll
      for (int k = 0; k < MS; ++k) s_pv[q][k] = pv[k];
      if (s_wf[q]) {
#pragma unroll
        for (int k = 0; k < MS; ++k) pv[k] = s_wv[q][k];
        pf = true;
      } else {
        u64 t[MS];
#pragma unroll
        for (int k = 0; k < MS; ++k) t[k] = s_wv[q][k];
        cf_combine<MS>(sd, pv, t);
      }
    }
    s_tf = pf ? 1 : 0;
#pragma unroll
    for (int k = 0; k < MS; ++k) s_tv[k] = pv[k];
    // ---- decoupled look-back: groups before this tile, carry-in state
    const u64 E = (u64)epoch << 34;
    u64* agg = pay + (size_t)tile * 2 * S;
    u64* inc = agg + S;
    u32 Hx = 0;
    u64 acc[MS];
    cf_identity<MS>(sd, acc);
    if (tile == 0) {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) inc[k] = pv[k];
      st_release_gpu(status, E | (2ull << 32) | htot);
    } else {
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) agg[k] = pv[k];
      st_release_gpu(status + tile, E | (1ull << 32) | htot);
      bool sdone = false;
      for (int q = (int)tile - 1; q >= 0;) {
        const u64 x = ld_acquire_gpu(status + q);
        if ((x >> 34) != (u64)epoch) continue;   // not published yet
        const u32 fl = (u32)(x >> 32) & 3u;
        const u64* qp = pay + (size_t)q * 2 * S + (fl == 2 ? S : 0);
        Hx += (u32)x;
        if (!sdone) {
          u64 t[MS];
#pragma unroll
          for (int k = 0; k < MS; ++k) t[k] = k < S ? qp[k] : 0;
          cf_combine<MS>(sd, t, acc);
#pragma unroll
          for (int k = 0; k < MS; ++k) acc[k] = t[k];
          if (fl == 1 && (u32)x > 0) sdone = true;
        }
        if (fl == 2) break;
        --q;
      }
      u64 ti[MS];
#pragma unroll
      for (int k = 0; k < MS; ++k) ti[k] = acc[k];
      if (!pf) cf_combine<MS>(sd, ti, pv);
#pragma unroll
      for (int k = 0; k < MS; ++k)
        if (k < S) inc[k] = pf ? pv[k] : ti[k];
      st_release_gpu(status + tile, E | (2ull << 32) | (Hx + htot));
    }
    s_hx = Hx;
#pragma unroll
    for (int k = 0; k < MS; ++k) s_carry[k] = acc[k];
    if (tile + 1 == ntiles) *total = Hx + htot;
  }
  __syncthreads();
  // ---- this thread's carry-in: the state of the group open at its first row
  const u32 Hx = s_hx;
  {
    const bool wf = s_pf[wid];
    if (!fx) {
      u64 t[MS];
#pragma unroll
      for (int k = 0; k < MS; ++k) t[k] = s_pv[wid][k];
      cf_combine<MS>(sd, t, cx);
#pragma unroll
      for (int k = 0; k < MS; ++k) cx[k] = t[k];
      fx = wf;
    }
    if (!fx) {
      u64 t[MS];
#pragma unroll
      for (int k = 0; k < MS; ++k) t[k] = s_carry[k];
      cf_combine<MS>(sd, t, cx);
#pragma unroll
      for (int k = 0; k < MS; ++k) cx[k] = t[k];
    }
  }
  // ---- writes: groups that close in this thread
  u32 g = Hx + hx;           // index of this thread's first head
  bool open = g > 0;         // a group is open at this thread's first row
  u64 acc[MS];
#pragma unroll
  for (int k = 0; k < MS; ++k) acc[k] = cx[k];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    if (!((imask >> it) & 1u)) continue;
    if ((hmask >> it) & 1u) {
      if (open && S) {
#pragma unroll
        for (int k = 0; k < MS; ++k)
          if (k < S) out_st[(size_t)(g - 1) * S + k] = acc[k];
      }
      out_lo[g] = kl[it];
      if (KW == 2) out_hi[g] = kh[it];
#pragma unroll
      for (int k = 0; k < MS; ++k) acc[k] = cur[it][k];
      open = true;
      ++g;
    } else {
      cf_combine<MS>(sd, acc, cur[it]);
    }
  }
  if (tile + 1 == ntiles && tid == CF_THREADS - 1 && open && S) {
#pragma unroll
    for (int k = 0; k < MS; ++k)
      if (k < S) out_st[(size_t)(g - 1) * S + k] = acc[k];
  }
}

static std::atomic<u32> g_cf_epoch{0};
static bool collapse_fused_env() {
  static int v = -1;
  // opt-in (ISA_COLLAPSE=fused): measured slower than the multi-kernel
  // collapse (config 5 35 -> 45 ms, config 3 43 -> 112 ms per 1e9 rows:
  // register-bound occupancy for the random gathers, and the single-thread
  // look-back walks long heavy-hitter segments tile by tile)
  if (v < 0) { const char* e = getenv("ISA_COLLAPSE"); v = (e && e[0] == 'f') ? 1 : 0; }
  return v == 1;
}
u32 collapse_tiles(u32 m, int S) {
  const int MS = S <= 1 ? 1 : (S <= 2 ? 2 : (S <= 4 ? 4 : (S <= 5 ? 5 : (S <= 8 ? 8 : 16))));
  const u32 tile = CF_THREADS * cf_items(MS);
  return (m + tile - 1) / tile;
}

// value columns addressed by sorted position (CollapseTmp::by_pos) need the block-count path
bool collapse_by_pos_ok(u32 m, int S) {
  const char* e = getenv("ISA_COLLAPSE");
  if (e && (e[0] == 'r' || e[0] == 'f')) return false;
  return (collapse_threads(m, S) + 127) / 128 <= 1024u * 1024u;
}

void collapse(int KW, const u64* lo, const u64* hi, const u32* val, u32 m, u32 limit, const SlotDesc& sd,
              int64_t row0, const u64* st_in, u64* out_lo, u64* out_hi, u64* out_st, CollapseTmp& tmp,
              cudaStream_t st) {
  if (m == 0) {
    if (tmp.dev_base) cudaMemcpyAsync(tmp.total, tmp.dev_base, sizeof(u32), cudaMemcpyDeviceToDevice, st);
    else cudaMemsetAsync(tmp.total, 0, sizeof(u32), st);
    return;
  }
  if (tmp.status && collapse_fused_env() && !tmp.dev_base) {
    const int S = sd.nslots;
    const u32 nt = collapse_tiles(m, S);
    const u32 ep = (g_cf_epoch.fetch_add(1) % 0x3FFFFFFEu) + 1u;
    cudaMemsetAsync(tmp.ticket, 0, sizeof(u32), st);
#define CF_LAUNCH(K, M) klaunch(k_collapse_fused<K, M>, nt, CF_THREADS, 0, st, lo, hi, val, m, limit, sd, (i64)row0, st_in, \
                                out_lo, out_hi, out_st, tmp.status, tmp.pay, tmp.ticket, ep, nt, tmp.total)
#define CF_KW(K) { if (S <= 1) CF_LAUNCH(K, 1); else if (S <= 2) CF_LAUNCH(K, 2); else if (S <= 4) CF_LAUNCH(K, 4); \
                   else if (S <= 5) CF_LAUNCH(K, 5); else if (S <= 8) CF_LAUNCH(K, 8); else CF_LAUNCH(K, 16); }
    if (KW == 2) CF_KW(2) else CF_KW(1)
#undef CF_KW
#undef CF_LAUNCH
    return;
  }
  u32 nthreads = collapse_threads(m, sd.nslots);
  int blocks = (nthreads + 127) / 128;
  const int S = sd.nslots;
  // block head counts (default; config 5 collapse 35 -> 29 ms, window collapse
  // 28 -> 22 ms per 1e9 rows, profiles/r2_ab_collapse.txt); ISA_COLLAPSE=rowflags:
  // per-row head flags + full scan (round-1 path)
  static int cb_env = -1;
  if (cb_env < 0) { const char* e = getenv("ISA_COLLAPSE"); cb_env = (e && e[0] == 'r') ? 0 : 1; }
  if ((cb_env || tmp.dev_base) && (u32)blocks <= 1024u * 1024u) {
    // block head counts -> one-CTA scan -> reduce numbering its own groups
#define CB_CNT(K, M) klaunch(k_cl_count<K, M>, blocks, CB_THREADS, 0, st, lo, hi, val, m, limit, tmp.flags)
#define CB_RED(K, M) klaunch(k_seg_reduce_b<K, M>, blocks, CB_THREADS, 0, st, lo, hi, val, m, limit, sd, (i64)row0, \
                             st_in, (const u32*)tmp.flags, out_lo, out_hi, out_st, tmp.partial, tmp.partial_slot, \
                             tmp.key_add_lo, tmp.key_add_hi, tmp.by_pos ? 1 : 0)
#define CB_KW(K, X) { if (S <= 1) X(K, 1); else if (S <= 2) X(K, 2); else if (S <= 4) X(K, 4); \
                      else if (S <= 5) X(K, 5); else if (S <= 8) X(K, 8); else X(K, 16); }
    if (KW == 2) CB_KW(2, CB_CNT) else CB_KW(1, CB_CNT)
    klaunch(k_cl_scan, 1, 1024, 0, st, tmp.flags, (u32)blocks, tmp.total, (const u32*)tmp.dev_base);
    if (KW == 2) CB_KW(2, CB_RED) else CB_KW(1, CB_RED)
#undef CB_KW
#undef CB_RED
#undef CB_CNT
  } else {
  int g = grid_for(m, 256);
  if (KW == 2) klaunch(k_head_flags<2>, g, 256, 0, st, lo, hi, val, m, limit, tmp.flags);
  else klaunch(k_head_flags<1>, g, 256, 0, st, lo, hi, val, m, limit, tmp.flags);
  scan_exclusive_u32(tmp.flags, m, tmp.scan_tmp, tmp.total, st);
#define SR_LAUNCH(K, M) klaunch(k_seg_reduce<K, M>, blocks, 128, 0, st, lo, hi, val, m, limit, sd, row0, st_in, \
                                tmp.flags, out_lo, out_hi, out_st, tmp.partial, tmp.partial_slot)
#define SR_KW(K) { if (S <= 1) SR_LAUNCH(K, 1); else if (S <= 2) SR_LAUNCH(K, 2); else if (S <= 4) SR_LAUNCH(K, 4); \
                   else if (S <= 5) SR_LAUNCH(K, 5); else if (S <= 8) SR_LAUNCH(K, 8); else SR_LAUNCH(K, 16); }
  if (KW == 2) SR_KW(2) else SR_KW(1)
#undef SR_KW
#undef SR_LAUNCH
  }
  if (S) {
    const int g = grid_for(nthreads, 256);
    if (S <= 2) klaunch(k_seg_fixup<2>, g, 256, 0, st, nthreads, sd, tmp.partial, tmp.partial_slot, out_st);
    else if (S <= 4) klaunch(k_seg_fixup<4>, g, 256, 0, st, nthreads, sd, tmp.partial, tmp.partial_slot, out_st);
    else if (S <= 8) klaunch(k_seg_fixup<8>, g, 256, 0, st, nthreads, sd, tmp.partial, tmp.partial_slot, out_st);
    else klaunch(k_seg_fixup<16>, g, 256, 0, st, nthreads, sd, tmp.partial, tmp.partial_slot, out_st);
  }
}

// Materialize a sorted sequence as run rows (duplicates kept): keys from the
// sorted buffers, states gathered by value index from already-built states
// (st_in) or built from the raw input rows (make_state).
template <int KW, int MS>
__global__ void k_materialize(const u64* __restrict__ lo, const u64* __restrict__ hi, const u32* __restrict__ val,
                              u32 m, SlotDesc sd, i64 row0, const u64* __restrict__ st_in, u64* __restrict__ out_lo,
                              u64* __restrict__ out_hi, u64* __restrict__ out_st) {
  const int S = sd.nslots;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    out_lo[i] = lo[i];
    if (KW == 2) out_hi[i] = hi[i];
    if (S) {
      u64 s[MS];
      load_state_row<MS>(sd, row0, st_in, val[i], s);
#pragma unroll
      for (int q = 0; q < MS; ++q)
        if (q < S) out_st[(size_t)i * S + q] = s[q];
    }
  }
}

template <int KW>
__global__ void k_count_heads(const u64* __restrict__ lo, const u64* __restrict__ hi, u32 m, u32* __restrict__ out) {
  u32 c = 0;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    c += (i == 0 || !key_eq<KW>(KW == 2 ? hi[i] : 0, lo[i], KW == 2 ? hi[i - 1] : 0, lo[i - 1])) ? 1u : 0u;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

void materialize(int KW, const u64* lo, const u64* hi, const u32* val, u32 m, const SlotDesc& sd, int64_t row0,
                 const u64* st_in, u64* out_lo, u64* out_hi, u64* out_st, u32* heads, cudaStream_t st) {
  if (m == 0) return;
  const int g = grid_for(m, 256), S = sd.nslots;
#define MT(K, M) klaunch(k_materialize<K, M>, g, 256, 0, st, lo, hi, val, m, sd, row0, st_in, out_lo, out_hi, out_st)
#define MT_KW(K) { if (S <= 1) MT(K, 1); else if (S <= 2) MT(K, 2); else if (S <= 4) MT(K, 4); else if (S <= 8) MT(K, 8); else MT(K, 16); }
  if (KW == 2) MT_KW(2) else MT_KW(1)
#undef MT_KW
#undef MT
  if (heads) {
    if (KW == 2) klaunch(k_count_heads<2>, g, 256, 0, st, lo, hi, m, heads);
    else klaunch(k_count_heads<1>, g, 256, 0, st, lo, (const u64*)nullptr, m, heads);
  }
}

// ============================================================= merge ====
template <int KW>
__global__ void k_rank(const u64* __restrict__ x_lo, const u64* __restrict__ x_hi, u32 nx,
                       const u64* __restrict__ y_lo, const u64* __restrict__ y_hi, u32 ny, u32* __restrict__ rank,
                       u32* __restrict__ match) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < nx; i += gridDim.x * blockDim.x) {
    u64 l = x_lo[i], h = KW == 2 ? x_hi[i] : 0;
    u32 p = lower_bound_key<KW>(y_lo, y_hi, ny, h, l);
    rank[i] = p;
    match[i] = (p < ny && key_eq<KW>(KW == 2 ? y_hi[p] : 0, y_lo[p], h, l)) ? 1u : 0u;
  }
}

struct OpsArr { int op[ISA_MAX_SLOTS]; int type[ISA_MAX_SLOTS]; };

template <int KW, int MS>
__global__ void k_merge_write_a(const u64* __restrict__ a_lo, const u64* __restrict__ a_hi,
                                const u64* __restrict__ a_st, u32 na, const u64* __restrict__ b_st,
                                const u32* __restrict__ rank, const u32* __restrict__ mpre,
                                const u32* __restrict__ match, int S, OpsArr ops, u64* __restrict__ c_lo,
                                u64* __restrict__ c_hi, u64* __restrict__ c_st) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
    u32 j = rank[i];
    u32 o = i + j - mpre[i];
    c_lo[o] = a_lo[i];
    if (KW == 2) c_hi[o] = a_hi[i];
    bool mt = match[i] != 0;
#pragma unroll
    for (int k = 0; k < MS; ++k) {
      if (k < S) {
        u64 s = a_st[(size_t)i * S + k];
        if (mt) s = combine_slot(ops.op[k], ops.type[k], s, b_st[(size_t)j * S + k]);
        c_st[(size_t)o * S + k] = s;
      }
    }
  }
}

template <int KW>
__global__ void k_merge_write_b(const u64* __restrict__ b_lo, const u64* __restrict__ b_hi,
                                const u64* __restrict__ b_st, u32 nb, const u32* __restrict__ rank,
                                const u32* __restrict__ mpre, const u32* __restrict__ match, int S,
                                u64* __restrict__ c_lo, u64* __restrict__ c_hi, u64* __restrict__ c_st) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += gridDim.x * blockDim.x) {
    if (match[j]) continue;
    u32 o = j + rank[j] - mpre[j];
    c_lo[o] = b_lo[j];
    if (KW == 2) c_hi[o] = b_hi[j];
    for (int k = 0; k < S; ++k) c_st[(size_t)o * S + k] = b_st[(size_t)j * S + k];
  }
}

__global__ void k_copy_u32(const u32* __restrict__ s, u32* __restrict__ d, u32 n) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) d[i] = s[i];
}

void rank_match(int KW, const u64* x_lo, const u64* x_hi, u32 nx, const u64* y_lo, const u64* y_hi, u32 ny,
                u32* rank, u32* match, cudaStream_t st) {
  if (!nx) return;
  const int g = grid_for(nx, 256);
  if (KW == 2) klaunch(k_rank<2>, g, 256, 0, st, x_lo, x_hi, nx, y_lo, y_hi, ny, rank, match);
  else klaunch(k_rank<1>, g, 256, 0, st, x_lo, x_hi, nx, y_lo, y_hi, ny, rank, match);
}

template <int KW>
__global__ void k_compact_keys(const u64* __restrict__ lo, const u64* __restrict__ hi, const u32* __restrict__ flag,
                               const u32* __restrict__ pre, u32 n, u64* __restrict__ out_lo,
                               u64* __restrict__ out_hi) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    out_lo[pre[i]] = lo[i];
    if (KW == 2) out_hi[pre[i]] = hi[i];
  }
}

void compact_keys(int KW, const u64* lo, const u64* hi, const u32* flag, const u32* pre, u32 n, u64* out_lo,
                  u64* out_hi, cudaStream_t st) {
  if (!n) return;
  const int g = grid_for(n, 256);
  if (KW == 2) klaunch(k_compact_keys<2>, g, 256, 0, st, lo, hi, flag, pre, n, out_lo, out_hi);
  else klaunch(k_compact_keys<1>, g, 256, 0, st, lo, hi, flag, pre, n, out_lo, out_hi);
}

void merge_combine(int KW, int S, const int* ops, const int* types, const u64* a_lo, const u64* a_hi,
                   const u64* a_st, u32 na, const u64* b_lo, const u64* b_hi, const u64* b_st, u32 nb,
                   u64* c_lo, u64* c_hi, u64* c_st, MergeTmp& tmp, cudaStream_t st) {
  OpsArr oa;
  for (int k = 0; k < ISA_MAX_SLOTS; ++k) { oa.op[k] = k < S ? ops[k] : 0; oa.type[k] = k < S ? types[k] : 0; }
  // ranks + match flags; prefix of match flags is built in a copy (match kept)
  if (na) {
    int g = grid_for(na, 256);
    if (KW == 2) klaunch(k_rank<2>, g, 256, 0, st, a_lo, a_hi, na, b_lo, b_hi, nb, tmp.rank_a, tmp.match_a);
    else klaunch(k_rank<1>, g, 256, 0, st, a_lo, a_hi, na, b_lo, b_hi, nb, tmp.rank_a, tmp.match_a);
  }
  if (nb) {
    int g = grid_for(nb, 256);
    if (KW == 2) klaunch(k_rank<2>, g, 256, 0, st, b_lo, b_hi, nb, a_lo, a_hi, na, tmp.rank_b, tmp.match_b);
    else klaunch(k_rank<1>, g, 256, 0, st, b_lo, b_hi, nb, a_lo, a_hi, na, tmp.rank_b, tmp.match_b);
  }
  // prefix counts live after the flags: match_x[n + 1 + i]
  u32* pre_a = tmp.match_a + na + 1;
  u32* pre_b = tmp.match_b + nb + 1;
  if (na) {
    klaunch(k_copy_u32, grid_for(na, 256), 256, 0, st, tmp.match_a, pre_a, na);
    scan_exclusive_u32(pre_a, na, tmp.scan_tmp, tmp.total, st);
    int g = grid_for(na, 256);
#define MW_LAUNCH(K, M) klaunch(k_merge_write_a<K, M>, g, 256, 0, st, a_lo, a_hi, a_st, na, b_st, tmp.rank_a, pre_a, \
                                tmp.match_a, S, oa, c_lo, c_hi, c_st)
#define MW_KW(K) { if (S <= 1) MW_LAUNCH(K, 1); else if (S <= 2) MW_LAUNCH(K, 2); else if (S <= 4) MW_LAUNCH(K, 4); \
                   else if (S <= 8) MW_LAUNCH(K, 8); else MW_LAUNCH(K, 16); }
    if (KW == 2) MW_KW(2) else MW_KW(1)
#undef MW_KW
#undef MW_LAUNCH
  } else {
    cudaMemsetAsync(tmp.total, 0, sizeof(u32), st);
  }
  if (nb) {
    klaunch(k_copy_u32, grid_for(nb, 256), 256, 0, st, tmp.match_b, pre_b, nb);
    scan_exclusive_u32(pre_b, nb, tmp.scan_tmp, tmp.total + 1, st);
    int g = grid_for(nb, 256);
    if (KW == 2) klaunch(k_merge_write_b<2>, g, 256, 0, st, b_lo, b_hi, b_st, nb, tmp.rank_b, pre_b, tmp.match_b, S, c_lo, c_hi, c_st);
    else klaunch(k_merge_write_b<1>, g, 256, 0, st, b_lo, b_hi, b_st, nb, tmp.rank_b, pre_b, tmp.match_b, S, c_lo, c_hi, c_st);
  } else {
    cudaMemsetAsync(tmp.total + 1, 0, sizeof(u32), st);
  }
}

// one warp per (table row, slot) cell: strided combine over the CTAs' partials, then a warp reduction
__global__ void k_fold_partials(int nt, SlotDesc sd, const u64* __restrict__ partials, u32 grid, u64* __restrict__ T_st) {
  const int S = sd.nslots;
  const int q = blockIdx.x;   // cell
  const int j = q / S, s = q % S;
  const int op = sd.op[s], ty = sd.type[s];
  u64 x = identity_slot(op, ty);
  for (u32 c = threadIdx.x; c < grid; c += 32) x = combine_slot(op, ty, x, partials[((size_t)c * nt + j) * S + s]);
  for (int o = 16; o; o >>= 1) x = combine_slot(op, ty, x, __shfl_xor_sync(0xffffffffu, x, o));
  if (threadIdx.x == 0) T_st[(size_t)j * S + s] = combine_slot(op, ty, T_st[(size_t)j * S + s], x);
}

void fold_partials(int nt, const SlotDesc& sd, const u64* partials, u32 grid, u64* T_st, cudaStream_t st) {
  int n = nt * sd.nslots;
  if (n) klaunch(k_fold_partials, n, 32, 0, st, nt, sd, partials, grid, T_st);
}

__global__ void k_compact_misses(const u32* __restrict__ miss_buf, const u32* __restrict__ miss_cnt,
                                 const u32* __restrict__ miss_off, u32 rpc, u32* __restrict__ out) {
  const u32 c = blockIdx.x;
  const u32 cnt = miss_cnt[c], off = miss_off[c];
  for (u32 i = threadIdx.x; i < cnt; i += blockDim.x) out[off + i] = miss_buf[(size_t)c * rpc + i];
}

void compact_misses(const u32* miss_buf, const u32* miss_cnt, const u32* miss_off, u32 grid, u32 rows_per_cta,
                    u32* out, cudaStream_t st) {
  klaunch(k_compact_misses, grid, 256, 0, st, miss_buf, miss_cnt, miss_off, rows_per_cta, out);
}

// ========================================================== export ====
__global__ void k_export_key(const u64* __restrict__ lo, const u64* __restrict__ hi, u32 n, int dtype, int shift,
                             int width, void* out) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 f = key_field(hi ? hi[i] : 0, lo[i], shift, width);
    if (dtype_signed(dtype)) f ^= (1ull << (width - 1));
    switch (width) {
      case 8: ((unsigned char*)out)[i] = (unsigned char)f; break;
      case 16: ((unsigned short*)out)[i] = (unsigned short)f; break;
      case 32: ((unsigned int*)out)[i] = (unsigned int)f; break;
      default: ((u64*)out)[i] = f; break;
    }
  }
}

void export_key_col(const u64* lo, const u64* hi, u32 n, int dtype, int shift, int width, void* out, cudaStream_t st) {
  if (n) klaunch(k_export_key, grid_for(n, 256), 256, 0, st, lo, hi, n, dtype, shift, width, out);
}

// every key column and every state slot of rows [0, n) in one pass
__global__ void k_export_all(const u64* __restrict__ lo, const u64* __restrict__ hi, const u64* __restrict__ stt,
                             u32 n, ExportDesc ed) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 l = lo[i], h = hi ? hi[i] : 0;
    for (int c = 0; c < ed.ncols; ++c) {
      if (!ed.key_dst[c]) continue;
      const int w = ed.width[c];
      u64 f = key_field(h, l, ed.shift[c], w);
      if (ed.is_signed[c]) f ^= (1ull << (w - 1));
      switch (w) {
        case 8: ((unsigned char*)ed.key_dst[c])[i] = (unsigned char)f; break;
        case 16: ((unsigned short*)ed.key_dst[c])[i] = (unsigned short)f; break;
        case 32: ((unsigned int*)ed.key_dst[c])[i] = (unsigned int)f; break;
        default: ((u64*)ed.key_dst[c])[i] = f; break;
      }
    }
    for (int s = 0; s < ed.nslots; ++s)
      if (ed.slot_dst[s]) ((u64*)ed.slot_dst[s])[i] = stt[(size_t)i * ed.nslots + s];
  }
}

void export_all(const u64* lo, const u64* hi, const u64* stt, u32 n, const ExportDesc& ed, cudaStream_t st) {
  if (n) klaunch(k_export_all, grid_for(n, 256), 256, 0, st, lo, hi, stt, n, ed);
}

__global__ void k_export_slot(const u64* __restrict__ stt, int S, int s, u32 n, u64* __restrict__ out) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = stt[(size_t)i * S + s];
}

void export_slot(const u64* stt, int S, int s, u32 n, u64* out, cudaStream_t st) {
  if (n) klaunch(k_export_slot, grid_for(n, 256), 256, 0, st, stt, S, s, n, out);
}

// ======================================================= partition ====
__global__ void k_sample_keys(KeyDesc kd, i64 n, i64 stride, u64* __restrict__ out_lo, u64* __restrict__ out_hi) {
  i64 ns = (n + stride - 1) / stride;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < ns; i += (i64)gridDim.x * blockDim.x) {
    u64 h, l;
    load_key(kd, i * stride, h, l);
    out_lo[i] = l;
    out_hi[i] = h;
  }
}

void sample_keys(const KeyDesc& kd, int64_t n, int64_t stride, u64* out_lo, u64* out_hi, cudaStream_t st) {
  int64_t ns = (n + stride - 1) / stride;
  if (ns > 0) klaunch(k_sample_keys, grid_for(ns, 256), 256, 0, st, kd, n, stride, out_lo, out_hi);
}

template <int KW>
__global__ void k_partition_dest(KeyDesc kd, u32 n, const u64* __restrict__ s_lo, const u64* __restrict__ s_hi, int ns,
                                 u64* __restrict__ dest, u32* __restrict__ val) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 h, l;
    load_key(kd, i, h, l);
    // number of splitters <= key (upper bound)
    int lo_i = 0, hi_i = ns;
    while (lo_i < hi_i) {
      int m = (lo_i + hi_i) >> 1;
      u64 mh = KW == 2 ? s_hi[m] : 0;
      if (!key_less<KW>(h, l, mh, s_lo[m])) lo_i = m + 1; else hi_i = m;
    }
    dest[i] = (u64)lo_i;
    val[i] = i;
  }
}

void partition_dest(int KW, const KeyDesc& kd, u32 n, const u64* s_lo, const u64* s_hi, int ns, u64* dest_lo, u32* val,
                    cudaStream_t st) {
  if (n == 0) return;
  int g = grid_for(n, 256);
  if (KW == 2) klaunch(k_partition_dest<2>, g, 256, 0, st, kd, n, s_lo, s_hi, ns, dest_lo, val);
  else klaunch(k_partition_dest<1>, g, 256, 0, st, kd, n, s_lo, s_hi, ns, dest_lo, val);
}

template <typename T>
__global__ void k_gather(const T* __restrict__ src, const u32* __restrict__ perm, u32 n, T* __restrict__ dst) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[perm[i]];
}

void gather_column(const void* src, int elem_bytes, const u32* perm, u32 n, void* dst, cudaStream_t st) {
  if (n == 0) return;
  int g = grid_for(n, 256);
  switch (elem_bytes) {
    case 1: klaunch(k_gather<unsigned char>, g, 256, 0, st, (const unsigned char*)src, perm, n, (unsigned char*)dst); break;
    case 2: klaunch(k_gather<unsigned short>, g, 256, 0, st, (const unsigned short*)src, perm, n, (unsigned short*)dst); break;
    case 4: klaunch(k_gather<unsigned int>, g, 256, 0, st, (const unsigned int*)src, perm, n, (unsigned int*)dst); break;
    default: klaunch(k_gather<u64>, g, 256, 0, st, (const u64*)src, perm, n, (u64*)dst); break;
  }
}

// Fused exchange: row i of the destination-sorted order (perm[i] = source
// row, dest[i] = destination rank) is gathered from the local columns and
// stored straight into the destination rank's receive columns (peer memory
// over NVLink / NVSwitch), at peer_off[d] + (i - seg_start[d]).
__global__ void k_scatter_peers(const PeerScatter ps, const u32* __restrict__ perm, const u64* __restrict__ dest,
                                u32 n, void* const* __restrict__ peer_cols, const u64* __restrict__ peer_off,
                                const u32* __restrict__ seg_start) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u32 d = (u32)dest[i];
    const u32 r = perm[i];
    const u64 o = peer_off[d] + (i - seg_start[d]);
    for (int c = 0; c < ps.ncols; ++c) {
      char* dst = (char*)peer_cols[(size_t)d * ps.ncols + c];
      const char* src = (const char*)ps.src[c];
      switch (ps.elem[c]) {
        case 1: ((unsigned char*)dst)[o] = ((const unsigned char*)src)[r]; break;
        case 2: ((unsigned short*)dst)[o] = ((const unsigned short*)src)[r]; break;
        case 4: ((unsigned int*)dst)[o] = ((const unsigned int*)src)[r]; break;
        default: ((u64*)dst)[o] = ((const u64*)src)[r]; break;
      }
    }
  }
}

void scatter_peers(const PeerScatter& ps, const u32* perm, const u64* dest, u32 n, void* const* peer_cols,
                   const u64* peer_off, const u32* seg_start, cudaStream_t st) {
  if (n) klaunch(k_scatter_peers, grid_for(n, 256), 256, 0, st, ps, perm, dest, n, peer_cols, peer_off, seg_start);
}

__global__ void k_count_dest(const u64* __restrict__ d, u32 n, int ndest, u32* __restrict__ counts) {
  // counts[k] = upper_bound(d, k) for the sorted destination array
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ndest) return;
  u32 l = 0, h = n;
  while (l < h) {
    u32 m = (l + h) >> 1;
    if (d[m] <= (u64)k) l = m + 1; else h = m;
  }
  counts[k] = l;
}

void count_dest(const u64* dest_sorted, u32 n, int ndest, u32* counts, cudaStream_t st) {
  klaunch(k_count_dest, 1, 256, 0, st, dest_sorted, n, ndest, counts);
}

}  // namespace isa
