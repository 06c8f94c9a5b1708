// Wide merge by key-range tiles: one pass over the runs, k-way merge and
// duplicate combination inside shared memory.
//
// Reference: wide_merge + forecasting LoserTree + strict watermark
// (sortagg.py:588-674, losertree.py:29-135, memindex.py:265-273): all runs
// are merged in one step and a key is emitted, aggregated over every run,
// once no run can still hold it.  On the GPU the key space is cut into
// tiles small enough for shared memory; a tile's rows are, in every run, one
// contiguous segment, so a CTA loads the k segments, merges them (stable
// radix sort of the tile's rows on the key bits that vary inside the tile,
// ties kept in run order), combines equal keys (Schema.merge_states,
// core.py:184-208) and writes the groups straight to their final place in
// the result (decoupled look-back over the tiles' group counts).  Every run
// row is read once and every group written once.
//
// Tiles come from run directories.  A monotone bucket function beta(key) =
// clamp((key - g) >> shift, 0, nb - 1), fixed per execute, cuts the key
// space into nb buckets; every run gets a directory dir[b] = first row whose
// bucket is >= b (a pass over the run when it is spilled, isa_engine.cu).
// Transposed to D[b][r] and summed over runs (P[b] = rows below bucket b),
// the directories give exact per-run positions of every bucket boundary:
// windows and tiles are bucket ranges, no search over the runs is needed.
#include "isa_kernels.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace isa {

__device__ __forceinline__ u32 bucket_of(const Bucketing& bk, u64 hi, u64 lo) {
  if (hi < bk.g_hi || (hi == bk.g_hi && lo < bk.g_lo)) return 0;
  const u64 dlo = lo - bk.g_lo;
  const u64 dhi = hi - bk.g_hi - (lo < bk.g_lo ? 1ull : 0ull);
  const int s = bk.shift;
  u64 qlo, qhi;
  if (s >= 64) { qlo = dhi >> (s - 64); qhi = 0; }
  else if (s == 0) { qlo = dlo; qhi = dhi; }
  else { qlo = (dlo >> s) | (dhi << (64 - s)); qhi = dhi >> s; }
  if (qhi || qlo >= (u64)bk.nb) return bk.nb - 1;
  return (u32)qlo;
}

// dir[b] (b in [0, nb]) = first row i of a sorted run with bucket(key_i) >= b
// (n when none): row i owns the buckets (bucket(i - 1), bucket(i)], the
// last row also (bucket(n - 1), nb].  Short ranges are written by the row's
// thread; long ones (the empty margins below the first and above the last
// key, gaps in clustered key sets) go to a list that a second kernel fills
// with whole CTAs, so no thread writes more than DIR_INLINE entries.
#define DIR_INLINE 32
#define DIR_GAP_CAP (1u << 16)
struct DirGap { u32 q0, q1, v, pad; };   // dir[q0 .. q1) = v

template <int KW>
__global__ void k_dir_build(const u64* __restrict__ lo, const u64* __restrict__ hi, u32 n, Bucketing bk,
                            u32* __restrict__ dir, DirGap* __restrict__ gaps, u32* __restrict__ ngaps, u32 gap_cap) {
  auto emit = [&](u32 q0, u32 q1, u32 v) {   // dir[q0, q1) = v
    if (q1 <= q0) return;
    if (q1 - q0 <= DIR_INLINE) {
      for (u32 q = q0; q < q1; ++q) dir[q] = v;
      return;
    }
    const u32 g = atomicAdd(ngaps, 1u);
    if (g < gap_cap) gaps[g] = DirGap{q0, q1, v, 0u};
    else for (u32 q = q0; q < q1; ++q) dir[q] = v;   // list full: slow but correct
  };
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u32 b = bucket_of(bk, KW == 2 ? hi[i] : 0, lo[i]);
    const u32 q0 = i == 0 ? 0u : bucket_of(bk, KW == 2 ? hi[i - 1] : 0, lo[i - 1]) + 1;
    emit(q0, b + 1, i);
    if (i == n - 1) emit(b + 1, bk.nb + 1, n);
  }
}

// one CTA per listed range (grid-stride over the list)
__global__ void k_dir_gaps(u32* __restrict__ dir, const DirGap* __restrict__ gaps, const u32* __restrict__ ngaps,
                           u32 gap_cap) {
  const u32 ng = min(*ngaps, gap_cap);
  for (u32 g = blockIdx.x; g < ng; g += gridDim.x) {
    const DirGap d = gaps[g];
    for (u32 q = d.q0 + threadIdx.x; q < d.q1; q += blockDim.x) dir[q] = d.v;
  }
}

__global__ void k_fill_u32(u32* __restrict__ p, u32 n, u32 v) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

size_t dir_tmp_bytes() { return 16 + (size_t)DIR_GAP_CAP * sizeof(DirGap); }

void dir_build(int KW, const u64* lo, const u64* hi, u32 n, const Bucketing& bk, u32* dir, void* tmp,
               cudaStream_t st) {
  if (n == 0) {
    klaunch(k_fill_u32, std::min<u32>((bk.nb + 256) / 256, 148u * 16u), 256, 0, st, dir, bk.nb + 1, 0u);
    return;
  }
  u32* ngaps = (u32*)tmp;
  DirGap* gaps = (DirGap*)((char*)tmp + 16);
  cudaMemsetAsync(ngaps, 0, sizeof(u32), st);
  const int g = (int)std::min<u32>((n + 255) / 256, 148u * 16u);
  if (KW == 2) klaunch(k_dir_build<2>, g, 256, 0, st, lo, hi, n, bk, dir, gaps, ngaps, (u32)DIR_GAP_CAP);
  else klaunch(k_dir_build<1>, g, 256, 0, st, lo, hi, n, bk, dir, gaps, ngaps, (u32)DIR_GAP_CAP);
  klaunch(k_dir_gaps, 148 * 2, 256, 0, st, dir, (const DirGap*)gaps, (const u32*)ngaps, (u32)DIR_GAP_CAP);
}

// D[b * k + r] = dirs[r][b]: 32 x 32 tiles through shared memory
__global__ void k_dir_transpose(u32* const* __restrict__ dirs, int k, u32 nb1, u32* __restrict__ D) {
  __shared__ u32 t[32][33];
  const u32 b0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const u32 r = r0 + y, b = b0 + threadIdx.x;
    t[y][threadIdx.x] = (r < (u32)k && b < nb1) ? dirs[r][b] : 0u;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const u32 b = b0 + y, r = r0 + threadIdx.x;
    if (b < nb1 && r < (u32)k) D[(size_t)b * k + r] = t[threadIdx.x][y];
  }
}

// P[b] = sum over runs of D[b][r] (= rows with bucket < b): one warp per bucket
__global__ void k_dir_rowsum(const u32* __restrict__ D, int k, u32 nb1, u64* __restrict__ P) {
  const u32 lane = threadIdx.x & 31;
  for (u32 b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb1; b += (gridDim.x * blockDim.x) >> 5) {
    u64 s = 0;
    for (int r = lane; r < k; r += 32) s += D[(size_t)b * k + r];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) P[b] = s;
  }
}

void dir_transpose(u32* const* dirs_dev, int k, u32 nb1, u32* D, cudaStream_t st) {
  dim3 grid((nb1 + 31) / 32, (k + 31) / 32);
  klaunch(k_dir_transpose, grid, dim3(32, 8), 0, st, dirs_dev, k, nb1, D);
}

void dir_rowsum(const u32* D, int k, u32 nb1, u64* P, cudaStream_t st) {
  const int g = (int)std::min<u32>((nb1 + 7) / 8, 148u * 32u);
  klaunch(k_dir_rowsum, g, 256, 0, st, D, k, nb1, P);
}

// ------------------------------------------------------------ tile merge --
#define TM_THREADS 256
#define TM_WARPS (TM_THREADS / 32)
#define TM_MAX_IT 16                      // items per warp lane per radix pass
#define TM_MAX_CAP (TM_THREADS * TM_MAX_IT)

__device__ __forceinline__ u64 tm_ld(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void tm_st(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// first b in [lo, hi] with P[b] >= v (hi when none)
__device__ __forceinline__ u32 p_lower_bound(const u64* __restrict__ P, u32 lo, u32 hi, u64 v) {
  while (lo < hi) {
    const u32 m = (lo + hi) >> 1;
    if (P[m] < v) lo = m + 1; else hi = m;
  }
  return lo;
}

// Per row: key words, states, two u32 sort words, u32 group id, u8 head.
size_t tile_merge_smem(int KW, int S, int k, u32 cap) {
  return (size_t)cap * (8 * KW + 8 * S + 4 + 4 + 4 + 1) + 16 + (size_t)(k + 1) * 4 + (size_t)k * 8 + 16 +
         TM_WARPS * 256 * 4 + 256 * 4 + 64;
}

u32 tile_merge_cap(int KW, int S, int k) {
  // three CTAs per SM: ~64 KB of shared memory each (measured: 100 KB 88 ms, 64 KB 70 ms, 44 KB 90 ms
  // per 1e9 config-5 rows; ISA_TM_SMEM_KB overrides)
  static int kb = -1;
  if (kb < 0) { const char* e = getenv("ISA_TM_SMEM_KB"); kb = e ? std::max(16, std::min(200, atoi(e))) : 64; }
  const size_t budget = (size_t)kb * 1024;
  const size_t fixed = tile_merge_smem(KW, S, k, 0);
  if (fixed >= budget) return 0;
  size_t cap = (budget - fixed) / (size_t)(8 * KW + 8 * S + 13);
  cap = std::min<size_t>(cap, TM_MAX_CAP);
  return (u32)(cap & ~(size_t)255);
}

// (key - base) >> sh, 128-bit difference (KW == 1: hi words are 0)
template <int KW>
__device__ __forceinline__ u64 tm_off(u64 h, u64 l, u64 bh, u64 bl, int sh) {
  if (KW == 1) return sh >= 64 ? 0 : ((l - bl) >> sh);
  const u64 dl = l - bl, dh = h - bh - (l < bl ? 1ull : 0ull);
  if (sh >= 64) return dh >> (sh - 64);
  if (sh == 0) return dl;
  return (dl >> sh) | (dh << (64 - sh));
}

// One stable LSD pass over the tile's u32 sort words.  Rows are split into
// warp-contiguous ranges of WI (a multiple of 32); every warp walks its
// range in order, ranking 32 rows per step with MATCH.ANY and per-warp digit
// counters, and keeps (digit, rank) per row in `scratch`; after the
// per-digit scan the same warp scatters its rows.  Rolled loops: the cost
// follows the tile's rows, not its capacity.
template <typename DigitFn>
__device__ __forceinline__ void tm_pass(const u32* __restrict__ cur, u32* __restrict__ nxt, u32* __restrict__ scratch,
                                        u32 n, u32 WI, u32* wcnt, u32* dstart, u32* sw, DigitFn digit) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const u32 lt = lanemask_lt();
  for (int q = lane; q < 256; q += 32) wcnt[w * 256 + q] = 0;
  __syncwarp();
  const u32 r0 = w * WI, r1 = min(n, r0 + WI);
  for (u32 i = r0 + lane; i < ((r1 + 31) & ~31u) && r0 < r1; i += 32) {
    const bool valid = i < r1;
    const u32 d = valid ? digit(cur[i]) : 256 + lane;
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
  {   // per digit: exclusive over warps, then over digits
    const int dg = tid;
    u32 run = 0;
#pragma unroll
    for (int ww = 0; ww < TM_WARPS; ++ww) {
      const u32 c = wcnt[ww * 256 + dg];
      wcnt[ww * 256 + dg] = run;
      run += c;
    }
    u32 tot;
    dstart[dg] = block_excl_scan256(run, sw, &tot);
  }
  __syncthreads();
  for (u32 i = r0 + lane; i < r1; i += 32) {
    const u32 v = scratch[i], d = v >> 16;
    nxt[dstart[d] + wcnt[w * 256 + d] + (v & 0xFFFFu)] = cur[i];
  }
  __syncthreads();
}

// One tile: rows of the k run segments [D[B0][r], D[B1][r]) loaded into
// shared memory (one thread per row, its segment found by binary search over
// the segment offsets), sorted stably by key, equal keys combined in run
// order, groups written at their final place in the result.
//
// Sort: the tile's key span comes from the segments' end rows (each segment
// is sorted).  Every row gets a u32 word (prefix << 12 | row), prefix = the
// top <= 20 bits of (key - min); an LSD radix sort of the words orders the
// tile exactly when the span fits 20 bits (dense keys: config 5) and up to
// runs of equal prefix otherwise (sparse keys: those runs are short and are
// finished by an insertion sort on the full key; a run longer than 64 makes
// the tile fall back to an LSD sort over every span bit).
template <int KW, int MS>
__global__ void __launch_bounds__(TM_THREADS, 3) k_tile_merge(TileMergeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const u32 cap = a.cap;
  const int S = a.sd.nslots;
  const int k = a.k;
  u64* klo = (u64*)smem;
  u64* khi = klo + cap;                                   // KW == 2
  u64* sst = klo + (size_t)cap * KW;                      // [cap][S]
  u32* wa = (u32*)(sst + (size_t)cap * S);
  u32* wb = wa + cap;
  u32* gid = wb + cap;
  unsigned char* head = (unsigned char*)(gid + cap);
  u32* seg_off = (u32*)(((uintptr_t)(head + cap) + 15) & ~(uintptr_t)15);   // [k + 1]
  i64* seg_src = (i64*)(((uintptr_t)(seg_off + k + 1) + 15) & ~(uintptr_t)15);   // [k] run row of the segment's first row
  u32* wcnt = (u32*)(seg_src + k);                        // [TM_WARPS][256]
  u32* dstart = wcnt + TM_WARPS * 256;                    // [256]
  __shared__ u32 s_j, s_B0, s_B1, s_n, s_base, s_bits, s_long;
  __shared__ u32 sw[TM_WARPS];
  __shared__ u64 s_min_lo[TM_WARPS], s_min_hi[TM_WARPS], s_max_lo[TM_WARPS], s_max_hi[TM_WARPS];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    const u32 j = atomicAdd(a.ticket, 1u);
    s_j = j;
    s_B0 = a.tb[j];
    s_B1 = a.tb[j + 1];
    s_long = 0;
  }
  __syncthreads();
  const u32 j = s_j, B0 = s_B0, B1 = s_B1;

  // ---- segments: run r contributes rows [D[B0][r], D[B1][r])
  {
    u32 carry = 0;
    for (int r0 = 0; r0 < k; r0 += TM_THREADS) {
      const int r = r0 + tid;
      u32 len = 0;
      if (r < k) {
        const u32 s0 = a.D[(size_t)B0 * k + r], s1 = a.D[(size_t)B1 * k + r];
        len = s1 - s0;
        seg_src[r] = (i64)s0;
      }
      u32 tot;
      const u32 ex = block_excl_scan256(len, sw, &tot);
      if (r < k) seg_off[r] = carry + ex;
      carry += tot;
    }
    if (tid == 0) { seg_off[k] = carry; s_n = carry; }
  }
  __syncthreads();
  const u32 n = s_n;
  const bool over = n > cap;
  if (over && tid == 0) atomicExch(a.overflow, 1u);

  u32 ng = 0;
  unsigned char exact = 1;
  u32* cur = wa;
  if (!over && n > 0) {
    // ---- load: one thread per row (LU rows in flight per thread); raw rows
    //      are read where they are, packed HBM runs decoded in place
    constexpr int LU = MS <= 2 ? 4 : (MS <= 5 ? 2 : 1);
    const int ncol = KW + S;
    for (u32 i0 = tid; i0 < n; i0 += LU * TM_THREADS) {
      int run[LU];
      u32 pos[LU];
#pragma unroll
      for (int u = 0; u < LU; ++u) {
        const u32 i = i0 + u * TM_THREADS;
        run[u] = -1;
        if (i < n) {
          int l = 0, h = k;   // last r with seg_off[r] <= i (a non-empty segment)
          while (h - l > 1) {
            const int m = (l + h) >> 1;
            if (seg_off[m] <= i) l = m; else h = m;
          }
          run[u] = l;
          pos[u] = (u32)(seg_src[l] + (i64)(i - seg_off[l]));
        }
      }
      u64 kl[LU], kh[LU], sv[LU][MS];
#pragma unroll
      for (int u = 0; u < LU; ++u) {
        if (run[u] < 0) continue;
        const MergeSrc* ms = a.src + run[u];
        const char* pk = ms->pk;
        if (pk) {
          const u64* h = (const u64*)(pk + ms->blk_off[pos[u] >> 10]);
          const u32 ip = pos[u] & 1023u;
          const u64* payload = h + 2 * ncol;
          kl[u] = h[0] + pk_extract(payload + (h[1] >> 8), ip, (u32)(h[1] & 0xFF));
          if (KW == 2) kh[u] = h[2] + pk_extract(payload + (h[3] >> 8), ip, (u32)(h[3] & 0xFF));
#pragma unroll
          for (int s = 0; s < MS; ++s)
            if (s < S) {
              const u64 b = h[2 * (KW + s)], m = h[2 * (KW + s) + 1];
              sv[u][s] = pk_inv(b + pk_extract(payload + (m >> 8), ip, (u32)(m & 0xFF)), (a.fmask >> s) & 1u, 0);
            }
        } else {
          const i64 x = ms->off + (i64)pos[u];
          kl[u] = ms->lo[x];
          if (KW == 2) kh[u] = ms->hi[x];
#pragma unroll
          for (int s = 0; s < MS; ++s)
            if (s < S) sv[u][s] = ms->st[(size_t)x * S + s];
        }
      }
#pragma unroll
      for (int u = 0; u < LU; ++u) {
        if (run[u] < 0) continue;
        const u32 i = i0 + u * TM_THREADS;
        klo[i] = kl[u];
        if (KW == 2) khi[i] = kh[u];
#pragma unroll
        for (int s = 0; s < MS; ++s)
          if (s < S) sst[(size_t)i * S + s] = sv[u][s];
      }
    }
    __syncthreads();
    // ---- key span: min of the segments' first rows, max of their last rows
    u64 mnl = ~0ull, mnh = KW == 2 ? ~0ull : 0, mxl = 0, mxh = 0;
    for (int r = tid; r < k; r += TM_THREADS) {
      const u32 o0 = seg_off[r], o1 = seg_off[r + 1];
      if (o1 == o0) continue;
      const u64 l0 = klo[o0], h0 = KW == 2 ? khi[o0] : 0, l1 = klo[o1 - 1], h1 = KW == 2 ? khi[o1 - 1] : 0;
      if (key_less<KW>(h0, l0, mnh, mnl)) { mnh = h0; mnl = l0; }
      if (key_less<KW>(mxh, mxl, h1, l1)) { mxh = h1; mxl = l1; }
    }
    for (int o = 16; o; o >>= 1) {
      const u64 al = __shfl_xor_sync(0xffffffffu, mnl, o), ah = __shfl_xor_sync(0xffffffffu, mnh, o);
      if (key_less<KW>(ah, al, mnh, mnl)) { mnh = ah; mnl = al; }
      const u64 bl = __shfl_xor_sync(0xffffffffu, mxl, o), bh = __shfl_xor_sync(0xffffffffu, mxh, o);
      if (key_less<KW>(mxh, mxl, bh, bl)) { mxh = bh; mxl = bl; }
    }
    if (lane == 0) { s_min_lo[w] = mnl; s_min_hi[w] = mnh; s_max_lo[w] = mxl; s_max_hi[w] = mxh; }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < TM_WARPS; ++q) {
        if (key_less<KW>(s_min_hi[q], s_min_lo[q], mnh, mnl)) { mnh = s_min_hi[q]; mnl = s_min_lo[q]; }
        if (key_less<KW>(mxh, mxl, s_max_hi[q], s_max_lo[q])) { mxh = s_max_hi[q]; mxl = s_max_lo[q]; }
      }
      s_min_lo[0] = mnl; s_min_hi[0] = mnh;
      const u64 dl = mxl - mnl, dh = mxh - mnh - (mxl < mnl ? 1ull : 0ull);
      s_bits = dh ? 128 - __clzll((long long)dh) : (dl ? 64 - __clzll((long long)dl) : 0);
    }
    __syncthreads();
    const u64 bl = s_min_lo[0], bh = s_min_hi[0];
    const int bits = (int)s_bits;
    const int pb = bits < a.pbits ? bits : a.pbits;   // prefix bits (20; tests lower it)
    const int psh = bits - pb;              // prefix = (key - min) >> psh
    exact = psh == 0;
    for (u32 i = tid; i < n; i += TM_THREADS)
      wa[i] = ((u32)tm_off<KW>(KW == 2 ? khi[i] : 0, klo[i], bh, bl, psh) << 12) | i;
    __syncthreads();
    const u32 WI = (((n + TM_WARPS - 1) / TM_WARPS) + 31) & ~31u;   // rows per warp, in order
    u32* nxt = wb;
    for (int sh = 12; sh < 12 + pb; sh += 8) {
      tm_pass(cur, nxt, gid, n, WI, wcnt, dstart, sw, [sh](u32 x) { return (x >> sh) & 0xFFu; });
      u32* t = cur; cur = nxt; nxt = t;
    }
    const u32 ipt = (n + TM_THREADS - 1) / TM_THREADS;
    const u32 i0 = min(n, tid * ipt), i1 = min(n, i0 + ipt);
    if (!exact) {
      // runs of equal prefix starting in this thread's range: insertion sort
      // by the full key (stable: ties keep their order)
      for (u32 s0 = i0; s0 < i1; ++s0) {
        const u32 pfx = cur[s0] >> 12;
        if (s0 > 0 && (cur[s0 - 1] >> 12) == pfx) continue;   // not a run start
        u32 e = s0 + 1;
        while (e < n && (cur[e] >> 12) == pfx) ++e;
        if (e - s0 < 2) continue;
        if (e - s0 > 64) { s_long = 1; continue; }
        for (u32 x = s0 + 1; x < e; ++x) {
          const u32 v = cur[x];
          const u32 vi = v & 0xFFFu;
          const u64 vl = klo[vi], vh = KW == 2 ? khi[vi] : 0;
          u32 y = x;
          while (y > s0) {
            const u32 ui = cur[y - 1] & 0xFFFu;
            if (!key_less<KW>(vh, vl, KW == 2 ? khi[ui] : 0, klo[ui])) break;
            cur[y] = cur[y - 1];
            --y;
          }
          cur[y] = v;
        }
      }
      __syncthreads();
      if (s_long) {
        // a long run of equal prefix: LSD over every span bit (keys read
        // through the row index), starting from the prefix order
        for (int sh = 0; sh < bits; sh += 8) {
          tm_pass(cur, nxt, gid, n, WI, wcnt, dstart, sw, [&](u32 x) {
            const u32 xi = x & 0xFFFu;
            return (u32)tm_off<KW>(KW == 2 ? khi[xi] : 0, klo[xi], bh, bl, sh) & 0xFFu;
          });
          u32* t = cur; cur = nxt; nxt = t;
        }
      }
    }
    // ---- heads + group ids (thread-contiguous items, block scan of counts)
    u32 c = 0;
    for (u32 i = i0; i < i1; ++i) {
      bool hd = i == 0;
      if (!hd) {
        const u32 x = cur[i], y = cur[i - 1];
        if (exact) {
          hd = (x >> 12) != (y >> 12);
        } else {
          const u32 xi = x & 0xFFFu, yi = y & 0xFFFu;
          hd = !key_eq<KW>(KW == 2 ? khi[xi] : 0, klo[xi], KW == 2 ? khi[yi] : 0, klo[yi]);
        }
      }
      head[i] = hd ? 1 : 0;
      c += hd ? 1u : 0u;
    }
    u32 tot;
    u32 g = block_excl_scan256(c, sw, &tot);
    for (u32 i = i0; i < i1; ++i) {
      gid[i] = g;
      g += head[i];
    }
    ng = tot;
  }
  // ---- decoupled look-back over the tiles' group counts
  if (w == 0) {
    const u64 E = (u64)a.epoch << 34;
    u32 excl = 0;
    if (j == 0) {
      if (lane == 0) tm_st(a.status, E | (2ull << 32) | ng);
    } else {
      if (lane == 0) tm_st(a.status + j, E | (1ull << 32) | ng);
      int jj = (int)j - 1;
      for (;;) {
        const int q = jj - lane;
        const u64 x = q >= 0 ? tm_ld(a.status + q) : (E | (2ull << 32));
        if (!__all_sync(0xffffffffu, (x >> 34) == (u64)a.epoch)) continue;
        const u32 inc = __ballot_sync(0xffffffffu, ((x >> 32) & 3u) == 2u);
        const int first = inc ? __ffs(inc) - 1 : 32;
        u32 v = lane <= first ? (u32)x : 0u;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        jj -= 32;
      }
      if (lane == 0) tm_st(a.status + j, E | (2ull << 32) | (excl + ng));
    }
    if (lane == 0) {
      s_base = excl;
      if (j + 1 == a.ntiles) *a.total = excl + ng;
    }
  }
  __syncthreads();
  if (over || n == 0) return;
  // ---- groups: the head's thread combines the group's rows in order
  const u32 base = s_base;
  for (u32 i = tid; i < n; i += TM_THREADS) {
    if (!head[i]) continue;
    const u32 o = base + gid[i];
    const u32 x = cur[i] & 0xFFFu;
    a.out_lo[o] = klo[x];
    if (KW == 2) a.out_hi[o] = khi[x];
    if (S) {
      u64 acc[MS];
#pragma unroll
      for (int s = 0; s < MS; ++s)
        if (s < S) acc[s] = sst[(size_t)x * S + s];
      for (u32 jn = i + 1; jn < n && !head[jn]; ++jn) {
        const u32 y = cur[jn] & 0xFFFu;
#pragma unroll
        for (int s = 0; s < MS; ++s)
          if (s < S) acc[s] = combine_slot(a.sd.op[s], a.sd.type[s], acc[s], sst[(size_t)y * S + s]);
      }
#pragma unroll
      for (int s = 0; s < MS; ++s)
        if (s < S) a.out_st[(size_t)o * S + s] = acc[s];
    }
  }
}

// tile j of the window = buckets [tb[j], tb[j + 1]): tb[j] = first bucket
// whose P reaches P[b_lo] + j * target (one thread per bound)
__global__ void k_tile_bounds(const u64* __restrict__ P, u32 b_lo, u32 b_hi, u32 target, u32 ntiles,
                              u32* __restrict__ tb) {
  const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > ntiles) return;
  const u64 p0 = P[b_lo];
  tb[j] = j == 0 ? b_lo : (j == ntiles ? b_hi : p_lower_bound(P, b_lo, b_hi, p0 + (u64)j * target));
}

static std::atomic<u32> g_tm_epoch{0};

template <int KW, int MS>
static void tm_launch(TileMergeArgs& a, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(k_tile_merge<KW, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
  klaunch(k_tile_merge<KW, MS>, a.ntiles, TM_THREADS, smem, st, a);
}

void tile_merge(int KW, TileMergeArgs& a, cudaStream_t st) {
  if (a.ntiles == 0) return;
  a.epoch = (g_tm_epoch.fetch_add(1) % 0x3FFFFFFEu) + 1u;
  // ISA_TM_PREFIX_BITS (1..20, tests): fewer prefix bits exercise the
  // insertion-sort finish and the full-width fallback on ordinary inputs
  const char* e = getenv("ISA_TM_PREFIX_BITS");
  a.pbits = e ? std::max(1, std::min(20, atoi(e))) : 20;
  cudaMemsetAsync(a.ticket, 0, sizeof(u32), st);
  klaunch(k_tile_bounds, (a.ntiles + 256) / 256, 256, 0, st, a.P, a.b_lo, a.b_hi, a.target, a.ntiles, a.tb);
  const size_t smem = tile_merge_smem(KW, a.sd.nslots, a.k, a.cap);
  const int S = a.sd.nslots;
#define TM_KW(K)                                   \
  do {                                             \
    if (S <= 1) tm_launch<K, 1>(a, smem, st);      \
    else if (S <= 2) tm_launch<K, 2>(a, smem, st); \
    else if (S <= 4) tm_launch<K, 4>(a, smem, st); \
    else if (S <= 5) tm_launch<K, 5>(a, smem, st); \
    else if (S <= 8) tm_launch<K, 8>(a, smem, st); \
    else tm_launch<K, 16>(a, smem, st);            \
  } while (0)
  if (KW == 2) TM_KW(2);
  else TM_KW(1);
#undef TM_KW
}

}  // namespace isa
