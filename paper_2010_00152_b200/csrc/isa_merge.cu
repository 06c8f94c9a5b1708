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
// (n when none): row i writes the buckets (bucket(i - 1), bucket(i)], the
// last row also (bucket(n - 1), nb].
template <int KW>
__global__ void k_dir_build(const u64* __restrict__ lo, const u64* __restrict__ hi, u32 n, Bucketing bk,
                            u32* __restrict__ dir) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u32 b = bucket_of(bk, KW == 2 ? hi[i] : 0, lo[i]);
    const long long bp = i == 0 ? -1 : (long long)bucket_of(bk, KW == 2 ? hi[i - 1] : 0, lo[i - 1]);
    for (long long q = bp + 1; q <= (long long)b; ++q) dir[q] = i;
    if (i == n - 1)
      for (u32 q = b + 1; q <= bk.nb; ++q) dir[q] = n;
  }
}

__global__ void k_fill_u32(u32* __restrict__ p, u32 n, u32 v) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

void dir_build(int KW, const u64* lo, const u64* hi, u32 n, const Bucketing& bk, u32* dir, cudaStream_t st) {
  if (n == 0) {
    klaunch(k_fill_u32, (bk.nb + 256) / 256, 256, 0, st, dir, bk.nb + 1, 0u);
    return;
  }
  const int g = (int)std::min<u32>((n + 255) / 256, 148u * 16u);
  if (KW == 2) klaunch(k_dir_build<2>, g, 256, 0, st, lo, hi, n, bk, dir);
  else klaunch(k_dir_build<1>, g, 256, 0, st, lo, hi, n, bk, dir);
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

size_t tile_merge_smem(int KW, int S, int k, u32 cap) {
  // keys, states, two u16 order arrays, u32 group ids, u8 heads; segment
  // offsets (k + 1 u32) and sources (k i64); per-warp digit counters
  return (size_t)cap * (8 * KW + 8 * S + 2 + 2 + 4 + 1) + 16 + (size_t)(k + 1) * 4 + (size_t)k * 8 + 16 +
         TM_WARPS * 256 * 4 + 256 * 4 + 64;
}

u32 tile_merge_cap(int KW, int S, int k) {
  // two CTAs per SM: ~100 KB of shared memory each
  const size_t budget = 100 * 1024;
  const size_t fixed = tile_merge_smem(KW, S, k, 0);
  if (fixed >= budget) return 0;
  size_t cap = (budget - fixed) / (size_t)(8 * KW + 8 * S + 9);
  cap = std::min<size_t>(cap, TM_MAX_CAP);
  return (u32)(cap & ~(size_t)255);
}

template <int KW, int MS>
__global__ void __launch_bounds__(TM_THREADS, 2) k_tile_merge(TileMergeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const u32 cap = a.cap;
  const int S = a.sd.nslots;
  const int k = a.k;
  u64* klo = (u64*)smem;
  u64* khi = klo + cap;                                   // KW == 2
  u64* sst = klo + (size_t)cap * KW;                      // [cap][S]
  unsigned short* ord0 = (unsigned short*)(sst + (size_t)cap * S);
  unsigned short* ord1 = ord0 + cap;
  u32* gid = (u32*)(((uintptr_t)(ord1 + cap) + 15) & ~(uintptr_t)15);
  unsigned char* head = (unsigned char*)(gid + cap);
  u32* seg_off = (u32*)(((uintptr_t)(head + cap) + 15) & ~(uintptr_t)15);   // [k + 1]
  i64* seg_src = (i64*)(((uintptr_t)(seg_off + k + 1) + 15) & ~(uintptr_t)15);   // [k]
  u32* wcnt = (u32*)(seg_src + k);                        // [TM_WARPS][256]
  u32* dstart = wcnt + TM_WARPS * 256;                    // [256]
  __shared__ u32 s_j, s_B0, s_B1, s_n, s_ng, s_base, s_bits;
  __shared__ u32 sw[TM_WARPS];
  __shared__ u64 s_min_lo[TM_WARPS], s_min_hi[TM_WARPS], s_max_lo[TM_WARPS], s_max_hi[TM_WARPS];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    const u32 j = atomicAdd(a.ticket, 1u);
    s_j = j;
    const u64 p0 = a.P[a.b_lo];
    s_B0 = j == 0 ? a.b_lo : p_lower_bound(a.P, a.b_lo, a.b_hi, p0 + (u64)j * a.target);
    s_B1 = j + 1 >= a.ntiles ? a.b_hi : p_lower_bound(a.P, a.b_lo, a.b_hi, p0 + (u64)(j + 1) * a.target);
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
        seg_src[r] = a.base[r] + (i64)s0;
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
  if (!over && n > 0) {
    // ---- load the segments (one warp per segment: coalesced rows and states)
    for (int r = w; r < k; r += TM_WARPS) {
      const u32 o = seg_off[r], len = seg_off[r + 1] - o;
      if (!len) continue;
      const i64 src = seg_src[r];
      for (u32 i = lane; i < len; i += 32) {
        klo[o + i] = a.s_lo[src + i];
        if (KW == 2) khi[o + i] = a.s_hi[src + i];
      }
      if (S) {
        const u64* sp = a.s_st + (size_t)src * S;
        u64* dp = sst + (size_t)o * S;
        for (u32 q = lane; q < len * (u32)S; q += 32) dp[q] = sp[q];
      }
    }
    __syncthreads();
    // ---- key span of the tile: min, max -> bits that vary
    u64 mnl = ~0ull, mnh = KW == 2 ? ~0ull : 0, mxl = 0, mxh = 0;
    for (u32 i = tid; i < n; i += TM_THREADS) {
      const u64 l = klo[i], h = KW == 2 ? khi[i] : 0;
      if (key_less<KW>(h, l, mnh, mnl)) { mnh = h; mnl = l; }
      if (key_less<KW>(mxh, mxl, h, l)) { mxh = h; mxl = l; }
      ord0[i] = (unsigned short)i;
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
    const int npass = ((int)s_bits + 7) / 8;
    // ---- stable LSD radix sort of the row order on (key - min)
    unsigned short* cur = ord0;
    unsigned short* nxt = ord1;
    const u32 WI = (((n + TM_WARPS - 1) / TM_WARPS) + 31) & ~31u;   // rows per warp, in order
    const u32 lt = lanemask_lt();
    for (int p = 0; p < npass; ++p) {
      const int sh = 8 * p;
      for (int q = lane; q < 256; q += 32) wcnt[w * 256 + q] = 0;
      __syncwarp();
      u32 it_d[TM_MAX_IT], it_r[TM_MAX_IT];
      unsigned short it_x[TM_MAX_IT];
#pragma unroll
      for (int it = 0; it < TM_MAX_IT; ++it) {
        const u32 i = w * WI + it * 32 + lane;
        const bool in_w = (u32)it * 32 < WI;
        const bool valid = in_w && i < n;
        u32 d = 256 + lane;
        unsigned short x = 0;
        if (valid) {
          x = cur[i];
          const u64 l = klo[x];
          u64 v;
          if (KW == 2) {
            const u64 h = khi[x];
            const u64 dl = l - bl, dh = h - bh - (l < bl ? 1ull : 0ull);
            v = sh >= 64 ? (dh >> (sh - 64)) : (sh == 0 ? dl : ((dl >> sh) | (dh << (64 - sh))));
          } else {
            v = (l - bl) >> sh;
          }
          d = (u32)(v & 0xFFu);
        }
        it_d[it] = d;
        it_x[it] = x;
        if (in_w) {
          const u32 peers = __match_any_sync(0xffffffffu, d);
          const int leader = __ffs(peers) - 1;
          u32 c = 0;
          if (valid && lane == leader) {
            c = wcnt[w * 256 + d];
            wcnt[w * 256 + d] = c + __popc(peers);
          }
          c = __shfl_sync(0xffffffffu, c, leader);
          it_r[it] = c + __popc(peers & lt);
          __syncwarp();
        }
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
#pragma unroll
      for (int it = 0; it < TM_MAX_IT; ++it) {
        const u32 i = w * WI + it * 32 + lane;
        if ((u32)it * 32 < WI && i < n) {
          const u32 d = it_d[it];
          nxt[dstart[d] + wcnt[w * 256 + d] + it_r[it]] = it_x[it];
        }
      }
      __syncthreads();
      unsigned short* t = cur; cur = nxt; nxt = t;
    }
    // ---- heads + group ids (thread-contiguous items, block scan of counts)
    const u32 ipt = (n + TM_THREADS - 1) / TM_THREADS;
    const u32 i0 = min(n, tid * ipt), i1 = min(n, i0 + ipt);
    u32 c = 0;
    for (u32 i = i0; i < i1; ++i) {
      const unsigned short x = cur[i];
      bool hd = i == 0;
      if (!hd) {
        const unsigned short y = cur[i - 1];
        hd = !key_eq<KW>(KW == 2 ? khi[x] : 0, klo[x], KW == 2 ? khi[y] : 0, klo[y]);
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
  unsigned short* cur = (((s_bits + 7) / 8) & 1) ? ord1 : ord0;
  for (u32 i = tid; i < n; i += TM_THREADS) {
    if (!head[i]) continue;
    const u32 o = base + gid[i];
    const unsigned short x = cur[i];
    a.out_lo[o] = klo[x];
    if (KW == 2) a.out_hi[o] = khi[x];
    if (S) {
      u64 acc[MS];
#pragma unroll
      for (int s = 0; s < MS; ++s)
        if (s < S) acc[s] = sst[(size_t)x * S + s];
      for (u32 jn = i + 1; jn < n && !head[jn]; ++jn) {
        const unsigned short y = cur[jn];
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

static std::atomic<u32> g_tm_epoch{0};

template <int KW, int MS>
static void tm_launch(TileMergeArgs& a, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(k_tile_merge<KW, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  klaunch(k_tile_merge<KW, MS>, a.ntiles, TM_THREADS, smem, st, a);
}

void tile_merge(int KW, TileMergeArgs& a, cudaStream_t st) {
  if (a.ntiles == 0) return;
  a.epoch = (g_tm_epoch.fetch_add(1) % 0x3FFFFFFEu) + 1u;
  cudaMemsetAsync(a.ticket, 0, sizeof(u32), st);
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
