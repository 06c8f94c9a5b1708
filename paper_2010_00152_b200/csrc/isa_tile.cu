// K1: tile-local pre-aggregation (early aggregation of a batch "in cache",
// PAPER.md:689; the collapse of sortagg.py:195-228 applied per tile).
//
// One CTA per tile of TC_TILE consecutive rows.  Rows are grouped by key
// through a shared-memory hash table (insertion in synchronized rounds, so
// no partially published key is ever read), each group's state is combined
// with shared-memory atomics, and the tile's groups are written to a
// slotted layout: group g of tile t lives at index t * TC_TILE + g, with
// its key, its first row (chunk-relative, exact) and its state.  The sort
// path then sorts only the groups (stable, so a key's groups stay in tile =
// row order) and gathers states through the slotted index.
#include "isa_kernels.h"

namespace isa {

#define TC_THREADS 256
#define TC_ROWS 4
#define TC_TILE (TC_THREADS * TC_ROWS)   // 1024
#define TC_HASH (2 * TC_TILE)
#define TC_EMPTY 0xFFFFFFFFu
#define TC_CLAIM 0xFFFFFFFEu

__device__ __forceinline__ u32 tc_hash(u64 hi, u64 lo) {
  u64 x = lo ^ (hi * 0x9E3779B97F4A7C15ull);
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 29;
  return (u32)x & (TC_HASH - 1);
}

__device__ __forceinline__ void tc_atomic_shared(u64* addr, int op, int type, u64 v) {
  if (type == ST_I64) {
    if (op == OP_ADD) atomicAdd((unsigned long long*)addr, (unsigned long long)v);
    else if (op == OP_MIN) atomicMin((long long*)addr, (long long)v);
    else atomicMax((long long*)addr, (long long)v);
    return;
  }
  if (op == OP_ADD) { atomicAdd((double*)addr, u2d(v)); return; }
  unsigned long long old = *(volatile unsigned long long*)addr, assumed;
  do {
    assumed = old;
    u64 nv = combine_slot(op, type, assumed, v);
    if (nv == assumed) break;
    old = atomicCAS((unsigned long long*)addr, assumed, (unsigned long long)nv);
  } while (old != assumed);
}

template <int KW, int MS>
__global__ void __launch_bounds__(TC_THREADS) k_tile_collapse(KeyDesc kd, SlotDesc sd, i64 row0, u32 n,
                                                             u64* __restrict__ g_lo, u64* __restrict__ g_hi,
                                                             u32* __restrict__ g_first, u64* __restrict__ g_st,
                                                             u32* __restrict__ g_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  u32* tag = (u32*)smem;                          // [TC_HASH]
  u64* s_lo = (u64*)(tag + TC_HASH);              // [TC_TILE]
  u64* s_hi = s_lo + TC_TILE;                     // [TC_TILE] (KW == 2)
  u32* s_first = (u32*)(s_lo + KW * TC_TILE);     // [TC_TILE]
  u64* s_st = (u64*)(s_first + TC_TILE);          // [TC_TILE * S]
  __shared__ u32 s_ngroups;
  const int S = sd.nslots;
  const int tid = threadIdx.x;
  const u32 tile = blockIdx.x;
  const u32 base = tile * TC_TILE;
  const u32 lim = n > base ? n - base : 0;

  for (int i = tid; i < TC_HASH; i += TC_THREADS) tag[i] = TC_EMPTY;
  if (tid == 0) s_ngroups = 0;

  u64 kl[TC_ROWS], kh[TC_ROWS];
  u64 st[TC_ROWS][MS];
  u32 h[TC_ROWS], gid[TC_ROWS];
  bool pend[TC_ROWS];
#pragma unroll
  for (int k = 0; k < TC_ROWS; ++k) {
    const u32 r = k * TC_THREADS + tid;
    pend[k] = r < lim;
    kl[k] = kh[k] = 0;
    gid[k] = 0;
    if (pend[k]) {
      load_key(kd, row0 + base + r, kh[k], kl[k]);
#pragma unroll
      for (int s = 0; s < MS; ++s)
        if (s < S) {
          const int a = sd.alias[s];
          u64 x = 0;
#pragma unroll
          for (int q = 0; q < s; ++q)
            if (q == a) x = st[k][q];
          st[k][s] = a >= 0 ? x : load_slot_value(sd.src[s], sd.type[s], sd.dtype[s], sd.ptr[s], row0 + base + r);
        }
    }
    h[k] = tc_hash(kh[k], kl[k]);
  }
  __syncthreads();
  // insertion rounds: claim empty slots, publish, then compare
  for (;;) {
    bool won[TC_ROWS];
#pragma unroll
    for (int k = 0; k < TC_ROWS; ++k) {
      won[k] = false;
      if (pend[k] && tag[h[k]] == TC_EMPTY) won[k] = atomicCAS(&tag[h[k]], TC_EMPTY, TC_CLAIM) == TC_EMPTY;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TC_ROWS; ++k) {
      if (won[k]) {
        const u32 g = atomicAdd(&s_ngroups, 1u);
        s_lo[g] = kl[k];
        if (KW == 2) s_hi[g] = kh[k];
        s_first[g] = k * TC_THREADS + tid;
#pragma unroll
        for (int s = 0; s < MS; ++s)
          if (s < S) s_st[(size_t)g * S + s] = st[k][s];
        tag[h[k]] = g;
        gid[k] = g;
        pend[k] = false;
      }
    }
    __syncthreads();
    bool any = false;
#pragma unroll
    for (int k = 0; k < TC_ROWS; ++k) {
      if (pend[k]) {
        const u32 t = tag[h[k]];
        if (t < TC_CLAIM && key_eq<KW>(kh[k], kl[k], KW == 2 ? s_hi[t] : 0, s_lo[t])) {
          gid[k] = t;
          pend[k] = false;
          atomicMin(&s_first[t], k * TC_THREADS + tid);
#pragma unroll
          for (int s = 0; s < MS; ++s)
            if (s < S) tc_atomic_shared(&s_st[(size_t)t * S + s], sd.op[s], sd.type[s], st[k][s]);
        } else if (t < TC_CLAIM) {
          h[k] = (h[k] + 1) & (TC_HASH - 1);   // occupied by another key: probe on
        }
        any |= pend[k];
      }
    }
    if (!__syncthreads_or(any)) break;
  }
  __syncthreads();
  const u32 ng = s_ngroups;
  const size_t ob = (size_t)tile * TC_TILE;
  for (u32 g = tid; g < ng; g += TC_THREADS) {
    g_lo[ob + g] = s_lo[g];
    if (KW == 2) g_hi[ob + g] = s_hi[g];
    g_first[ob + g] = base + s_first[g];
    for (int s = 0; s < S; ++s) g_st[(ob + g) * S + s] = s_st[(size_t)g * S + s];
  }
  if (tid == 0) g_count[tile] = ng;
}

static size_t tc_smem(int KW, int S) {
  return (size_t)TC_HASH * 4 + (size_t)TC_TILE * (8 * KW + 4 + 8 * S);
}

template <int KW, int MS>
static void tc_launch(const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, u64* g_lo, u64* g_hi, u32* g_first,
                      u64* g_st, u32* g_count, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(k_tile_collapse<KW, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem(2, 16));
  const u32 tiles = (n + TC_TILE - 1) / TC_TILE;
  klaunch(k_tile_collapse<KW, MS>, tiles, TC_THREADS, tc_smem(KW, sd.nslots), st, kd, sd, row0, n, g_lo, g_hi, g_first,
          g_st, g_count);
}

u32 tile_rows() { return TC_TILE; }

void tile_collapse(int KW, const KeyDesc& kd, const SlotDesc& sd, int64_t row0, u32 n, u64* g_lo, u64* g_hi,
                   u32* g_first, u64* g_st, u32* g_count, cudaStream_t st) {
  if (n == 0) return;
  const int S = sd.nslots;
#define TCL(K, M) tc_launch<K, M>(kd, sd, row0, n, g_lo, g_hi, g_first, g_st, g_count, st)
  if (KW == 2) {
    if (S <= 1) TCL(2, 1); else if (S <= 2) TCL(2, 2); else if (S <= 4) TCL(2, 4); else if (S <= 8) TCL(2, 8); else TCL(2, 16);
  } else {
    if (S <= 1) TCL(1, 1); else if (S <= 2) TCL(1, 2); else if (S <= 4) TCL(1, 4); else if (S <= 8) TCL(1, 8); else TCL(1, 16);
  }
#undef TCL
}

// compact the slotted tile groups into the sort buffers: keys + value = slotted index
template <int KW>
__global__ void k_compact_groups(const u64* __restrict__ g_lo, const u64* __restrict__ g_hi,
                                 const u32* __restrict__ g_count, const u32* __restrict__ g_off, u64* __restrict__ lo,
                                 u64* __restrict__ hi, u32* __restrict__ val, u64* __restrict__ varying) {
  const u32 tile = blockIdx.x;
  const u32 cnt = g_count[tile], off = g_off[tile];
  const size_t ib = (size_t)tile * TC_TILE;
  const u64 r_lo = g_lo[0], r_hi = KW == 2 ? g_hi[0] : 0;   // tile 0 always holds >= 1 group
  u64 acc_lo = 0, acc_hi = 0;
  for (u32 g = threadIdx.x; g < cnt; g += blockDim.x) {
    const u64 l = g_lo[ib + g];
    lo[off + g] = l;
    acc_lo |= l ^ r_lo;
    if (KW == 2) {
      const u64 h2 = g_hi[ib + g];
      hi[off + g] = h2;
      acc_hi |= h2 ^ r_hi;
    }
    val[off + g] = (u32)(ib + g);
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

void compact_groups(int KW, const u64* g_lo, const u64* g_hi, const u32* g_count, const u32* g_off, u32 tiles,
                    u64* lo, u64* hi, u32* val, u64* varying, cudaStream_t st) {
  if (!tiles) return;
  if (KW == 2) klaunch(k_compact_groups<2>, tiles, 256, 0, st, g_lo, g_hi, g_count, g_off, lo, hi, val, varying);
  else klaunch(k_compact_groups<1>, tiles, 256, 0, st, g_lo, g_hi, g_count, g_off, lo, hi, val, varying);
}

}  // namespace isa
