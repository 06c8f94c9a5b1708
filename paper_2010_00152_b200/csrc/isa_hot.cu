// Early aggregation against a large resident table (hash image of T).
//
// Reference: the ABSORBED branch of OrderedIndex.insert_or_aggregate
// (memindex.py:209-215): a row whose key is already resident is combined
// into the resident group in place and never reaches the run.  When the
// table is large (config 3: millions of groups, Zipf keys), most rows of a
// fill cycle hit it; sorting them with the misses (the plain chunk path) does
// the work of a sort for rows that need none.  Here:
//
//   1. k_hash_build: an open-addressing hash image of the sorted table T
//      (slot -> T index, the key copied into the slot), rebuilt whenever T
//      changed;
//   2. k_hot_probe: every row of the chunk looks its key up; hits record
//      their T index, misses go to a per-CTA list in row order (exactly the
//      rows the sort path then sorts: their keys are the chunk's new keys);
//   3. the flush analysis runs on the sorted misses, giving the flush row f
//      (the rows at and after f belong to the next fill cycle);
//   4. k_hot_absorb: the hits of rows before f are combined into T's states.
//      Each CTA privatizes the table rows its hits touch in a shared-memory
//      hash (heavy hitters combine in shared memory), then folds them into T
//      with one global atomic per (CTA, group, slot); rows that find no free
//      private slot combine into T directly.
//
// Result: identical fill cycles, runs and groups (integer states bit-exact;
// float sums combine in another order, within the stated tolerance).
#include "isa_kernels.h"

#include <algorithm>
#include <atomic>

namespace isa {

#define HB_EMPTY 0xFFFFFFFFu

__device__ __forceinline__ u32 hot_hash(u64 hi, u64 lo) {
  u64 x = lo ^ (hi * 0x9E3779B97F4A7C15ull);
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return (u32)x;
}

u32 hot_hash_capacity(u32 n) {
  u32 c = 1024;
  while (c < 2u * n && c < (1u << 31)) c <<= 1;
  return c;
}

template <int KW>
__global__ void k_hash_build(const u64* __restrict__ t_lo, const u64* __restrict__ t_hi, u32 n, HotHash h) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 lo = t_lo[i], hi = KW == 2 ? t_hi[i] : 0;
    u32 s = hot_hash(hi, lo) & h.mask;
    for (;;) {
      if (atomicCAS(h.idx + s, HB_EMPTY, i) == HB_EMPTY) {
        h.klo[s] = lo;
        if (KW == 2) h.khi[s] = hi;
        break;
      }
      s = (s + 1) & h.mask;
    }
  }
}

void hot_hash_build(int KW, const u64* t_lo, const u64* t_hi, u32 n, const HotHash& h, cudaStream_t st) {
  cudaMemsetAsync(h.idx, 0xFF, (size_t)(h.mask + 1) * 4, st);
  if (!n) return;
  const int g = (int)std::min<u32>((n + 255) / 256, 148u * 16u);
  if (KW == 2) klaunch(k_hash_build<2>, g, 256, 0, st, t_lo, t_hi, n, h);
  else klaunch(k_hash_build<1>, g, 256, 0, st, t_lo, (const u64*)nullptr, n, h);
}

template <int KW>
__device__ __forceinline__ u32 hot_lookup(const HotHash& h, u64 hi, u64 lo) {
  u32 s = hot_hash(hi, lo) & h.mask;
  for (;;) {
    const u32 x = __ldg(h.idx + s);
    if (x == HB_EMPTY) return HB_EMPTY;
    if (__ldg(h.klo + s) == lo && (KW == 1 || __ldg(h.khi + s) == hi)) return x;
    s = (s + 1) & h.mask;
  }
}

// ---- probe: hit index per row, per-CTA miss lists in row order
#define HP_THREADS 256
#define HP_IT 4
template <int KW>
__global__ void __launch_bounds__(HP_THREADS) k_hot_probe(KeyDesc kd, i64 row0, u32 n, u32 rows_per_cta, HotHash h,
                                                          u32* __restrict__ hit, u32* __restrict__ miss_buf,
                                                          u32* __restrict__ miss_cnt) {
  __shared__ u32 sw[HP_THREADS / 32 + 1];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const u32 b0 = blockIdx.x * rows_per_cta, b1 = min(n, b0 + rows_per_cta);
  u32* my_miss = miss_buf + (size_t)blockIdx.x * rows_per_cta;
  u32 cnt = 0;
  const u32 lt = lanemask_lt();
  for (u32 base = b0; base < b1; base += HP_THREADS * HP_IT) {
    u32 idx[HP_IT];
#pragma unroll
    for (int it = 0; it < HP_IT; ++it) {
      const u32 i = base + it * HP_THREADS + tid;
      idx[it] = 0;
      if (i < b1) {
        u64 hi, lo;
        load_key(kd, row0 + i, hi, lo);
        idx[it] = hot_lookup<KW>(h, hi, lo);
        hit[i] = idx[it];
      }
    }
    // misses of the batch, in row order: (it, tid) is row order
#pragma unroll
    for (int it = 0; it < HP_IT; ++it) {
      const u32 i = base + it * HP_THREADS + tid;
      const bool m = i < b1 && idx[it] == HB_EMPTY;
      const u32 bal = __ballot_sync(0xffffffffu, m);
      if (lane == 0) sw[w] = __popc(bal);
      __syncthreads();
      if (tid == 0) {
        u32 run = 0;
        for (int q = 0; q < HP_THREADS / 32; ++q) { const u32 c = sw[q]; sw[q] = run; run += c; }
        sw[HP_THREADS / 32] = run;
      }
      __syncthreads();
      if (m) my_miss[cnt + sw[w] + __popc(bal & lt)] = i;
      cnt += sw[HP_THREADS / 32];
      __syncthreads();
    }
  }
  if (tid == 0) miss_cnt[blockIdx.x] = cnt;
}

void hot_probe_geometry(u32 n, int num_sms, u32* grid, u32* rows_per_cta) {
  const u32 step = HP_THREADS * HP_IT;
  const u32 max_grid = (u32)num_sms * 8;
  u32 rpc = (n + max_grid - 1) / max_grid;
  rpc = ((rpc + step - 1) / step) * step;
  if (rpc == 0) rpc = step;
  *rows_per_cta = rpc;
  *grid = std::max<u32>(1, (n + rpc - 1) / rpc);
}

void hot_probe(int KW, const KeyDesc& kd, int64_t row0, u32 n, const HotHash& h, u32 grid, u32 rows_per_cta,
               u32* hit, u32* miss_buf, u32* miss_cnt, cudaStream_t st) {
  if (KW == 2) klaunch(k_hot_probe<2>, grid, HP_THREADS, 0, st, kd, (i64)row0, n, rows_per_cta, h, hit, miss_buf, miss_cnt);
  else klaunch(k_hot_probe<1>, grid, HP_THREADS, 0, st, kd, (i64)row0, n, rows_per_cta, h, hit, miss_buf, miss_cnt);
}

// ---- absorb: hits of rows [0, n) combined into T's states
#define HA_THREADS 1024
#define HA_PROBES 8

// private table rows per CTA (shared-memory hash): 4096 for <= 5 slots
// (180 KB), fewer for wider states
template <int MS>
constexpr int ha_slots() { return MS <= 5 ? 4096 : (MS <= 8 ? 2048 : 1024); }
template <int MS>
__global__ void __launch_bounds__(HA_THREADS) k_hot_absorb(SlotDesc sd, i64 row0, u32 n, const u32* __restrict__ hit,
                                                           u64* __restrict__ t_st) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr u32 HA_SLOTS = ha_slots<MS>();
  constexpr int HA_SHIFT = 32 - (MS <= 5 ? 12 : (MS <= 8 ? 11 : 10));
  u32* pk = (u32*)smem;                               // [HA_SLOTS] T index or empty
  u64* acc = (u64*)(pk + HA_SLOTS);                   // [HA_SLOTS][S]
  const int S = sd.nslots;
  for (u32 q = threadIdx.x; q < HA_SLOTS; q += HA_THREADS) {
    pk[q] = HB_EMPTY;
#pragma unroll
    for (int s = 0; s < MS; ++s)
      if (s < S) acc[(size_t)q * S + s] = identity_slot(sd.op[s], sd.type[s]);
  }
  __syncthreads();
  for (u32 i = blockIdx.x * HA_THREADS + threadIdx.x; i < n; i += gridDim.x * HA_THREADS) {
    const u32 x = hit[i];
    if (x == HB_EMPTY) continue;
    u64 v[MS];
    load_state_row<MS>(sd, row0, nullptr, i, v);
    u32 q = (x * 2654435761u) >> HA_SHIFT;
    int p = 0;
    for (; p < HA_PROBES; ++p, q = (q + 1) & (HA_SLOTS - 1)) {
      u32 cur = pk[q];
      if (cur == HB_EMPTY) {
        const u32 old = atomicCAS(pk + q, HB_EMPTY, x);
        cur = old == HB_EMPTY ? x : old;
      }
      if (cur == x) break;
    }
    u64* dst = p < HA_PROBES ? acc + (size_t)q * S : t_st + (size_t)x * S;
#pragma unroll
    for (int s = 0; s < MS; ++s)
      if (s < S) atomic_combine(dst + s, sd.op[s], sd.type[s], v[s]);
  }
  __syncthreads();
  for (u32 q = threadIdx.x; q < HA_SLOTS; q += HA_THREADS) {
    const u32 x = pk[q];
    if (x == HB_EMPTY) continue;
#pragma unroll
    for (int s = 0; s < MS; ++s)
      if (s < S) atomic_combine(t_st + (size_t)x * S + s, sd.op[s], sd.type[s], acc[(size_t)q * S + s]);
  }
}

void hot_absorb(const SlotDesc& sd, int64_t row0, u32 n, const u32* hit, u64* t_st, int num_sms, cudaStream_t st) {
  const int S = sd.nslots;
  if (!n || !S) return;
  const u32 g = std::max<u32>(1, std::min<u32>((n + HA_THREADS * 16 - 1) / (HA_THREADS * 16), (u32)num_sms));
#define HA_GO(M)                                                                                         \
  do {                                                                                                   \
    static std::atomic<unsigned long long> attr{0};                                                      \
    const size_t smem = (size_t)ha_slots<M>() * (4 + (size_t)S * 8);                                     \
    if (first_on_device(attr))                                                                           \
      cudaFuncSetAttribute(k_hot_absorb<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,                 \
                           (int)((size_t)ha_slots<M>() * (4 + (size_t)M * 8)));                          \
    klaunch(k_hot_absorb<M>, g, HA_THREADS, smem, st, sd, (i64)row0, n, hit, t_st);                      \
  } while (0)
  if (S <= 1) HA_GO(1);
  else if (S <= 2) HA_GO(2);
  else if (S <= 4) HA_GO(4);
  else if (S <= 5) HA_GO(5);
  else if (S <= 8) HA_GO(8);
  else HA_GO(16);
#undef HA_GO
}

}  // namespace isa

// ============================================================================
// Hash aggregation baseline (hashagg.py:73-198, the paper's like-for-like
// comparison): one open-addressing table of every group in HBM (the GPU's
// memory holds the whole output, so the reference's budget-driven
// partitioning is never needed), rows mapped to their group's slot, states
// combined by k_hot_absorb (shared-memory privatized), the groups emitted in
// first-arrival order -- the reference's in-memory table order (dict
// insertion order, hashagg.py:124-146).
namespace isa {

#define HT_FREE 0u
#define HT_BUSY 1u
#define HT_READY 2u

template <int KW>
__global__ void k_ha_insert(KeyDesc kd, u32 n, u64* __restrict__ tlo, u64* __restrict__ thi, u32* __restrict__ occ,
                            u32* __restrict__ first, u32 mask, u32* __restrict__ slot_of, u32* __restrict__ ngroups) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 hi, lo;
    load_key(kd, (i64)i, hi, lo);
    u32 s = hot_hash(hi, lo) & mask;
    for (;;) {
      u32 o = *(volatile u32*)(occ + s);
      if (o == HT_FREE) {
        o = atomicCAS(occ + s, HT_FREE, HT_BUSY);
        if (o == HT_FREE) {   // claimed: publish the key
          tlo[s] = lo;
          if (KW == 2) thi[s] = hi;
          __threadfence();
          atomicExch(occ + s, HT_READY);
          atomicAdd(ngroups, 1u);
          break;
        }
      }
      while (o == HT_BUSY) o = *(volatile u32*)(occ + s);   // another row is publishing this slot
      if (*(volatile u64*)(tlo + s) == lo && (KW == 1 || *(volatile u64*)(thi + s) == hi)) break;
      s = (s + 1) & mask;
    }
    slot_of[i] = s;
    if (i < *(volatile u32*)(first + s)) atomicMin(first + s, i);
  }
}

// occupied slots -> (first arrival row, slot) pairs, compacted through an exclusive scan of the flags
__global__ void k_ha_flags(const u32* __restrict__ occ, u32 cap, u32* __restrict__ flag) {
  for (u32 s = blockIdx.x * blockDim.x + threadIdx.x; s < cap; s += gridDim.x * blockDim.x)
    flag[s] = occ[s] == HT_READY ? 1u : 0u;
}
__global__ void k_ha_compact(const u32* __restrict__ occ, const u32* __restrict__ pre, const u32* __restrict__ first,
                             u32 cap, u64* __restrict__ key_first, u32* __restrict__ val_slot) {
  for (u32 s = blockIdx.x * blockDim.x + threadIdx.x; s < cap; s += gridDim.x * blockDim.x)
    if (occ[s] == HT_READY) {
      key_first[pre[s]] = first[s];
      val_slot[pre[s]] = s;
    }
}
template <int MS>
__global__ void k_ha_emit(const u32* __restrict__ order, u32 g, const u64* __restrict__ tlo,
                          const u64* __restrict__ thi, const u64* __restrict__ tst, int S, u64* __restrict__ out_lo,
                          u64* __restrict__ out_hi, u64* __restrict__ out_st) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < g; i += gridDim.x * blockDim.x) {
    const u32 s = order[i];
    out_lo[i] = tlo[s];
    if (out_hi) out_hi[i] = thi[s];
#pragma unroll
    for (int k = 0; k < MS; ++k)
      if (k < S) out_st[(size_t)i * S + k] = tst[(size_t)s * S + k];
  }
}
__global__ void k_ha_init_states(u64* __restrict__ tst, u32 cap, SlotDesc sd) {
  const int S = sd.nslots;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < (size_t)cap * S; q += (size_t)gridDim.x * blockDim.x)
    tst[q] = identity_slot(sd.op[q % S], sd.type[q % S]);
}

void ha_insert(int KW, const KeyDesc& kd, u32 n, const HashAggTable& t, u32* slot_of, cudaStream_t st) {
  cudaMemsetAsync(t.occ, 0, (size_t)(t.mask + 1) * 4, st);
  cudaMemsetAsync(t.first, 0xFF, (size_t)(t.mask + 1) * 4, st);
  cudaMemsetAsync(t.ngroups, 0, 4, st);
  if (!n) return;
  const int g = (int)std::min<u32>((n + 255) / 256, 148u * 16u);
  if (KW == 2) klaunch(k_ha_insert<2>, g, 256, 0, st, kd, n, t.lo, t.hi, t.occ, t.first, t.mask, slot_of, t.ngroups);
  else klaunch(k_ha_insert<1>, g, 256, 0, st, kd, n, t.lo, t.hi, t.occ, t.first, t.mask, slot_of, t.ngroups);
}
void ha_init_states(const HashAggTable& t, const SlotDesc& sd, cudaStream_t st) {
  if (sd.nslots) klaunch(k_ha_init_states, 148 * 8, 256, 0, st, t.st, t.mask + 1, sd);
}
void ha_flags(const HashAggTable& t, u32* flag, cudaStream_t st) {
  klaunch(k_ha_flags, (int)std::min<u32>((t.mask + 256) / 256, 148u * 16u), 256, 0, st, (const u32*)t.occ, t.mask + 1, flag);
}
void ha_compact(const HashAggTable& t, const u32* pre, u64* key_first, u32* val_slot, cudaStream_t st) {
  klaunch(k_ha_compact, (int)std::min<u32>((t.mask + 256) / 256, 148u * 16u), 256, 0, st, (const u32*)t.occ, pre,
          (const u32*)t.first, t.mask + 1, key_first, val_slot);
}
void ha_emit(const HashAggTable& t, const u32* order, u32 g, int KW, int S, u64* out_lo, u64* out_hi, u64* out_st,
             cudaStream_t st) {
  if (!g) return;
  const int gr = (int)std::min<u32>((g + 255) / 256, 148u * 16u);
#define HE(M) klaunch(k_ha_emit<M>, gr, 256, 0, st, order, g, (const u64*)t.lo, (const u64*)t.hi, (const u64*)t.st, S, \
                      out_lo, KW == 2 ? out_hi : (u64*)nullptr, out_st)
  if (S <= 1) HE(1); else if (S <= 2) HE(2); else if (S <= 4) HE(4); else if (S <= 8) HE(8); else HE(16);
#undef HE
}

}  // namespace isa
