// Run codec: frame-of-reference bit packing of spilled runs.
//
// A host-tier run crosses PCIe twice (spill, then wide-merge read-back); at
// ~55 GB/s per direction against ~6.5 TB/s of HBM that link is the bound of
// every spilling configuration.  Runs are sorted and their state columns are
// narrow in practice (counts, bounded sums, keys spread over a block of
// consecutive sorted values), so each run is packed on the GPU before the
// D2H copy and unpacked on the GPU after the H2D copy: HBM-speed integer
// work traded for link bytes.  Lossless for every bit pattern.
//
// Block of PK_ROWS consecutive run rows; columns = key words (lo, then hi
// for 128-bit keys), then the S state slots.  Every column value is mapped
// to an order-preserving u64 (keys: as is; int64 slots: x ^ 2^63; f64 slots:
// the IEEE sortable transform), then coded as (value - block minimum) in
// `width` bits, width = bits of (max - min).  Random access (a row's value
// from its block header and two payload words) keeps binary search over
// packed runs possible in place (the wide merge's exact slice bounds).
//
// Block layout (8-byte words): ncol headers {base, width | word_off << 8},
// then every column's payload words (word_off counted from the payload).
#include "isa_kernels.h"

#include <algorithm>
#include <atomic>

namespace isa {

#define PK_THREADS 256

__host__ __device__ __forceinline__ int pk_ncol(int kw, int S) { return kw + S; }

__device__ __forceinline__ u64 pk_get(const PackSrc& p, int c, u32 row) {
  if (c < p.kw) return c == 0 ? p.lo[row] : p.hi[row];
  const int s = c - p.kw;
  return pk_fwd(p.st[(size_t)row * p.S + s], (p.fmask >> s) & 1u, 0);
}

__device__ __forceinline__ u64 block_reduce_min_max(u64 v, bool is_max, u64* sw) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    const u64 t = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? (t > v ? t : v) : (t < v ? t : v);
  }
  __syncthreads();
  if (lane == 0) sw[w] = v;
  __syncthreads();
  u64 r = sw[0];
  for (int i = 1; i < PK_THREADS / 32; ++i) r = is_max ? (sw[i] > r ? sw[i] : r) : (sw[i] < r ? sw[i] : r);
  return r;
}

// per (block, column): base, width, payload word offset; per block: bytes
__global__ void __launch_bounds__(PK_THREADS) k_pack_sizes(PackSrc p, u64* __restrict__ hdr, u32* __restrict__ blk_bytes) {
  __shared__ u64 sw[PK_THREADS / 32];
  const u32 b = blockIdx.x, r0 = b * PK_ROWS;
  const u32 rows = min((u32)PK_ROWS, p.n - r0);
  const int ncol = pk_ncol(p.kw, p.S);
  u64 word_off = 0;
  for (int c = 0; c < ncol; ++c) {
    u64 mn = ~0ull, mx = 0;
    for (u32 i = threadIdx.x; i < rows; i += PK_THREADS) {
      const u64 v = pk_get(p, c, r0 + i);
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
    mn = block_reduce_min_max(mn, false, sw);
    mx = block_reduce_min_max(mx, true, sw);
    const u32 width = mx == mn ? 0u : (u32)(64 - __clzll((long long)(mx - mn)));
    if (threadIdx.x == 0) {
      hdr[((size_t)b * ncol + c) * 2] = mn;
      hdr[((size_t)b * ncol + c) * 2 + 1] = (u64)width | (word_off << 8);
    }
    word_off += ((u64)rows * width + 63) / 64;
  }
  if (threadIdx.x == 0) blk_bytes[b] = (u32)((ncol * 2 + word_off) * 8);
}

// write every block at its offset: headers, then each column's packed words
__global__ void __launch_bounds__(PK_THREADS) k_pack_write(PackSrc p, const u64* __restrict__ hdr,
                                                           const u32* __restrict__ blk_off, char* __restrict__ out) {
  __shared__ u64 vals[PK_ROWS];
  const u32 b = blockIdx.x, r0 = b * PK_ROWS;
  const u32 rows = min((u32)PK_ROWS, p.n - r0);
  const int ncol = pk_ncol(p.kw, p.S);
  u64* blk = (u64*)(out + blk_off[b]);
  for (int i = threadIdx.x; i < ncol * 2; i += PK_THREADS) blk[i] = hdr[(size_t)b * ncol * 2 + i];
  u64* payload = blk + ncol * 2;
  for (int c = 0; c < ncol; ++c) {
    const u64 base = hdr[((size_t)b * ncol + c) * 2];
    const u64 meta = hdr[((size_t)b * ncol + c) * 2 + 1];
    const u32 width = (u32)(meta & 0xFF);
    if (width == 0) continue;
    __syncthreads();
    for (u32 i = threadIdx.x; i < rows; i += PK_THREADS) vals[i] = pk_get(p, c, r0 + i) - base;
    __syncthreads();
    u64* wout = payload + (meta >> 8);
    const u32 nwords = (u32)(((u64)rows * width + 63) / 64);
    for (u32 q = threadIdx.x; q < nwords; q += PK_THREADS) {
      const u64 lo_bit = (u64)q * 64;
      const u32 i0 = (u32)(lo_bit / width);
      const u32 i1 = min(rows - 1, (u32)((lo_bit + 63) / width));
      u64 word = 0;
      for (u32 i = i0; i <= i1; ++i) {
        const long long pos = (long long)((u64)i * width) - (long long)lo_bit;   // bit of value i in this word
        const u64 v = vals[i];
        word |= pos >= 0 ? (v << pos) : (v >> (-pos));
      }
      wout[q] = word;
    }
  }
}

// Single-pass packing: every CTA takes the next block (atomic ticket),
// stages its rows of every column in shared memory with coalesced reads
// (state slots are AoS: one flat read of the block's records), reduces all
// columns' min/max at once, learns its byte offset by decoupled look-back
// over the previous blocks' sizes, and writes header + payload.  Replaces
// sizes -> scan -> write (three passes, two reads of the run) when the
// columns fit the shared-memory stage.
#define PKF_MAXC 8
__device__ __forceinline__ u64 pkf_ld(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void pkf_st(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// NC = kw + S columns (template: the per-column min / max live in registers,
// the staging loops carry no division by a runtime column count).
template <int NC>
__global__ void __launch_bounds__(PK_THREADS) k_pack_fused(PackSrc p, u64* __restrict__ status, u32 epoch,
                                                           u32* __restrict__ ticket, u32* __restrict__ blk_off,
                                                           char* __restrict__ out) {
  extern __shared__ __align__(16) u64 stage[];   // [NC][PK_ROWS]
  __shared__ u64 s_mn[PK_THREADS / 32][NC], s_mx[PK_THREADS / 32][NC];
  __shared__ u64 s_base[NC];
  __shared__ u32 s_width[NC], s_woff[NC], s_b, s_off, s_bytes;
  const int kw = p.kw, S = NC - kw;
  const u32 nblk = (p.n + PK_ROWS - 1) / PK_ROWS;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_b = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 b = s_b, r0 = b * PK_ROWS;
  const u32 rows = min((u32)PK_ROWS, p.n - r0);
  // 1. stage the transformed values of every column, min / max on the way
  u64 mn[NC], mx[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) { mn[c] = ~0ull; mx[c] = 0; }
  const u64* src = p.st + (size_t)r0 * S;
  for (u32 i = tid; i < rows; i += PK_THREADS) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      u64 v;
      if (c < kw) v = c == 0 ? p.lo[r0 + i] : p.hi[r0 + i];
      else v = pk_fwd(src[(size_t)i * S + (c - kw)], (p.fmask >> (c - kw)) & 1u, 0);
      stage[c * PK_ROWS + i] = v;
      mn[c] = v < mn[c] ? v : mn[c];
      mx[c] = v > mx[c] ? v : mx[c];
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    for (int o = 16; o; o >>= 1) {
      const u64 a = __shfl_xor_sync(0xffffffffu, mn[c], o), z = __shfl_xor_sync(0xffffffffu, mx[c], o);
      mn[c] = a < mn[c] ? a : mn[c];
      mx[c] = z > mx[c] ? z : mx[c];
    }
    if (lane == 0) { s_mn[w][c] = mn[c]; s_mx[w][c] = mx[c]; }
  }
  __syncthreads();
  if (w == 0) {
    // lane c reduces column c over the warps; the payload word offsets are a
    // prefix over the columns (shuffle scan)
    u32 words = 0, width = 0;
    if (lane < NC) {
      u64 a = s_mn[0][lane], z = s_mx[0][lane];
#pragma unroll
      for (int ww = 1; ww < PK_THREADS / 32; ++ww) {
        a = s_mn[ww][lane] < a ? s_mn[ww][lane] : a;
        z = s_mx[ww][lane] > z ? s_mx[ww][lane] : z;
      }
      width = z == a ? 0u : (u32)(64 - __clzll((long long)(z - a)));
      words = (rows * width + 63) / 64;
      s_base[lane] = a;
      s_width[lane] = width;
    }
    u32 incl = words;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane < NC) s_woff[lane] = incl - words;
    if (lane == NC - 1) s_bytes = (NC * 2 + incl) * 8;
  }
  __syncthreads();
  // 2. decoupled look-back over the previous blocks' byte counts, one warp:
  //    32 predecessors per round trip
  if (w == 0) {
    const u32 bytes = s_bytes;
    const u64 E = (u64)epoch << 34;
    u32 excl = 0;
    if (b == 0) {
      if (lane == 0) pkf_st(status, E | (2ull << 32) | bytes);
    } else {
      if (lane == 0) pkf_st(status + b, E | (1ull << 32) | bytes);
      int jj = (int)b - 1;
      for (;;) {
        const int q = jj - lane;
        const u64 x = q >= 0 ? pkf_ld(status + q) : (E | (2ull << 32));
        if (!__all_sync(0xffffffffu, (x >> 34) == (u64)epoch)) continue;
        const u32 inc = __ballot_sync(0xffffffffu, ((x >> 32) & 3u) == 2u);
        const int first = inc ? __ffs(inc) - 1 : 32;
        u32 v = lane <= first ? (u32)x : 0u;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        jj -= 32;
      }
      if (lane == 0) pkf_st(status + b, E | (2ull << 32) | (excl + bytes));
    }
    if (lane == 0) {
      s_off = excl;
      blk_off[b] = excl;
      if (b == nblk - 1) blk_off[nblk] = excl + bytes;
    }
  }
  __syncthreads();
  // 3. header + payload at the block's offset; one payload word per thread
  //    step, bit positions in 32-bit arithmetic (rows * width <= 2^16)
  u64* blk = (u64*)(out + s_off);
  if (tid < NC) {
    blk[tid * 2] = s_base[tid];
    blk[tid * 2 + 1] = (u64)s_width[tid] | ((u64)s_woff[tid] << 8);
  }
  u64* payload = blk + NC * 2;
#pragma unroll 1
  for (int c = 0; c < NC; ++c) {
    const u32 width = s_width[c];
    if (width == 0) continue;
    const u64 base = s_base[c];
    const u64* vals = stage + c * PK_ROWS;
    u64* wout = payload + s_woff[c];
    const u32 nwords = (rows * width + 63) / 64;
    for (u32 q = tid; q < nwords; q += PK_THREADS) {
      const u32 lo_bit = q * 64;
      const u32 i0 = lo_bit / width;
      const u32 i1 = min(rows - 1, (lo_bit + 63) / width);
      int pos = (int)(i0 * width) - (int)lo_bit;   // bit of value i0 in this word (<= 0)
      u64 word = (vals[i0] - base) >> (-pos);
      pos += (int)width;
      for (u32 i = i0 + 1; i <= i1; ++i, pos += (int)width) word |= (vals[i] - base) << pos;
      wout[q] = word;
    }
  }
}

bool pack_fused_ok(const PackSrc& p) { return pk_ncol(p.kw, p.S) <= PKF_MAXC; }

static std::atomic<u32> g_pk_epoch{0};

void pack_fused(const PackSrc& p, u64* status, u32* ticket, u32* blk_off, char* out, cudaStream_t st) {
  const u32 nb = pack_blocks(p.n);
  if (!nb) return;
  const size_t smem = (size_t)pk_ncol(p.kw, p.S) * PK_ROWS * 8;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
#define PKF_ATTR(N) cudaFuncSetAttribute(k_pack_fused<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, N * PK_ROWS * 8)
    PKF_ATTR(1); PKF_ATTR(2); PKF_ATTR(3); PKF_ATTR(4); PKF_ATTR(5); PKF_ATTR(6); PKF_ATTR(7); PKF_ATTR(8);
#undef PKF_ATTR
  }
  const u32 ep = (g_pk_epoch.fetch_add(1) % 0x3FFFFFFEu) + 1u;
  cudaMemsetAsync(ticket, 0, sizeof(u32), st);
#define PKF_GO(N) case N: klaunch(k_pack_fused<N>, nb, PK_THREADS, smem, st, p, status, ep, ticket, blk_off, out); break
  switch (pk_ncol(p.kw, p.S)) {
    PKF_GO(1); PKF_GO(2); PKF_GO(3); PKF_GO(4); PKF_GO(5); PKF_GO(6); PKF_GO(7); PKF_GO(8);
    default: break;
  }
#undef PKF_GO
}

u32 pack_blocks(u32 n) { return (n + PK_ROWS - 1) / PK_ROWS; }

void pack_sizes(const PackSrc& p, u64* hdr, u32* blk_bytes, cudaStream_t st) {
  const u32 nb = pack_blocks(p.n);
  if (nb) klaunch(k_pack_sizes, nb, PK_THREADS, 0, st, p, hdr, blk_bytes);
}

void pack_write(const PackSrc& p, const u64* hdr, const u32* blk_off, char* out, cudaStream_t st) {
  const u32 nb = pack_blocks(p.n);
  if (nb) klaunch(k_pack_write, nb, PK_THREADS, 0, st, p, hdr, blk_off, out);
}

// one CTA per descriptor: rows [e0, e1) of a packed block -> dst rows
__global__ void __launch_bounds__(PK_THREADS) k_unpack(const UnpackBlk* __restrict__ d, const char* __restrict__ src,
                                                       int kw, int S, u32 fmask, u64* __restrict__ lo,
                                                       u64* __restrict__ hi, u64* __restrict__ st) {
  const UnpackBlk u = d[blockIdx.x];
  const u64* blk = (const u64*)(uintptr_t)u.src_off;   // absolute (staged copy or HBM-resident run)
  (void)src;
  const int ncol = pk_ncol(kw, S);
  const u64* payload = blk + ncol * 2;
  for (int c = 0; c < ncol; ++c) {
    const u64 base = blk[c * 2], meta = blk[c * 2 + 1];
    const u32 width = (u32)(meta & 0xFF);
    const u64* w = payload + (meta >> 8);
    for (u32 i = u.e0 + threadIdx.x; i < u.e1; i += PK_THREADS) {
      const u64 v = base + pk_extract(w, i, width);
      const u32 o = u.dst + (i - u.e0);
      if (c < kw) {
        if (c == 0) lo[o] = v;
        else hi[o] = v;
      } else {
        const int s = c - kw;
        st[(size_t)o * S + s] = pk_inv(v, (fmask >> s) & 1u, 0);
      }
    }
  }
}

// Slices of HBM-resident packed runs: one descriptor per (run, window) --
// the covering blocks are found on the device (CTA q -> slice by binary
// search over the slices' first block numbers), so the host builds k
// descriptors per window instead of one per 1,024-row block.
__global__ void __launch_bounds__(PK_THREADS) k_unpack_slices(const UnpackSlice* __restrict__ sl, int ns, u32 nblk,
                                                              int kw, int S, u32 fmask, u64* __restrict__ lo,
                                                              u64* __restrict__ hi, u64* __restrict__ st) {
  const int ncol = pk_ncol(kw, S);
  __shared__ u32 s_cnt;
  for (u32 q = blockIdx.x; q < nblk; q += gridDim.x) {
    // last slice with blk0 <= q: counted by all threads at once (one memory
    // round trip instead of a binary search's dependent chain)
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    u32 below = 0;
    for (int t = threadIdx.x; t < ns; t += PK_THREADS) below += sl[t].blk0 <= q ? 1u : 0u;
    for (int o = 16; o; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
    if ((threadIdx.x & 31) == 0 && below) atomicAdd(&s_cnt, below);
    __syncthreads();
    const int l = (int)s_cnt - 1;
    __syncthreads();   // everyone has read the count before the next block resets it
    const UnpackSlice u = sl[l];
    const u32 b = u.s0 / PK_ROWS + (q - u.blk0);
    const u32 r0 = b * PK_ROWS;
    const u32 e0 = max(u.s0, r0) - r0, e1 = min(u.s1, r0 + PK_ROWS) - r0;
    const u64* blk = (const u64*)(u.pk + u.off[b]);
    const u64* payload = blk + ncol * 2;
    for (int c = 0; c < ncol; ++c) {
      const u64 base = blk[c * 2], meta = blk[c * 2 + 1];
      const u32 width = (u32)(meta & 0xFF);
      const u64* w = payload + (meta >> 8);
      for (u32 i = e0 + threadIdx.x; i < e1; i += PK_THREADS) {
        const u64 v = base + pk_extract(w, i, width);
        const u32 o = u.dst + (r0 + i - u.s0);
        if (c < kw) {
          if (c == 0) lo[o] = v;
          else hi[o] = v;
        } else {
          const int s_ = c - kw;
          st[(size_t)o * S + s_] = pk_inv(v, (fmask >> s_) & 1u, 0);
        }
      }
    }
  }
}

void unpack_slices(const UnpackSlice* sl, int ns, u32 nblk, int kw, int S, u32 fmask, u64* lo, u64* hi, u64* st,
                   cudaStream_t stream) {
  if (ns && nblk)
    klaunch(k_unpack_slices, (int)std::min<u32>(nblk, 148u * 16u), PK_THREADS, 0, stream, sl, ns, nblk, kw, S, fmask,
            lo, hi, st);
}

// Raw (unpacked) HBM-resident run slices into a window's staging columns:
// one CTA per piece of <= RAW_PIECE rows instead of one cudaMemcpy per
// slice and column (a window over a few hundred small runs spent ~1 ms in
// copy launches).
__global__ void __launch_bounds__(256) k_gather_raw(const RawCopy* __restrict__ d, int kw, int S, u64* __restrict__ lo,
                                                    u64* __restrict__ hi, u64* __restrict__ st) {
  const RawCopy c = d[blockIdx.x];
  for (u32 i = threadIdx.x; i < c.cnt; i += 256) {
    lo[c.dst + i] = c.lo[i];
    if (kw == 2) hi[c.dst + i] = c.hi[i];
  }
  const u32 ns = c.cnt * (u32)S;
  for (u32 i = threadIdx.x; i < ns; i += 256) st[c.dst * S + i] = c.st[i];
}

void gather_raw(const RawCopy* d, u32 nd, int kw, int S, u64* lo, u64* hi, u64* st, cudaStream_t stream) {
  if (nd) klaunch(k_gather_raw, nd, 256, 0, stream, d, kw, S, lo, hi, st);
}

void unpack_blocks(const UnpackBlk* d, u32 nd, const char* src, int kw, int S, u32 fmask, u64* lo, u64* hi, u64* st,
                   cudaStream_t stream) {
  if (nd) klaunch(k_unpack, nd, PK_THREADS, 0, stream, d, src, kw, S, fmask, lo, hi, st);
}

// ---------------------------------------------------------------------------
// Dense-window wide merge (sortagg.py:588-674 on a dense integer key domain).
// When the runs' keys are dense in their range (a few run rows per possible
// key), a key-range window of D consecutive keys is merged by direct
// addressing: every run row of the window combines its state into entry
// (key - window low) of a D-entry state array that stays in L2 -- no sort,
// no staging of the rows -- and the occupied entries, in index order, are the
// window's groups in key order.  Runs hold unique keys, so an entry receives
// at most one row per run: contention is bounded by the run count whatever
// the key skew.  Integer slots only (atomics commute exactly).
//
// k_dense_accum: one CTA per 1,024-row block of a (run, window) slice, read
// in place from the HBM-resident run (bit-packed blocks decoded on the fly,
// or raw columns); the key pass keeps each row's entry index in registers,
// then one pass per state column issues the reductions.
template <int IT>
__global__ void __launch_bounds__(PK_THREADS) k_dense_accum(const DenseSlice* __restrict__ sl, int ns, u32 nblk, SlotDesc sd,
                                                            u64 key_lo, u32 D, u64* __restrict__ dense,
                                                            unsigned char* __restrict__ occ) {
  static_assert(IT * PK_THREADS == PK_ROWS, "one block of run rows per CTA step");
  const int S = sd.nslots;
  __shared__ u32 s_cnt;
  for (u32 q = blockIdx.x; q < nblk; q += gridDim.x) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    u32 below = 0;
    for (int t = threadIdx.x; t < ns; t += PK_THREADS) below += sl[t].blk0 <= q ? 1u : 0u;
    for (int o = 16; o; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
    if ((threadIdx.x & 31) == 0 && below) atomicAdd(&s_cnt, below);
    __syncthreads();
    const int l = (int)s_cnt - 1;
    __syncthreads();
    const DenseSlice u = sl[l];
    u32 idx[IT];
    if (u.pk) {
      const u32 b = u.s0 / PK_ROWS + (q - u.blk0);
      const u32 r0 = b * PK_ROWS;
      const u32 e0 = max(u.s0, r0) - r0, e1 = min(u.s1, r0 + PK_ROWS) - r0;
      const u64* blk = (const u64*)(u.pk + u.off[b]);
      const u64* payload = blk + (1 + S) * 2;
      {
        const u64 base = blk[0], meta = blk[1];
        const u32 width = (u32)(meta & 0xFF);
        const u64* w = payload + (meta >> 8);
#pragma unroll
        for (int j = 0; j < IT; ++j) {
          const u32 i = e0 + threadIdx.x + j * PK_THREADS;
          const u64 k = i < e1 ? base + pk_extract(w, i, width) - key_lo : ~0ull;
          idx[j] = k < (u64)D ? (u32)k : 0xFFFFFFFFu;
          if (occ && idx[j] != 0xFFFFFFFFu) occ[idx[j]] = 1;
        }
      }
      for (int c = 0; c < S; ++c) {
        const u64 base = blk[(1 + c) * 2], meta = blk[(1 + c) * 2 + 1];
        const u32 width = (u32)(meta & 0xFF);
        const u64* w = payload + (meta >> 8);
        const int op = sd.op[c];
#pragma unroll
        for (int j = 0; j < IT; ++j) {
          if (idx[j] == 0xFFFFFFFFu) continue;
          const u32 i = e0 + threadIdx.x + j * PK_THREADS;
          const u64 v = pk_inv(base + pk_extract(w, i, width), 0, 0);
          atomic_combine(dense + (size_t)idx[j] * S + c, op, ST_I64, v);
        }
      }
    } else {
      const u32 r0 = u.s0 + (q - u.blk0) * PK_ROWS, r1 = min(u.s1, r0 + PK_ROWS);
#pragma unroll
      for (int j = 0; j < IT; ++j) {
        const u32 i = r0 + threadIdx.x + j * PK_THREADS;
        const u64 k = i < r1 ? u.lo[i] - key_lo : ~0ull;
        idx[j] = k < (u64)D ? (u32)k : 0xFFFFFFFFu;
        if (idx[j] == 0xFFFFFFFFu) continue;
        if (occ) occ[idx[j]] = 1;
        for (int c = 0; c < S; ++c)
          atomic_combine(dense + (size_t)idx[j] * S + c, sd.op[c], ST_I64, u.st[(size_t)i * S + c]);
      }
    }
  }
}

// identity states (and cleared occupancy) for entries [0, D)
__global__ void k_dense_init(u64* __restrict__ dense, unsigned char* __restrict__ occ, SlotDesc sd, u32 D) {
  const int S = sd.nslots;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
    for (int c = 0; c < S; ++c) dense[(size_t)i * S + c] = identity_slot(sd.op[c], ST_I64);
    if (occ) occ[i] = 0;
  }
}

#define DN_ITEMS 4
__device__ __forceinline__ bool dense_present(const u64* dense, const unsigned char* occ, int S, int cnt_slot, u32 i) {
  return occ ? occ[i] != 0 : dense[(size_t)i * S + cnt_slot] != 0;
}

// occupied entries per 1,024-entry block
__global__ void __launch_bounds__(256) k_dense_count(const u64* __restrict__ dense, const unsigned char* __restrict__ occ,
                                                     int S, int cnt_slot, u32 D, u32* __restrict__ counts) {
  __shared__ u32 ws[8];
  const u32 i0 = (blockIdx.x * 256 + threadIdx.x) * DN_ITEMS;
  u32 c = 0;
#pragma unroll
  for (int j = 0; j < DN_ITEMS; ++j)
    if (i0 + j < D && dense_present(dense, occ, S, cnt_slot, i0 + j)) ++c;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 t = 0;
    for (int q = 0; q < 8; ++q) t += ws[q];
    counts[blockIdx.x] = t;
  }
}

// occupied entries -> result rows bbase[block] + rank (key = key_lo + entry),
// every entry read is put back to its identity for the next window
__global__ void __launch_bounds__(256) k_dense_emit(u64* __restrict__ dense, unsigned char* __restrict__ occ, SlotDesc sd,
                                                    int cnt_slot, u32 D, u64 key_lo, const u32* __restrict__ bbase,
                                                    u64* __restrict__ out_lo, u64* __restrict__ out_st) {
  __shared__ u32 sw[8];
  const int S = sd.nslots;
  const u32 i0 = (blockIdx.x * 256 + threadIdx.x) * DN_ITEMS;
  bool pres[DN_ITEMS];
  u32 c = 0;
#pragma unroll
  for (int j = 0; j < DN_ITEMS; ++j) {
    pres[j] = i0 + j < D && dense_present(dense, occ, S, cnt_slot, i0 + j);
    c += pres[j] ? 1u : 0u;
  }
  u32 tot;
  u32 pos = bbase[blockIdx.x] + block_excl_scan256(c, sw, &tot);
#pragma unroll
  for (int j = 0; j < DN_ITEMS; ++j) {
    if (!pres[j]) continue;
    const u32 i = i0 + j;
    out_lo[pos] = key_lo + i;
    for (int s = 0; s < S; ++s) {
      out_st[(size_t)pos * S + s] = dense[(size_t)i * S + s];
      dense[(size_t)i * S + s] = identity_slot(sd.op[s], ST_I64);
    }
    if (occ) occ[i] = 0;
    ++pos;
  }
}

// the same, straight into the caller's output columns (isa_set_output_allocator
// with device input): keys denormalized per column, one column per state slot;
// rows at or beyond `cap` are not written (*over = 1: the columns were too small)
__global__ void __launch_bounds__(256) k_dense_emit_cols(u64* __restrict__ dense, unsigned char* __restrict__ occ,
                                                         SlotDesc sd, int cnt_slot, u32 D, u64 key_lo,
                                                         const u32* __restrict__ bbase, ExportDesc ed, u32 cap,
                                                         u32* __restrict__ over) {
  __shared__ u32 sw[8];
  const int S = sd.nslots;
  const u32 i0 = (blockIdx.x * 256 + threadIdx.x) * DN_ITEMS;
  bool pres[DN_ITEMS];
  u32 c = 0;
#pragma unroll
  for (int j = 0; j < DN_ITEMS; ++j) {
    pres[j] = i0 + j < D && dense_present(dense, occ, S, cnt_slot, i0 + j);
    c += pres[j] ? 1u : 0u;
  }
  u32 tot;
  u32 pos = bbase[blockIdx.x] + block_excl_scan256(c, sw, &tot);
#pragma unroll
  for (int j = 0; j < DN_ITEMS; ++j) {
    if (!pres[j]) continue;
    const u32 i = i0 + j;
    if (pos < cap) {
      const u64 nk = key_lo + i;
      for (int q = 0; q < ed.ncols; ++q) {
        const int w = ed.width[q];
        u64 f = key_field(0, nk, ed.shift[q], w);
        if (ed.is_signed[q]) f ^= (1ull << (w - 1));
        switch (w) {
          case 8: ((unsigned char*)ed.key_dst[q])[pos] = (unsigned char)f; break;
          case 16: ((unsigned short*)ed.key_dst[q])[pos] = (unsigned short)f; break;
          case 32: ((unsigned int*)ed.key_dst[q])[pos] = (unsigned int)f; break;
          default: ((u64*)ed.key_dst[q])[pos] = f; break;
        }
      }
      for (int s = 0; s < S; ++s) ((u64*)ed.slot_dst[s])[pos] = dense[(size_t)i * S + s];
    } else {
      *over = 1u;
    }
    for (int s = 0; s < S; ++s) dense[(size_t)i * S + s] = identity_slot(sd.op[s], ST_I64);
    if (occ) occ[i] = 0;
    ++pos;
  }
}

void dense_emit_cols(u64* dense, unsigned char* occ, const SlotDesc& sd, int cnt_slot, u32 D, u64 key_lo,
                     const u32* bbase, const ExportDesc& ed, u32 cap, u32* over, cudaStream_t st) {
  klaunch(k_dense_emit_cols, (int)((D + 256 * DN_ITEMS - 1) / (256 * DN_ITEMS)), 256, 0, st, dense, occ, sd, cnt_slot, D,
          key_lo, bbase, ed, cap, over);
}

void dense_init(u64* dense, unsigned char* occ, const SlotDesc& sd, u32 D, cudaStream_t st) {
  if (D) klaunch(k_dense_init, (int)std::min<u32>((D + 255) / 256, 148u * 8u), 256, 0, st, dense, occ, sd, D);
}
void dense_accum(const DenseSlice* sl, int ns, u32 nblk, const SlotDesc& sd, u64 key_lo, u32 D, u64* dense,
                 unsigned char* occ, cudaStream_t st) {
  if (ns && nblk)
    klaunch(k_dense_accum<PK_ROWS / PK_THREADS>, (int)std::min<u32>(nblk, 148u * 8u), PK_THREADS, 0, st, sl, ns, nblk, sd,
            key_lo, D, dense, occ);
}
u32 dense_blocks(u32 D) { return (D + 256 * DN_ITEMS - 1) / (256 * DN_ITEMS); }
void dense_count(const u64* dense, const unsigned char* occ, int S, int cnt_slot, u32 D, u32* counts, cudaStream_t st) {
  klaunch(k_dense_count, (int)dense_blocks(D), 256, 0, st, dense, occ, S, cnt_slot, D, counts);
}
void dense_emit(u64* dense, unsigned char* occ, const SlotDesc& sd, int cnt_slot, u32 D, u64 key_lo, const u32* bbase,
                u64* out_lo, u64* out_st, cudaStream_t st) {
  klaunch(k_dense_emit, (int)dense_blocks(D), 256, 0, st, dense, occ, sd, cnt_slot, D, key_lo, bbase, out_lo, out_st);
}

// key of `row` of a packed run, read in place (mapped host memory)
template <int KW>
__device__ __forceinline__ void pk_key_at(const RunRef& r, u32 row, u64& khi, u64& klo) {
  const u32 b = row / PK_ROWS, i = row % PK_ROWS;
  const u64* blk = (const u64*)(r.pk + r.blk_off[b]);
  const int ncol = pk_ncol(KW, r.S);
  const u64* payload = blk + ncol * 2;
  klo = blk[0] + pk_extract(payload + (blk[1] >> 8), i, (u32)(blk[1] & 0xFF));
  khi = 0;
  if (KW == 2) khi = blk[2] + pk_extract(payload + (blk[3] >> 8), i, (u32)(blk[3] & 0xFF));
}

// first and last key of every run (KW == 1): out[2r], out[2r + 1]
__global__ void k_run_key_range(const RunRef* __restrict__ runs, int nruns, u64* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= 2 * nruns) return;
  const RunRef rr = runs[q >> 1];
  const u32 row = (q & 1) ? rr.rows - 1 : 0u;
  u64 khi = 0, klo;
  if (rr.pk) pk_key_at<1>(rr, row, khi, klo);
  else klo = rr.lo[row];
  out[q] = klo;
}
void run_key_range(const RunRef* runs, int nruns, u64* out, cudaStream_t st) {
  if (nruns) klaunch(k_run_key_range, (2 * nruns + 127) / 128, 128, 0, st, runs, nruns, out);
}

template <int KW>
__global__ void k_run_lower_bounds(const RunRef* __restrict__ runs, int nruns, const u64* __restrict__ b_lo,
                                   const u64* __restrict__ b_hi, int nb, u32* __restrict__ out) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nruns * nb) return;
  int r = q / nb, b = q % nb;
  const RunRef rr = runs[r];
  u32 l = 0, h = rr.rows;
  const u64 khi = KW == 2 ? b_hi[b] : 0, klo = b_lo[b];
  while (l < h) {
    const u32 m = (l + h) >> 1;
    u64 mhi = 0, mlo;
    if (rr.pk) {
      pk_key_at<KW>(rr, m, mhi, mlo);
    } else {
      mlo = rr.lo[m];
      if (KW == 2) mhi = rr.hi[m];
    }
    if (key_less<KW>(mhi, mlo, khi, klo)) l = m + 1; else h = m;
  }
  out[q] = l;
}

// keys of rows 0, F, 2F, ... of every run (sample q of run r at soff[r] + i;
// runs without samples have soff[r] == soff[r + 1])
template <int KW>
__global__ void k_run_samples(const RunRef* __restrict__ runs, int nruns, const int64_t* __restrict__ soff, int64_t F,
                              int64_t total, u64* __restrict__ out_lo, u64* __restrict__ out_hi) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    int l = 0, h = nruns;   // largest l with soff[l] <= q: a run that has samples
    while (h - l > 1) {
      const int m = (l + h) >> 1;
      if (soff[m] <= q) l = m; else h = m;
    }
    const RunRef rr = runs[l];
    const u32 row = (u32)((q - soff[l]) * F);
    u64 khi = 0, klo;
    if (rr.pk) {
      pk_key_at<KW>(rr, row, khi, klo);
    } else {
      klo = rr.lo[row];
      if (KW == 2) khi = rr.hi[row];
    }
    out_lo[q] = klo;
    if (KW == 2) out_hi[q] = khi;
  }
}

void run_samples(int KW, const RunRef* runs_dev, int nruns, const int64_t* soff_dev, int64_t F, int64_t total,
                 u64* out_lo, u64* out_hi, cudaStream_t st) {
  if (total <= 0) return;
  const int g = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  if (KW == 2) klaunch(k_run_samples<2>, g, 256, 0, st, runs_dev, nruns, soff_dev, F, total, out_lo, out_hi);
  else klaunch(k_run_samples<1>, g, 256, 0, st, runs_dev, nruns, soff_dev, F, total, out_lo, out_hi);
}

void run_lower_bounds(int KW, const RunRef* runs_dev, int nruns, const u64* b_lo, const u64* b_hi, int nb, u32* out,
                      cudaStream_t st) {
  int n = nruns * nb;
  if (n == 0) return;
  int g = (n + 127) / 128;
  if (KW == 2) klaunch(k_run_lower_bounds<2>, g, 128, 0, st, runs_dev, nruns, b_lo, b_hi, nb, out);
  else klaunch(k_run_lower_bounds<1>, g, 128, 0, st, runs_dev, nruns, b_lo, b_hi, nb, out);
}

}  // namespace isa
