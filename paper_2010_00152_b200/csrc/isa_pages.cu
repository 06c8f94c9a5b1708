// Runs in the reference's on-disk page format (runstore.py:1-20, 120-142),
// for the FileStore tier: byte-identical to what the reference's RunWriter
// writes for the same rows and page capacity, so `read_page` of the
// reference can read them back (and this operator reads theirs).
//
//   page = header (row_count u32, byte_length u32, crc32 u32)
//          + high key (arity x int64: the page's last key)
//          + rows (arity key int64s, then S int64 state slots), little-endian
//   crc32 = zlib CRC-32 of everything after the header.
//
// Pages are laid back to back; all but the last hold P rows, so page p
// starts at p * (12 + body_full).  Page starts are only 4-byte aligned
// (12-byte header), so every access is in 32-bit words.
#include "isa_kernels.h"

namespace isa {

__device__ __forceinline__ void crc_table_init(u32* t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    u32 c = (u32)i;
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
    t[i] = c;
  }
}

__device__ __forceinline__ u32 crc_words(const u32* t, const u32* p, u32 nwords) {
  u32 c = 0xFFFFFFFFu;
  for (u32 w = 0; w < nwords; ++w) {
    u32 x = p[w];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      c = t[(c ^ x) & 0xFFu] ^ (c >> 8);
      x >>= 8;
    }
  }
  return ~c;
}

// normalized key -> the column's int64 value (page encoding)
__device__ __forceinline__ i64 pg_key_value(const PageSpec& ps, int c, u64 hi, u64 lo, u32* bad) {
  u64 f = key_field(hi, lo, ps.shift[c], ps.width[c]);
  const int w = ps.width[c];
  if (ps.sgn[c]) {
    f ^= 1ull << (w - 1);
    if (w < 64 && (f >> (w - 1)) & 1ull) f |= ~0ull << w;   // sign-extend
    return (i64)f;
  }
  if (w == 64 && (f >> 63)) atomicOr(bad, 1u);   // uint64 >= 2^63: not an int64 (runstore.py:50, 59)
  return (i64)f;
}

__device__ __forceinline__ void st64(u32* p, u64 v) { p[0] = (u32)v; p[1] = (u32)(v >> 32); }
__device__ __forceinline__ u64 ld64(const u32* p) { return (u64)p[0] | ((u64)p[1] << 32); }

// every row's key + state int64s (and the page's high key at its last row)
__global__ void k_page_body(PageSpec ps, const u64* __restrict__ lo, const u64* __restrict__ hi,
                            const u64* __restrict__ st, u32 n, char* __restrict__ out, u32* __restrict__ bad) {
  const u32 stride = 12 + ps.body_full;
  for (u32 r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const u32 p = r / ps.P, i = r % ps.P;
    u32* body = (u32*)(out + (size_t)p * stride + 12);
    const u64 khi = ps.kw == 2 ? hi[r] : 0, klo = lo[r];
    u32* row = body + 2 * ps.arity + (size_t)i * 2 * (ps.arity + ps.S);
    const bool last = i == (u32)ps.P - 1 || r == n - 1;
    for (int c = 0; c < ps.arity; ++c) {
      const u64 v = (u64)pg_key_value(ps, c, khi, klo, bad);
      st64(row + 2 * c, v);
      if (last) st64(body + 2 * c, v);
    }
    for (int s = 0; s < ps.S; ++s) st64(row + 2 * (ps.arity + s), st[(size_t)r * ps.S + s]);
  }
}

// one thread per page: header (rows, byte length, crc32 of the body)
__global__ void k_page_crc(PageSpec ps, u32 n, char* __restrict__ out) {
  __shared__ u32 tab[256];
  crc_table_init(tab);
  __syncthreads();
  const u32 npages = (n + ps.P - 1) / ps.P;
  const u32 stride = 12 + ps.body_full;
  for (u32 p = blockIdx.x * blockDim.x + threadIdx.x; p < npages; p += gridDim.x * blockDim.x) {
    const u32 rows = min((u32)ps.P, n - p * ps.P);
    const u32 len = 8u * ps.arity + rows * 8u * (ps.arity + ps.S);
    u32* h = (u32*)(out + (size_t)p * stride);
    h[0] = rows;
    h[1] = len;
    h[2] = crc_words(tab, h + 3, len / 4);
  }
}

u32 page_run_bytes(const PageSpec& ps, u32 n) {
  if (n == 0) return 0;
  const u32 npages = (n + ps.P - 1) / ps.P;
  const u32 last = n - (npages - 1) * ps.P;
  return (npages - 1) * (12 + ps.body_full) + 12 + 8u * ps.arity + last * 8u * (ps.arity + ps.S);
}

void page_encode(const PageSpec& ps, const u64* lo, const u64* hi, const u64* st, u32 n, char* out, u32* bad,
                 cudaStream_t stream) {
  if (!n) return;
  klaunch(k_page_body, std::min<u32>((n + 255) / 256, 148u * 16u), 256, 0, stream, ps, lo, hi, st, n, out, bad);
  const u32 npages = (n + ps.P - 1) / ps.P;
  klaunch(k_page_crc, std::min<u32>((npages + 127) / 128, 148u * 8u), 128, 0, stream, ps, n, out);
}

// one CTA per page: thread 0 verifies the crc, all threads parse rows
// [e0, e1) of the page into normalized keys + states at dst
__global__ void k_page_decode(PageSpec ps, const PageRef* __restrict__ refs, const char* __restrict__ src,
                              u64* __restrict__ lo, u64* __restrict__ hi, u64* __restrict__ st,
                              u32* __restrict__ bad) {
  __shared__ u32 tab[256];
  const PageRef pr = refs[blockIdx.x];
  const u32* h = (const u32*)(src + pr.src_off);
  if (threadIdx.x < 32) {
    for (int i = threadIdx.x; i < 256; i += 32) {
      u32 c = (u32)i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
      tab[i] = c;
    }
    __syncwarp();
    if (threadIdx.x == 0) {
      const u32 rows = h[0], len = h[1];
      const u32 want = 8u * ps.arity + rows * 8u * (ps.arity + ps.S);
      if (len != want || rows != pr.rows || crc_words(tab, h + 3, len / 4) != h[2]) atomicOr(bad, 1u);
    }
  }
  const u32* body = h + 3;
  for (u32 i = pr.e0 + threadIdx.x; i < pr.e1; i += blockDim.x) {
    const u32* row = body + 2 * ps.arity + (size_t)i * 2 * (ps.arity + ps.S);
    u64 klo = 0, khi = 0;
    for (int c = 0; c < ps.arity; ++c) {
      u64 f = ld64(row + 2 * c);
      const int w = ps.width[c], s = ps.shift[c];
      if (ps.sgn[c]) f ^= 1ull << (w - 1);
      if (w < 64) f &= (1ull << w) - 1;
      if (s < 64) {
        klo |= f << s;
        if (s > 0 && s + w > 64) khi |= f >> (64 - s);
      } else {
        khi |= f << (s - 64);
      }
    }
    const u32 o = pr.dst + (i - pr.e0);
    lo[o] = klo;
    if (ps.kw == 2) hi[o] = khi;
    for (int s = 0; s < ps.S; ++s) st[(size_t)o * ps.S + s] = ld64(row + 2 * (ps.arity + s));
  }
}

void page_decode(const PageSpec& ps, const PageRef* refs, u32 nrefs, const char* src, u64* lo, u64* hi, u64* st,
                 u32* bad, cudaStream_t stream) {
  if (nrefs) klaunch(k_page_decode, nrefs, 128, 0, stream, ps, refs, src, lo, hi, st, bad);
}

}  // namespace isa
