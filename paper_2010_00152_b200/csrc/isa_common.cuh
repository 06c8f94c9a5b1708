// Shared device types and helpers: normalized keys, state slots, combine ops.
//
// Keys.  A grouping key is a tuple of integer columns compared
// lexicographically (core.py:265-288, Python tuple order in memindex.py:56-69).
// Each column is mapped to an order-preserving unsigned field (signed types
// get their sign bit flipped) and the fields are concatenated most
// significant column first into one 128-bit word pair (hi:lo).  Unsigned
// comparison of (hi, lo) is then the reference's tuple order.
//
// States.  An aggregate state is a tuple of 8-byte slots (core.py:141-157):
// COUNT/SUM/MIN/MAX take one slot, AVG two (sum, count).  Every slot has a
// combine op (ADD/MIN/MAX, core.py:184-208) and an accumulator type (int64,
// exact like Python ints within 2^63; or float64 like Python floats).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace isa {
// number of kernels this library has launched (process-wide)
extern std::atomic<long long> g_launches;

// Per-kernel-family device timing (CUDA events around the launches of the
// library's main kernels, on their stream), on when kt_enabled(): the
// bench's kernel-true roofline.  alg_bytes = the algorithmic bytes the
// launch moves (inputs read once + outputs written once).
enum KFam { KF_SCATTER = 0, KF_HIST, KF_COLLAPSE, KF_PACK, KF_UNPACK, KF_ABSORB, KF_MERGE, KF_FLUSH, KF_EXPORT,
            KF_HOT_PROBE, KF_HOT_ABSORB, KF_COUNT };
bool kt_enabled();
void kt_set(bool on);
void kt_reserve(int64_t events);
void kt_begin(int fam, cudaStream_t st);
void kt_end(int fam, int64_t alg_bytes, cudaStream_t st);
void kt_add_bytes(int fam, int64_t alg_bytes);   // to the family's last record (bytes known after the launch)
// after the stream(s) synchronized: per family summed ms, launches, bytes
void kt_collect(double* ms, int64_t* launches, int64_t* bytes);

// Kernel attributes (e.g. the dynamic shared-memory limit) are per device:
// true the first time a call site reaches this for the current device.
inline bool first_on_device(std::atomic<unsigned long long>& seen) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned long long bit = 1ull << (d & 63);
  return !(seen.fetch_or(bit) & bit);
}
}

// Every kernel launch of the library goes through klaunch so that the
// operator can report exactly how many of its kernels ran.
template <typename... KArgs, typename... Args>
inline void klaunch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  k<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
  isa::g_launches.fetch_add(1, std::memory_order_relaxed);
}

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

#define ISA_MAX_KEY_COLS 8
#define ISA_MAX_SLOTS 16
#define ISA_MAX_VAL_COLS 16

enum { DT_U8 = 1, DT_I8 = 2, DT_U16 = 3, DT_I16 = 4, DT_U32 = 5, DT_I32 = 6,
       DT_U64 = 7, DT_I64 = 8, DT_F32 = 9, DT_F64 = 10 };
enum { OP_ADD = 0, OP_MIN = 1, OP_MAX = 2 };
enum { ST_I64 = 0, ST_F64 = 1 };
enum { SRC_ONE = 0, SRC_COL = 1 };

struct KeyDesc {
  int ncols;
  int total_bits;
  int dtype[ISA_MAX_KEY_COLS];
  int shift[ISA_MAX_KEY_COLS];   // LSB position of the column's field in the 128-bit key
  int width[ISA_MAX_KEY_COLS];
  const void* ptr[ISA_MAX_KEY_COLS];
};

struct SlotDesc {
  int nslots;
  int op[ISA_MAX_SLOTS];
  int type[ISA_MAX_SLOTS];
  int src[ISA_MAX_SLOTS];
  int dtype[ISA_MAX_SLOTS];      // dtype of the source column (SRC_COL)
  int alias[ISA_MAX_SLOTS];      // earlier slot reading the same column as the same type, or -1
  const void* ptr[ISA_MAX_SLOTS];
  int stride[ISA_MAX_SLOTS];     // bytes between rows of ptr (0: the dtype's size; >0: packed row records)
};

__host__ __device__ __forceinline__ int dtype_bits(int dt) {
  switch (dt) {
    case DT_U8: case DT_I8: return 8;
    case DT_U16: case DT_I16: return 16;
    case DT_U32: case DT_I32: case DT_F32: return 32;
    default: return 64;
  }
}
__host__ __device__ __forceinline__ bool dtype_signed(int dt) {
  return dt == DT_I8 || dt == DT_I16 || dt == DT_I32 || dt == DT_I64;
}
__host__ __device__ __forceinline__ bool dtype_float(int dt) {
  return dt == DT_F32 || dt == DT_F64;
}

// ---------------------------------------------------------------- keys ---
// Order-preserving unsigned image of one key column value.
__device__ __forceinline__ u64 load_key_field(int dt, const void* p, i64 row) {
  switch (dt) {
    case DT_U8:  return (u64)__ldg((const unsigned char*)p + row);
    case DT_I8:  return (u64)(unsigned char)__ldg((const char*)p + row) ^ 0x80ull;
    case DT_U16: return (u64)__ldg((const unsigned short*)p + row);
    case DT_I16: return (u64)(unsigned short)__ldg((const short*)p + row) ^ 0x8000ull;
    case DT_U32: return (u64)__ldg((const unsigned int*)p + row);
    case DT_I32: return (u64)(unsigned int)__ldg((const int*)p + row) ^ 0x80000000ull;
    case DT_U64: return (u64)__ldg((const unsigned long long*)p + row);
    default:     return (u64)__ldg((const long long*)p + row) ^ 0x8000000000000000ull;
  }
}

// Normalized key of one input row -> (hi, lo).
__device__ __forceinline__ void load_key(const KeyDesc& kd, i64 row, u64& hi, u64& lo) {
  hi = 0; lo = 0;
  for (int c = 0; c < kd.ncols; ++c) {
    u64 f = load_key_field(kd.dtype[c], kd.ptr[c], row);
    int s = kd.shift[c];
    if (s < 64) {
      lo |= f << s;
      if (s > 0 && s + kd.width[c] > 64) hi |= f >> (64 - s);
    } else {
      hi |= f << (s - 64);
    }
  }
}

// Inverse of load_key for one column: field value -> column dtype bits.
__device__ __forceinline__ u64 key_field(u64 hi, u64 lo, int shift, int width) {
  u64 v;
  if (shift >= 64) v = hi >> (shift - 64);
  else if (shift == 0) v = lo;
  else v = (lo >> shift) | (hi << (64 - shift));
  if (width < 64) v &= ((1ull << width) - 1);
  return v;
}

template <int KW>
__device__ __forceinline__ bool key_less(u64 ahi, u64 alo, u64 bhi, u64 blo) {
  if (KW == 2) return ahi < bhi || (ahi == bhi && alo < blo);
  return alo < blo;
}
template <int KW>
__device__ __forceinline__ bool key_eq(u64 ahi, u64 alo, u64 bhi, u64 blo) {
  if (KW == 2) return ahi == bhi && alo == blo;
  return alo == blo;
}

// first index i in [0, n) with key[i] >= k (keys sorted ascending)
template <int KW>
__device__ __forceinline__ u32 lower_bound_key(const u64* __restrict__ lo, const u64* __restrict__ hi,
                                               u32 n, u64 khi, u64 klo) {
  u32 l = 0, r = n;
  while (l < r) {
    u32 m = (l + r) >> 1;
    u64 mhi = (KW == 2) ? hi[m] : 0;
    if (key_less<KW>(mhi, lo[m], khi, klo)) l = m + 1; else r = m;
  }
  return l;
}

// --------------------------------------------------------------- states ---
__device__ __forceinline__ double u2d(u64 v) { return __longlong_as_double((long long)v); }
__device__ __forceinline__ u64 d2u(double d) { return (u64)__double_as_longlong(d); }

// Schema.merge_states (core.py:184-208): ADD, MIN (a if a <= b else b),
// MAX (a if a >= b else b), exactly as the reference orders the operands.
__device__ __forceinline__ u64 combine_slot(int op, int type, u64 a, u64 b) {
  if (type == ST_F64) {
    double x = u2d(a), y = u2d(b);
    double r = (op == OP_ADD) ? x + y : (op == OP_MIN ? (x <= y ? x : y) : (x >= y ? x : y));
    return d2u(r);
  }
  i64 x = (i64)a, y = (i64)b;
  i64 r = (op == OP_ADD) ? (i64)((u64)x + (u64)y) : (op == OP_MIN ? (x <= y ? x : y) : (x >= y ? x : y));
  return (u64)r;
}

__host__ __device__ __forceinline__ u64 identity_slot(int op, int type) {
  if (op == OP_ADD) return 0;  // 0 and +0.0 share the bit pattern
  if (type == ST_F64) return op == OP_MIN ? 0x7FF0000000000000ull : 0xFFF0000000000000ull;
  return op == OP_MIN ? 0x7FFFFFFFFFFFFFFFull : 0x8000000000000000ull;
}

// Schema.make_state (core.py:162-182) for one slot of one input row.
__device__ __forceinline__ u64 load_slot_value(int src, int type, int dt, const void* p, i64 row) {
  if (src == SRC_ONE) return type == ST_F64 ? d2u(1.0) : 1ull;
  if (type == ST_F64) {
    switch (dt) {
      case DT_F64: return (u64)__ldg((const long long*)p + row);
      case DT_F32: return d2u((double)__ldg((const float*)p + row));
      case DT_U8:  return d2u((double)__ldg((const unsigned char*)p + row));
      case DT_I8:  return d2u((double)__ldg((const char*)p + row));
      case DT_U16: return d2u((double)__ldg((const unsigned short*)p + row));
      case DT_I16: return d2u((double)__ldg((const short*)p + row));
      case DT_U32: return d2u((double)__ldg((const unsigned int*)p + row));
      case DT_I32: return d2u((double)__ldg((const int*)p + row));
      case DT_U64: return d2u((double)__ldg((const unsigned long long*)p + row));
      default:     return d2u((double)__ldg((const long long*)p + row));
    }
  }
  switch (dt) {
    case DT_U8:  return (u64)__ldg((const unsigned char*)p + row);
    case DT_I8:  return (u64)(i64)__ldg((const char*)p + row);
    case DT_U16: return (u64)__ldg((const unsigned short*)p + row);
    case DT_I16: return (u64)(i64)__ldg((const short*)p + row);
    case DT_U32: return (u64)__ldg((const unsigned int*)p + row);
    case DT_I32: return (u64)(i64)__ldg((const int*)p + row);
    default:     return (u64)__ldg((const unsigned long long*)p + row);  // U64/I64 bit pattern
  }
}

__device__ __forceinline__ void atomic_combine(u64* addr, int op, int type, u64 v) {
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

__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ----------------------------------------------------------- scans ---
__device__ __forceinline__ u32 warp_incl_scan(u32 x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// exclusive scan across a 256-thread block; *total = block sum
__device__ __forceinline__ u32 block_excl_scan256(u32 v, u32* sw, u32* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32 x = warp_incl_scan(v);
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    u32 s = lane < 8 ? sw[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < 8) sw[lane] = s;
  }
  __syncthreads();
  u32 pre = w ? sw[w - 1] : 0;
  *total = sw[7];
  __syncthreads();
  return pre + x - v;
}

// exclusive scan across a block of NW warps; *total = block sum (sw: NW words)
template <int NW>
__device__ __forceinline__ u32 block_excl_scan_nw(u32 v, u32* sw, u32* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32 x = warp_incl_scan(v);
  if (lane == 31) sw[w] = x;
  __syncthreads();
  if (w == 0) {
    u32 s = lane < NW ? sw[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < NW) sw[lane] = s;
  }
  __syncthreads();
  u32 pre = w ? sw[w - 1] : 0;
  *total = sw[NW - 1];
  __syncthreads();
  return pre + x - v;
}

// ---- run codec value transforms (isa_codec.cu; shared with the tile merge's in-place decode)
__device__ __forceinline__ u64 pk_fwd(u64 bits, int is_f64, int is_key) {
  if (is_key) return bits;
  if (is_f64) return (bits >> 63) ? ~bits : (bits ^ 0x8000000000000000ull);
  return bits ^ 0x8000000000000000ull;
}
__device__ __forceinline__ u64 pk_inv(u64 v, int is_f64, int is_key) {
  if (is_key) return v;
  if (is_f64) return (v >> 63) ? (v ^ 0x8000000000000000ull) : ~v;
  return v ^ 0x8000000000000000ull;
}

__device__ __forceinline__ u64 pk_extract(const u64* w, u32 i, u32 width) {
  if (width == 0) return 0;
  const u64 bit = (u64)i * width;
  const u32 q = (u32)(bit >> 6), r = (u32)(bit & 63);
  u64 x = w[q] >> r;
  if (r + width > 64) x |= w[q + 1] << (64 - r);
  return width == 64 ? x : (x & ((1ull << width) - 1));
}

// Schema.make_state of one input row (st_in == nullptr: from the value
// columns, with aliases and packed row records) or an already-built state
// row st_in[v * S ..]
template <int MS>
__device__ __forceinline__ void load_state_row(const SlotDesc& sd, i64 row0, const u64* __restrict__ st_in, u32 v,
                                               u64 (&s)[MS]) {
  const int S = sd.nslots;
  if (st_in) {
    const u64* p = st_in + (size_t)v * S;
#pragma unroll
    for (int k = 0; k < MS; ++k)
      if (k < S) s[k] = p[k];
  } else {
#pragma unroll
    for (int k = 0; k < MS; ++k) {
      if (k < S) {
        const int a = sd.alias[k];
        u64 x = 0;
#pragma unroll
        for (int q = 0; q < k; ++q)
          if (q == a) x = s[q];
        s[k] = a >= 0 ? x
                      : (sd.stride[k] ? load_slot_value(sd.src[k], sd.type[k], sd.dtype[k],
                                                        (const char*)sd.ptr[k] + (size_t)(row0 + v) * sd.stride[k], 0)
                                      : load_slot_value(sd.src[k], sd.type[k], sd.dtype[k], sd.ptr[k], row0 + v));
      }
    }
  }
}

