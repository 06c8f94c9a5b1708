// Run generation for small budgets in one persistent CTA (no host round
// trips): read-sort-write (sortagg.py:333-351) and replacement selection
// (sortagg.py:335-343, 356-369; memindex.py:186-263).
//
// With M <= SQ_MAX_M resident groups, a fill cycle is a few thousand rows
// and the chunked path spends its time in launches and host round trips (one
// per cycle).  Here one CTA keeps the resident index's keys in shared memory
// and walks the input in sorted windows of SQ_CH rows:
//
//   window: rows [w0, w0 + n) sorted by key (stable LSD in shared memory,
//           positions kept), then consumed epoch by epoch from position c;
//   epoch:  every key segment's first live row (position >= c) is looked up
//           in the index (read-sort-write: one table; replacement selection:
//           the current generation, or the next one for keys at or below the
//           eviction cursor); keys not found are new, the (free + 1)-th new
//           key's first row is the trigger f (free = M - resident); rows in
//           [c, f) are applied (hits combined into their group, new keys
//           inserted with the combined state of their rows before f);
//   trigger: read-sort-write flushes the table as one run; replacement
//           selection evicts the P lowest keys of the current generation into
//           the open run (cursor = last evicted key) and, when the generation
//           is empty, closes the run and promotes the next generation; the
//           trigger row is then retried (c = f) exactly like the reference's
//           NEEDS_EVICTION loop.
//
// Runs are written back to back into one device buffer; the host turns them
// into HBM-resident runs for the wide merge.  Group states live in global
// memory (L2-resident at these sizes), keys in shared memory.
#include "isa_kernels.h"

#include <algorithm>
#include <atomic>

namespace isa {

#define SQ_THREADS 512
#define SQ_WARPS (SQ_THREADS / 32)
#define SQ_CH 4096            // window rows
#define SQ_IPT (SQ_CH / SQ_THREADS)

struct SeqOut {               // device counters written by the kernel
  u32 nruns;
  u32 ncycles;
  u32 windows;
  u32 epochs;
  u32 cur_n;                  // groups left in the index (no spill: the result)
  u32 cur_buf;                // which state buffer holds them
  u32 overflow;               // run-directory capacity exceeded
  u32 pad;
  u64 steady_probes, steady_absorbs, steady_resident_sum;   // OutputEstimator (replacement selection)
};

// Stable LSD sort of (key, position) pairs in shared memory over bits
// [0, bits) of key ^ base (bits of the window that vary).  Warp-contiguous
// row ranges, MATCH.ANY ranking with per-warp digit counters.
__device__ void sq_sort(u64* k0, unsigned short* p0, u64* k1, unsigned short* p1, u32 n, int bits, u32* wcnt,
                        u32* dstart, u32* sw, u32* scratch, u64** kout, unsigned short** pout) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const u32 WI = (((n + SQ_WARPS - 1) / SQ_WARPS) + 31) & ~31u;
  const u32 lt = lanemask_lt();
  u64* ck = k0; unsigned short* cp = p0;
  u64* nk = k1; unsigned short* np = p1;
  for (int sft = 0; sft < bits; sft += 8) {
    for (int q = lane; q < 256; q += 32) wcnt[w * 256 + q] = 0;
    __syncwarp();
    const u32 a0 = w * WI, a1 = min(n, a0 + WI);
    for (u32 i = a0 + lane; a0 < a1 && i < ((a1 + 31) & ~31u); i += 32) {
      const bool valid = i < a1;
      const u32 d = valid ? (u32)(ck[i] >> sft) & 0xFFu : 256 + lane;
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
    if (tid < 256) {
      u32 run = 0;
      for (int ww = 0; ww < SQ_WARPS; ++ww) {
        const u32 c = wcnt[ww * 256 + tid];
        wcnt[ww * 256 + tid] = run;
        run += c;
      }
      dstart[tid] = run;
    }
    __syncthreads();
    if (w == 0) {   // exclusive scan of the 256 digit totals
      u32 v[8], s = 0;
      for (int q = 0; q < 8; ++q) { v[q] = dstart[lane * 8 + q]; s += v[q]; }
      u32 x = s;
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      u32 e = x - s;
      for (int q = 0; q < 8; ++q) { dstart[lane * 8 + q] = e; e += v[q]; }
    }
    __syncthreads();
    for (u32 i = a0 + lane; i < a1; i += 32) {
      const u32 v = scratch[i], d = v >> 16;
      const u32 o = dstart[d] + wcnt[w * 256 + d] + (v & 0xFFFFu);
      nk[o] = ck[i];
      np[o] = cp[i];
    }
    __syncthreads();
    u64* tk = ck; ck = nk; nk = tk;
    unsigned short* tp = cp; cp = np; np = tp;
  }
  *kout = ck;
  *pout = cp;
  (void)sw;
}

// first index in [0, n) with a[i] >= k
__device__ __forceinline__ u32 sq_lower(const u64* a, u32 n, u64 k) {
  u32 l = 0, h = n;
  while (l < h) {
    const u32 m = (l + h) >> 1;
    if (a[m] < k) l = m + 1; else h = m;
  }
  return l;
}

template <int MS>
__device__ __forceinline__ void sq_copy_state(u64* dst, const u64* src, int S) {
#pragma unroll
  for (int s = 0; s < MS; ++s)
    if (s < S) dst[s] = src[s];
}

// Per-window scratch (shared): for every sorted slot: live head flag, class
// (0 absorbed into cur, 1 absorbed into next, 2 new for cur, 3 new for next),
// target index; the new heads' rank.
template <int MS, bool RS>
__global__ void __launch_bounds__(SQ_THREADS, 1) k_seq_rungen(
    KeyDesc kd, SlotDesc sd, u32 n_rows, u32 M, u32 P,
    u64* __restrict__ st_a0, u64* __restrict__ st_a1,     // cur states (ping-pong), M x S each
    u64* __restrict__ st_b0, u64* __restrict__ st_b1,     // next states (replacement selection)
    u64* __restrict__ grp_tmp,                            // SQ_CH x S: states of the window's groups
    u64* __restrict__ run_lo, u64* __restrict__ run_st,   // run rows, back to back
    u32* __restrict__ run_off, u32* __restrict__ run_len, u32 max_runs,
    u32* __restrict__ cycles, u64* __restrict__ cur_keys_out, SeqOut* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  u64* wk0 = (u64*)smem;                                  // [SQ_CH]
  u64* wk1 = wk0 + SQ_CH;                                 // [SQ_CH]
  u64* ck = wk1 + SQ_CH;                                  // [M] current generation / table keys
  u64* nkey = ck + M;                                     // [M] next generation keys (RS)
  u64* mk = nkey + (RS ? M : 0);                          // [M] merge output keys
  unsigned short* wp0 = (unsigned short*)(mk + M);        // [SQ_CH]
  unsigned short* wp1 = wp0 + SQ_CH;
  u32* scratch = (u32*)(wp1 + SQ_CH);                     // [SQ_CH]
  u32* info = scratch + SQ_CH;                            // [SQ_CH] class << 28 | target (new: rank)
  u32* wcnt = info + SQ_CH;                               // [SQ_WARPS][256]
  u32* dstart = wcnt + SQ_WARPS * 256;                    // [256]
  u32* bitmap = dstart + 256;                             // [SQ_CH / 32]
  __shared__ u32 sw[SQ_WARPS + 2];
  __shared__ u32 s_cnt[4];
  __shared__ u64 s_or;
  __shared__ u32 s_trig;
  const int S = sd.nslots;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  // index state (uniform across the CTA)
  u32 cn = 0, nn = 0, cb = 0, cbeg = 0;          // cur count, next count, cur state buffer, first live cur row
  bool has_cursor = false;
  u64 cursor = 0;
  bool spilling = false;
  u32 nruns = 0, ncyc = 0, spill_off = 0, open_run = 0xFFFFFFFFu;
  u32 cycle_start = 0, windows = 0, epochs = 0;
  u64 sp_probes = 0, sp_abs = 0, sp_res = 0;
  u64* cst[2] = {st_a0, st_a1};
  u64* nst[2] = {st_b0, st_b1};
  u32 nb = 0;                                    // next state buffer

  auto close_run = [&](u32 len) {
    if (tid == 0) {
      if (nruns < max_runs) { run_off[nruns] = spill_off - len; run_len[nruns] = len; }
      else out->overflow = 1;
    }
    ++nruns;
  };
  // append rows [from, from + len) of the current generation to the run area
  auto spill_cur = [&](u32 from, u32 len) {
    for (u32 i = tid; i < len; i += SQ_THREADS) {
      run_lo[spill_off + i] = ck[from + i];
      sq_copy_state<MS>(run_st + (size_t)(spill_off + i) * S, cst[cb] + (size_t)(from + i) * S, S);
    }
    spill_off += len;
    __syncthreads();   // the keys are read before anyone overwrites them (generation promotion)
  };

  u32 w0 = 0;
  while (w0 < n_rows) {
    const u32 wn = min((u32)SQ_CH, n_rows - w0);
    ++windows;
    // ---- load + sort the window
    u64 kor = 0, k0 = 0;
    {
      u64 hi0, lo0;
      load_key(kd, (i64)w0, hi0, lo0);
      k0 = lo0;
    }
    for (u32 i = tid; i < wn; i += SQ_THREADS) {
      u64 hi, lo;
      load_key(kd, (i64)(w0 + i), hi, lo);
      wk0[i] = lo;
      wp0[i] = (unsigned short)i;
      kor |= lo ^ k0;
    }
    for (int o = 16; o; o >>= 1) kor |= __shfl_xor_sync(0xffffffffu, kor, o);
    if (tid == 0) s_or = 0;
    __syncthreads();
    if (lane == 0) atomicOr((unsigned long long*)&s_or, (unsigned long long)kor);
    __syncthreads();
    const int bits = s_or ? 64 - __clzll((long long)s_or) : 0;
    u64* wk;
    unsigned short* wp;
    sq_sort(wk0, wp0, wk1, wp1, wn, bits, wcnt, dstart, sw, scratch, &wk, &wp);
    // ---- epochs over the window
    u32 c = 0;          // consumed rows (window-relative position)
    bool retry = false; // row c was a trigger: its probe is already counted
    while (c < wn) {
      ++epochs;
      // (1) live heads, lookup, classes
      for (u32 i = tid; i < SQ_CH / 32; i += SQ_THREADS) bitmap[i] = 0;
      if (tid < 4) s_cnt[tid] = 0;
      __syncthreads();
      u32 my_new = 0;
      for (u32 i = tid; i < wn; i += SQ_THREADS) {
        const u32 p = wp[i];
        u32 inf = 0xFFFFFFFFu;   // dead or not a head
        if (p >= c && (i == 0 || wk[i - 1] != wk[i] || wp[i - 1] < c)) {
          const u64 k = wk[i];
          const bool to_next = RS && has_cursor && k <= cursor;
          if (!to_next) {
            const u32 l = cbeg + sq_lower(ck + cbeg, cn, k);
            inf = (l < cbeg + cn && ck[l] == k) ? ((0u << 28) | l) : (2u << 28);
          } else {
            const u32 l = sq_lower(nkey, nn, k);
            inf = (l < nn && nkey[l] == k) ? ((1u << 28) | l) : (3u << 28);
          }
          if ((inf >> 28) >= 2) { atomicOr(bitmap + (p >> 5), 1u << (p & 31)); ++my_new; }
        }
        info[i] = inf;
      }
      for (int o = 16; o; o >>= 1) my_new += __shfl_xor_sync(0xffffffffu, my_new, o);
      if (lane == 0 && my_new) atomicAdd(&s_cnt[0], my_new);
      __syncthreads();
      const u32 n_new = s_cnt[0];
      const u32 resident = cn + nn;
      const u32 free_ = M > resident ? M - resident : 0;
      // (2) trigger: position of the (free + 1)-th new key (bit select)
      u32 f = wn;
      if (n_new > free_) {
        const u32 k = free_ + 1;
        // popcount prefix over the bitmap words (one warp)
        if (w == 0) {
          u32 base = 0;
          for (u32 q0 = 0; q0 < SQ_CH / 32; q0 += 32) {
            const u32 q = q0 + lane;
            const u32 pc = __popc(bitmap[q]);
            u32 x = pc;
            for (int o = 1; o < 32; o <<= 1) {
              const u32 y = __shfl_up_sync(0xffffffffu, x, o);
              if (lane >= o) x += y;
            }
            const u32 ex = base + x - pc;
            if (ex < k && k <= ex + pc) {   // the k-th set bit is in word q
              u32 word = bitmap[q], r = k - ex;
              for (;;) {
                const u32 b = __ffs(word) - 1;
                if (--r == 0) { s_trig = q * 32 + b; break; }
                word &= word - 1;
              }
            }
            base += __shfl_sync(0xffffffffu, x, 31);
          }
        }
        __syncthreads();
        f = s_trig;
      }
      // (3) replacement-selection estimator: rows [c + retry, f) probed, plus the trigger row
      if (RS && spilling) {
        // absorbed = not the first live row of a new key; resident before row p =
        // resident + new keys whose first row precedes p
        if (tid == 0) {
          u64 probes = 0, abs = 0, res = 0;
          // a retried row c applied here was inserted before the rows after it
          u32 newbefore = (retry && c < f && ((bitmap[c >> 5] >> (c & 31)) & 1u)) ? 1u : 0u;
          for (u32 p = c + (retry ? 1 : 0); p < f; ++p) {
            const bool isnew = (bitmap[p >> 5] >> (p & 31)) & 1u;
            ++probes;
            res += resident + newbefore;
            if (isnew) ++newbefore; else ++abs;
          }
          if (f < wn && !(retry && f == c)) { ++probes; res += resident + newbefore; }
          sp_probes += probes; sp_abs += abs; sp_res += res;
        }
      }
      // (4) apply rows [c, f): every live segment whose head is before f
      //     combines its rows before f (hits: into the group; new: a new group)
      for (u32 i = tid; i < wn; i += SQ_THREADS) {
        const u32 inf = info[i];
        if (inf == 0xFFFFFFFFu) continue;
        if (wp[i] >= f) { info[i] = 0xFFFFFFFFu; continue; }
        const u64 k = wk[i];
        u64 acc[MS];
        load_state_row<MS>(sd, (i64)w0, nullptr, wp[i], acc);
        for (u32 j = i + 1; j < wn && wk[j] == k; ++j) {
          const u32 pj = wp[j];
          if (pj >= f) break;
          u64 v[MS];
          load_state_row<MS>(sd, (i64)w0, nullptr, pj, v);
#pragma unroll
          for (int s = 0; s < MS; ++s)
            if (s < S) acc[s] = combine_slot(sd.op[s], sd.type[s], acc[s], v[s]);
        }
        const u32 cls = inf >> 28, tgt = inf & 0x0FFFFFFFu;
        u64* dst = cls == 0 ? cst[cb] + (size_t)tgt * S : (cls == 1 ? nst[nb] + (size_t)tgt * S : grp_tmp + (size_t)i * S);
#pragma unroll
        for (int s = 0; s < MS; ++s)
          if (s < S) dst[s] = cls <= 1 ? combine_slot(sd.op[s], sd.type[s], dst[s], acc[s]) : acc[s];
        if (cls <= 1) info[i] = 0xFFFFFFFFu;
      }
      __syncthreads();
      // (5) insert the new groups (sorted: the window is sorted) into cur / next
      for (int gen = 0; gen < (RS ? 2 : 1); ++gen) {
        const u32 want = gen == 0 ? 2u : 3u;
        // rank of every new group of this generation among them (block scan in sorted order)
        u32 cntl = 0;
        const u32 per = (wn + SQ_THREADS - 1) / SQ_THREADS;
        const u32 i0 = min(wn, tid * per), i1 = min(wn, i0 + per);
        for (u32 i = i0; i < i1; ++i) cntl += (info[i] >> 28) == want && info[i] != 0xFFFFFFFFu;
        u32 x = cntl;
        for (int o = 1; o < 32; o <<= 1) {
          const u32 y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) sw[w] = x;
        __syncthreads();
        if (tid == 0) {
          u32 run = 0;
          for (int q = 0; q < SQ_WARPS; ++q) { const u32 t = sw[q]; sw[q] = run; run += t; }
          sw[SQ_WARPS] = run;
        }
        __syncthreads();
        const u32 nu = sw[SQ_WARPS];
        u32 r = sw[w] + x - cntl;
        for (u32 i = i0; i < i1; ++i)
          if (info[i] != 0xFFFFFFFFu && (info[i] >> 28) == want) scratch[r++] = i;   // new group r -> window slot
        __syncthreads();
        if (nu == 0) continue;
        // merge: existing E (keys in smem, states in buffer eb) + new U -> out buffer
        u64* ek = gen == 0 ? ck + cbeg : nkey;
        const u32 ne = gen == 0 ? cn : nn;
        const u64* est_ = gen == 0 ? cst[cb] + (size_t)cbeg * S : nst[nb];
        u64* ost = gen == 0 ? cst[cb ^ 1] : nst[nb ^ 1];
        for (u32 j = tid; j < ne; j += SQ_THREADS) {   // existing row j -> j + #new keys below it
          const u64 k = ek[j];
          u32 l = 0, h = nu;
          while (l < h) {
            const u32 m = (l + h) >> 1;
            if (wk[scratch[m]] < k) l = m + 1; else h = m;
          }
          mk[j + l] = k;
          sq_copy_state<MS>(ost + (size_t)(j + l) * S, est_ + (size_t)j * S, S);
        }
        for (u32 q = tid; q < nu; q += SQ_THREADS) {   // new group q -> q + #existing keys below it
          const u32 i = scratch[q];
          const u64 k = wk[i];
          const u32 o = q + sq_lower(ek, ne, k);
          mk[o] = k;
          sq_copy_state<MS>(ost + (size_t)o * S, grp_tmp + (size_t)i * S, S);
        }
        __syncthreads();
        u64* dk = gen == 0 ? ck : nkey;
        for (u32 j = tid; j < ne + nu; j += SQ_THREADS) dk[j] = mk[j];
        __syncthreads();
        if (gen == 0) { cn = ne + nu; cb ^= 1; cbeg = 0; }
        else { nn = ne + nu; nb ^= 1; }
      }
      // (6) the trigger
      if (f >= wn) { c = wn; retry = false; break; }
      spilling = true;
      if (!RS) {
        // read-sort-write: the table (M groups) becomes one run
        spill_cur(cbeg, cn);
        close_run(cn);
        if (tid == 0 && ncyc < max_runs) cycles[ncyc] = w0 + f - cycle_start;
        ++ncyc;
        cycle_start = w0 + f;
        cn = 0; cbeg = 0;
      } else {
        // replacement selection: evict the P lowest keys of the current generation
        if (open_run == 0xFFFFFFFFu) open_run = spill_off;
        const u32 ev = min(P, cn);
        if (ev) {
          spill_cur(cbeg, ev);
          cursor = ck[cbeg + ev - 1];
          has_cursor = true;
          cbeg += ev;
          cn -= ev;
        }
        if (cn == 0) {   // generation exhausted: close the run, the next generation becomes current
          close_run(spill_off - open_run);
          open_run = 0xFFFFFFFFu;
          for (u32 j = tid; j < nn; j += SQ_THREADS) ck[j] = nkey[j];
          __syncthreads();
          cn = nn; nn = 0; cbeg = 0;
          { const u32 t = cb; cb = nb; nb = t; u64* t2 = cst[0]; cst[0] = nst[0]; nst[0] = t2;
            t2 = cst[1]; cst[1] = nst[1]; nst[1] = t2; }
          has_cursor = false;
        }
      }
      __syncthreads();
      retry = true;
      c = f;
    }
    w0 += wn;
    __syncthreads();
  }
  // ---- end of input
  if (spilling) {
    if (!RS) {
      if (cn) { spill_cur(cbeg, cn); close_run(cn); cn = 0; }
    } else {
      // drain: the rest of the current generation closes the open run, then
      // the next generation becomes the last run
      if (cn) { if (open_run == 0xFFFFFFFFu) open_run = spill_off; spill_cur(cbeg, cn); cn = 0; }
      if (open_run != 0xFFFFFFFFu) { close_run(spill_off - open_run); open_run = 0xFFFFFFFFu; }
      if (nn) {
        for (u32 j = tid; j < nn; j += SQ_THREADS) ck[j] = nkey[j];
        __syncthreads();
        cn = nn; nn = 0; cbeg = 0;
        { const u32 t = cb; cb = nb; nb = t; u64* t2 = cst[0]; cst[0] = nst[0]; nst[0] = t2;
          t2 = cst[1]; cst[1] = nst[1]; nst[1] = t2; }
        spill_cur(0, cn);
        close_run(cn);
        cn = 0;
      }
    }
  } else {
    // no spill: the index is the result (RS: cur and next never split before the first eviction)
    for (u32 j = tid; j < cn; j += SQ_THREADS) cur_keys_out[j] = ck[cbeg + j];
  }
  __syncthreads();
  if (tid == 0) {
    out->nruns = nruns;
    out->ncycles = ncyc;
    out->windows = windows;
    out->epochs = epochs;
    out->cur_n = cn;
    out->cur_buf = (u32)(cst[cb] == st_a0 ? 0 : (cst[cb] == st_a1 ? 1 : (cst[cb] == st_b0 ? 2 : 3)));
    out->steady_probes = sp_probes;
    out->steady_absorbs = sp_abs;
    out->steady_resident_sum = sp_res;
    (void)cbeg;
  }
}

size_t seq_smem(int M, bool rs) {
  return (size_t)SQ_CH * 8 * 2 + (size_t)M * 8 * (rs ? 3 : 2) + (size_t)SQ_CH * 2 * 2 + (size_t)SQ_CH * 4 * 2 +
         (size_t)SQ_WARPS * 256 * 4 + 256 * 4 + SQ_CH / 8 + 64;
}

bool seq_supported(int KW, int S, int64_t M, bool rs) {
  return KW == 1 && S <= 8 && M >= 2 && M <= SQ_MAX_M && seq_smem((int)M, rs) <= 220 * 1024;
}

void seq_rungen(bool rs, const KeyDesc& kd, const SlotDesc& sd, u32 n, u32 M, u32 P, const SeqBufs& b,
                cudaStream_t st) {
  const size_t smem = seq_smem((int)M, rs);
  const int S = sd.nslots;
#define SQ_GO(MSV, RSV)                                                                                        \
  do {                                                                                                         \
    static std::atomic<unsigned long long> attr{0};                                                            \
    if (first_on_device(attr))                                                                                 \
      cudaFuncSetAttribute(k_seq_rungen<MSV, RSV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);   \
    klaunch(k_seq_rungen<MSV, RSV>, 1, SQ_THREADS, smem, st, kd, sd, n, M, P, b.st_a0, b.st_a1, b.st_b0,       \
            b.st_b1, b.grp_tmp, b.run_lo, b.run_st, b.run_off, b.run_len, b.max_runs, b.cycles, b.cur_keys,   \
            (SeqOut*)b.out);                                                                                   \
  } while (0)
#define SQ_MS(RSV) { if (S <= 1) SQ_GO(1, RSV); else if (S <= 2) SQ_GO(2, RSV); else if (S <= 4) SQ_GO(4, RSV); \
                     else SQ_GO(8, RSV); }
  if (rs) SQ_MS(true) else SQ_MS(false)
#undef SQ_MS
#undef SQ_GO
}

}  // namespace isa
