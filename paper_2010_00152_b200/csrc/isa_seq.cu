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

// ============================================ cut-then-aggregate RSW ====
// Read-sort-write empties the index at every flush (evict_all,
// sortagg.py:333-351), so every fill cycle starts from an empty table and
// its end depends on the keys alone: cycle i is [f_i, f_{i+1}) where
// f_{i+1} is the first row at which the (M + 1)-th distinct key of the
// cycle appears (memindex.py:230-231).  With a small budget the cycles are
// short, so instead of one host round trip per cycle:
//
//   k_cut_scan (one CTA): walks the keys in batches of 1,024 rows with a
//     shared-memory hash set of the cycle's keys (slot -> first row, lowered
//     with atomicMin, so a row is "new" iff it is its key's first row in the
//     cycle), counts new keys in row order (block scan) and cuts at the
//     (M - count + 1)-th new key of the batch; the table is then cleared and
//     the scan resumes at the cut row.  It stops at the first cycle that
//     grows past CUT_GIVEUP rows (the chunked path takes over from that
//     cycle's first row, with an empty table: exact);
//   k_cut_runs (one CTA per cycle, all cycles in parallel): sorts the
//     cycle's rows by key in shared memory (stable LSD on the varying key
//     bits, positions as payload), combines every key segment's rows in row
//     order (the reference's combine order) and writes the run: exactly M
//     groups for a flushed cycle, the residue for the last one.
#define CUT_THREADS 1024
#define CUT_WARPS (CUT_THREADS / 32)
#define CUT_R 4                               // rows per thread per batch (contiguous: scan order = row order)
#define CUT_B (CUT_THREADS * CUT_R)           // batch rows
#define CUT_CAP 12288                         // rows of one cycle sorted in shared memory
#define CUT_GIVEUP (CUT_CAP - CUT_B)          // a cycle longer than this hands over to the chunked path
#define CR_THREADS 256
#define CR_WARPS (CR_THREADS / 32)

struct CutOut {
  u32 ncuts;     // flushed cycles found
  u32 stop;      // first row not covered (n: the scan reached the end)
  u32 batches;   // batch passes (a batch holding a cut is passed again from the cut row)
  u32 overflow;  // cut directory capacity exceeded
};

__device__ __forceinline__ u32 cut_hash(u64 k, int hbits) {
  k ^= k >> 31;
  k *= 0x9E3779B97F4A7C15ull;
  return (u32)(k >> (64 - hbits));
}

// cuts[0] = 0, cuts[1..ncuts] = flush rows, cuts[ncuts + 1] = stop.  A
// batch that holds a cut is passed again with the table cleared and only
// its rows from the cut on (they are still in registers), so the batches
// stay aligned and every row is loaded once.
__global__ void __launch_bounds__(CUT_THREADS, 1) k_cut_scan(KeyDesc kd, u32 n, u32 M, int hbits,
                                                             u32* __restrict__ cuts, u32 max_cuts,
                                                             CutOut* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const u32 HS = 1u << hbits, mask = HS - 1;
  unsigned long long* hkey = (unsigned long long*)smem;   // [HS + 1] (slot HS: the all-ones key)
  u32* hfirst = (u32*)(hkey + HS + 1);                    // [HS + 1] first row of the slot's key
  __shared__ u32 wsum[CUT_WARPS];
  __shared__ u32 s_f;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned long long EMPTY = ~0ull;
  for (u32 i = tid; i <= HS; i += CUT_THREADS) { hkey[i] = EMPTY; hfirst[i] = 0xFFFFFFFFu; }
  __syncthreads();
  u32 pos = 0, seg0 = 0, cnt = 0, ncuts = 0, batches = 0;
  u64 nk[CUT_R];   // the next batch's keys (loaded one batch ahead)
#pragma unroll
  for (int j = 0; j < CUT_R; ++j) {
    const u32 r = tid * CUT_R + j;
    u64 hi;
    nk[j] = 0;
    if (r < n) load_key(kd, (i64)r, hi, nk[j]);
  }
  while (pos < n) {
    u64 k[CUT_R];
#pragma unroll
    for (int j = 0; j < CUT_R; ++j) {
      k[j] = nk[j];
      const u32 r2 = pos + CUT_B + tid * CUT_R + j;
      u64 hi;
      if (r2 < n) load_key(kd, (i64)r2, hi, nk[j]);
    }
    const u32 r0 = pos + tid * CUT_R;   // this thread's first row
    u32 lo_row = pos;                   // rows below it belong to the cycle closed in this batch
    for (;;) {
      ++batches;
      u32 s[CUT_R];
#pragma unroll
      for (int j = 0; j < CUT_R; ++j) {
        const u32 r = r0 + j;
        s[j] = HS;
        if (r < n && r >= lo_row) {
          if (k[j] != EMPTY) {
            u32 q = cut_hash(k[j], hbits);
            for (;;) {
              const unsigned long long old = atomicCAS(hkey + q, EMPTY, (unsigned long long)k[j]);
              if (old == EMPTY || old == k[j]) break;
              q = (q + 1) & mask;
            }
            s[j] = q;
          }
          atomicMin(hfirst + s[j], r);
        }
      }
      __syncthreads();
      u32 nm = 0;   // bit j: row r0 + j is its key's first row in the cycle
#pragma unroll
      for (int j = 0; j < CUT_R; ++j) {
        const u32 r = r0 + j;
        if (r < n && r >= lo_row && hfirst[s[j]] == r) nm |= 1u << j;
      }
      const u32 c = __popc(nm);
      u32 x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[w] = x;
      __syncthreads();
      if (w == 0) {
        u32 t = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 y = __shfl_up_sync(0xffffffffu, t, o);
          if (lane >= o) t += y;
        }
        wsum[lane] = t;   // inclusive over warps
      }
      __syncthreads();
      const u32 total = wsum[CUT_WARPS - 1];
      if (cnt + total <= M) {
        cnt += total;
        __syncthreads();   // wsum is rewritten by the next pass
        break;
      }
      // the (M - cnt + 1)-th new key of the pass is the flush row
      const u32 kth = M - cnt;
      const u32 excl = (w ? wsum[w - 1] : 0) + x - c;
      if (kth >= excl && kth < excl + c) {
        u32 m = nm;
        for (u32 q = excl; q < kth; ++q) m &= m - 1;
        s_f = r0 + (__ffs(m) - 1);
      }
      __syncthreads();
      const u32 f = s_f;
      if (tid == 0) {
        if (ncuts + 2 < max_cuts) cuts[ncuts + 1] = f;
        else out->overflow = 1;
      }
      ++ncuts;
      for (u32 i = tid; i <= HS; i += CUT_THREADS) { hkey[i] = EMPTY; hfirst[i] = 0xFFFFFFFFu; }
      cnt = 0;
      seg0 = f;
      lo_row = f;
      __syncthreads();
    }
    pos += CUT_B;
    if (pos < n && pos - seg0 > CUT_GIVEUP) break;   // this cycle is long: the chunked path takes it
  }
  const u32 stop = pos >= n ? n : seg0;
  if (tid == 0) {
    cuts[0] = 0;
    if (ncuts + 2 <= max_cuts) cuts[ncuts + 1] = stop;
    out->ncuts = ncuts;
    out->stop = stop;
    out->batches = batches;
  }
}

size_t cut_scan_smem(int hbits) { return ((size_t)1 << hbits) * 12 + 16 + 64; }

// one CTA per cycle [cuts[c], cuts[c + 1]): sorted, combined run at run_lo/run_st + c * M
template <int MS>
__global__ void __launch_bounds__(CR_THREADS, 1) k_cut_runs(KeyDesc kd, SlotDesc sd, const u32* __restrict__ cuts,
                                                            u32 M, u64* __restrict__ run_lo,
                                                            u64* __restrict__ run_st, u32* __restrict__ run_len) {
  extern __shared__ __align__(16) unsigned char smem[];
  u64* key = (u64*)smem;                                  // [CUT_CAP] row order
  unsigned short* o0 = (unsigned short*)(key + CUT_CAP);  // [CUT_CAP]
  unsigned short* o1 = o0 + CUT_CAP;                      // [CUT_CAP]
  u32* scratch = (u32*)(o1 + CUT_CAP);                    // [CUT_CAP]
  u32* wcnt = scratch + CUT_CAP;                          // [CR_WARPS][256]
  u32* dstart = wcnt + CR_WARPS * 256;                    // [256]
  __shared__ u32 sw[CR_WARPS + 1];
  __shared__ unsigned long long s_or;
  const int S = sd.nslots;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const u32 c = blockIdx.x;
  const u32 r0 = cuts[c], n = cuts[c + 1] - r0;   // 1 <= n <= CUT_CAP
  u64 kor = 0;
  u64 k0;
  {
    u64 hi;
    load_key(kd, (i64)r0, hi, k0);
  }
  for (u32 i = tid; i < n; i += CR_THREADS) {
    u64 hi, lo;
    load_key(kd, (i64)(r0 + i), hi, lo);
    key[i] = lo;
    o0[i] = (unsigned short)i;
    kor |= lo ^ k0;
  }
  for (int o = 16; o; o >>= 1) kor |= __shfl_xor_sync(0xffffffffu, kor, o);
  if (tid == 0) s_or = 0;
  __syncthreads();
  if (lane == 0 && kor) atomicOr(&s_or, (unsigned long long)kor);
  __syncthreads();
  const int bits = s_or ? 64 - __clzll((long long)s_or) : 0;
  // stable LSD passes over the varying bits: positions move, keys stay
  const u32 WI = (((n + CR_WARPS - 1) / CR_WARPS) + 31) & ~31u;
  const u32 lt = lanemask_lt();
  unsigned short* cur = o0;
  unsigned short* nxt = o1;
  const u32 a0 = w * WI, a1 = min(n, a0 + WI);
  for (int sft = 0; sft < bits; sft += 8) {
    for (int q = lane; q < 256; q += 32) wcnt[w * 256 + q] = 0;
    __syncwarp();
    for (u32 i = a0 + lane; a0 < a1 && i < ((a1 + 31) & ~31u); i += 32) {
      const bool valid = i < a1;
      const u32 d = valid ? (u32)(key[cur[i]] >> sft) & 0xFFu : 256 + lane;
      const u32 peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      u32 cn = 0;
      if (valid && lane == leader) {
        cn = wcnt[w * 256 + d];
        wcnt[w * 256 + d] = cn + __popc(peers);
      }
      cn = __shfl_sync(0xffffffffu, cn, leader);
      if (valid) scratch[i] = (d << 16) | (cn + __popc(peers & lt));
      __syncwarp();
    }
    __syncthreads();
    {
      u32 run = 0;
#pragma unroll
      for (int ww = 0; ww < CR_WARPS; ++ww) {
        const u32 x = wcnt[ww * 256 + tid];
        wcnt[ww * 256 + tid] = run;
        run += x;
      }
      u32 tot;
      dstart[tid] = block_excl_scan256(run, sw, &tot);
    }
    __syncthreads();
    for (u32 i = a0 + lane; i < a1; i += 32) {
      const u32 v = scratch[i], d = v >> 16;
      nxt[dstart[d] + wcnt[w * 256 + d] + (v & 0xFFFFu)] = cur[i];
    }
    __syncthreads();
    unsigned short* t = cur; cur = nxt; nxt = t;
  }
  // group heads in sorted order; thread t owns sorted positions [i0, i1)
  const u32 per = (n + CR_THREADS - 1) / CR_THREADS;
  const u32 i0 = min(n, tid * per), i1 = min(n, i0 + per);
  u32 heads = 0;
  for (u32 i = i0; i < i1; ++i) heads += i == 0 || key[cur[i]] != key[cur[i - 1]];
  u32 tot;
  u32 g = block_excl_scan256(heads, sw, &tot);
  u64* olo = run_lo + (size_t)c * M;
  u64* ost = run_st + (size_t)c * M * S;
  for (u32 i = i0; i < i1; ++i) {
    const u64 k = key[cur[i]];
    if (i != 0 && k == key[cur[i - 1]]) continue;
    u64 acc[MS];
    load_state_row<MS>(sd, (i64)r0, nullptr, cur[i], acc);
    for (u32 j = i + 1; j < n && key[cur[j]] == k; ++j) {
      u64 v[MS];
      load_state_row<MS>(sd, (i64)r0, nullptr, cur[j], v);
#pragma unroll
      for (int q = 0; q < MS; ++q)
        if (q < S) acc[q] = combine_slot(sd.op[q], sd.type[q], acc[q], v[q]);
    }
    olo[g] = k;
#pragma unroll
    for (int q = 0; q < MS; ++q)
      if (q < S) ost[(size_t)g * S + q] = acc[q];
    ++g;
  }
  if (tid == 0) run_len[c] = tot;
}

size_t cut_runs_smem() { return (size_t)CUT_CAP * (8 + 2 + 2 + 4) + (CR_WARPS * 256 + 256) * 4 + 64; }

bool cut_supported(int KW, int S, int64_t M) { return KW == 1 && S <= 8 && M >= 1 && M <= SQ_MAX_M; }

int cut_hash_bits(u32 M) {
  int b = 10;
  while (((u64)1 << b) < (u64)2 * (M + CUT_B)) ++b;   // load <= 1/2 with a full batch of new keys
  return b;
}

void cut_scan(const KeyDesc& kd, u32 n, u32 M, u32* cuts, u32 max_cuts, void* out, cudaStream_t st) {
  const int hb = cut_hash_bits(M);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(k_cut_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  klaunch(k_cut_scan, 1, CUT_THREADS, cut_scan_smem(hb), st, kd, n, M, hb, cuts, max_cuts, (CutOut*)out);
}

void cut_runs(const KeyDesc& kd, const SlotDesc& sd, const u32* cuts, u32 ncycles, u32 M, u64* run_lo, u64* run_st,
              u32* run_len, cudaStream_t st) {
  if (!ncycles) return;
  const int S = sd.nslots;
  const size_t smem = cut_runs_smem();
#define CR_GO(MSV)                                                                                        \
  do {                                                                                                    \
    static std::atomic<unsigned long long> attr{0};                                                       \
    if (first_on_device(attr))                                                                            \
      cudaFuncSetAttribute(k_cut_runs<MSV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
    klaunch(k_cut_runs<MSV>, ncycles, CR_THREADS, smem, st, kd, sd, cuts, M, run_lo, run_st, run_len);    \
  } while (0)
  if (S <= 1) CR_GO(1); else if (S <= 2) CR_GO(2); else if (S <= 4) CR_GO(4); else CR_GO(8);
#undef CR_GO
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
