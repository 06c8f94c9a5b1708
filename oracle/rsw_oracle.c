/*
 * ORACLE — test infrastructure only.  CPU restatement of the reference's
 * wide-mode sort-based aggregation for parity checks and the CPU baseline:
 *
 *   index_run_generation, read-sort-write branch
 *       /root/reference/pkg/src/insortagg/sortagg.py:300-376 (flush :344-351,
 *       residue run :353-374); OrderedIndex.insert_or_aggregate budget test
 *       memindex.py:197-236 (NEEDS_EVICTION without mutation :230-231)
 *   wide_merge: final output = every run merged with states combined
 *       sortagg.py:588-674 (emits each key once, ascending)
 *   Schema.merge_states (core.py:184-208), RunWriter page/ledger accounting
 *       (runstore.py:284-292), OutputEstimator.note_cycle(consumed - 1)
 *       (sortagg.py:345).
 *
 * The ordered index is restated as a hash table whose resident entries are
 * sorted when a run is flushed: the run contents, run boundaries and ledger
 * are identical to the b-tree's because RSW flushes the whole index and the
 * flush point depends only on the distinct-key count.  Keys arrive already
 * normalized to order-preserving 128-bit (hi, lo) words; state slots arrive
 * already built by make_state (8-byte int64 or float64 bit patterns).
 *
 * Never linked into or called by the product path.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;

enum { OP_ADD = 0, OP_MIN = 1, OP_MAX = 2 };
enum { ST_I64 = 0, ST_F64 = 1 };

typedef struct {
  int S;
  int op[16];
  int type[16];
} slots_t;

static inline u64 combine(const slots_t* sl, int s, u64 a, u64 b) {
  if (sl->type[s] == ST_F64) {
    double x, y, r;
    memcpy(&x, &a, 8);
    memcpy(&y, &b, 8);
    if (sl->op[s] == OP_ADD) r = x + y;
    else if (sl->op[s] == OP_MIN) r = x <= y ? x : y;
    else r = x >= y ? x : y;
    u64 o;
    memcpy(&o, &r, 8);
    return o;
  }
  int64_t x = (int64_t)a, y = (int64_t)b, r;
  if (sl->op[s] == OP_ADD) r = (int64_t)((u64)x + (u64)y);
  else if (sl->op[s] == OP_MIN) r = x <= y ? x : y;
  else r = x >= y ? x : y;
  return (u64)r;
}

static inline int key_cmp(u64 ah, u64 al, u64 bh, u64 bl) {
  if (ah != bh) return ah < bh ? -1 : 1;
  if (al != bl) return al < bl ? -1 : 1;
  return 0;
}

/* growable sorted table (a run or the output) */
typedef struct {
  u64 *hi, *lo, *st;
  int64_t n, cap;
} table_t;

static void table_push(table_t* t, int S, u64 h, u64 l, const u64* st) {
  if (t->n == t->cap) {
    int64_t nc = t->cap ? t->cap * 2 : 1024;
    t->hi = realloc(t->hi, nc * 8);
    t->lo = realloc(t->lo, nc * 8);
    if (S) t->st = realloc(t->st, nc * 8 * S);
    t->cap = nc;
  }
  t->hi[t->n] = h;
  t->lo[t->n] = l;
  if (S) memcpy(t->st + t->n * S, st, 8 * S);
  t->n++;
}

static void table_free(table_t* t) {
  free(t->hi);
  free(t->lo);
  free(t->st);
  memset(t, 0, sizeof(*t));
}

/* ---- the index: open-addressing hash of at most M resident groups ---- */
typedef struct {
  int64_t M, cap, mask, resident;
  u64 *khi, *klo;
  int32_t* slot;      /* -1 empty, else row in states/keys arrays */
  u64* st;            /* M * S */
  u64 *ehi, *elo;     /* keys by row */
} index_t;

static inline u64 mix(u64 h, u64 l) {
  u64 x = l ^ (h * 0x9E3779B97F4A7C15ull);
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static void index_init(index_t* ix, int64_t M, int S) {
  ix->M = M;
  int64_t cap = 16;
  while (cap < 2 * M) cap <<= 1;
  ix->cap = cap;
  ix->mask = cap - 1;
  ix->resident = 0;
  ix->khi = malloc(cap * 8);
  ix->klo = malloc(cap * 8);
  ix->slot = malloc(cap * 4);
  memset(ix->slot, 0xFF, cap * 4);
  ix->st = malloc((M ? M : 1) * 8 * (S ? S : 1));
  ix->ehi = malloc(M * 8);
  ix->elo = malloc(M * 8);
}

static void index_free(index_t* ix) {
  free(ix->khi); free(ix->klo); free(ix->slot); free(ix->st); free(ix->ehi); free(ix->elo);
}

/* 1 absorbed, 0 inserted, -1 needs eviction (no mutation) */
static int index_insert(index_t* ix, const slots_t* sl, u64 h, u64 l, const u64* st) {
  int S = sl->S;
  int64_t p = (int64_t)(mix(h, l) & ix->mask);
  for (;;) {
    int32_t r = ix->slot[p];
    if (r < 0) break;
    if (ix->khi[p] == h && ix->klo[p] == l) {
      u64* d = ix->st + (int64_t)r * S;
      for (int s = 0; s < S; ++s) d[s] = combine(sl, s, d[s], st[s]);
      return 1;
    }
    p = (p + 1) & ix->mask;
  }
  if (ix->resident >= ix->M) return -1;
  int32_t r = (int32_t)ix->resident++;
  ix->slot[p] = r;
  ix->khi[p] = h;
  ix->klo[p] = l;
  ix->ehi[r] = h;
  ix->elo[r] = l;
  if (S) memcpy(ix->st + (int64_t)r * S, st, 8 * S);
  return 0;
}

static const u64* g_sort_hi;
static const u64* g_sort_lo;
static int cmp_rows(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return key_cmp(g_sort_hi[x], g_sort_lo[x], g_sort_hi[y], g_sort_lo[y]);
}

/* drain the index in ascending key order into `out` (evict_all) */
static void index_drain(index_t* ix, int S, table_t* out, pthread_mutex_t* mu) {
  int64_t n = ix->resident;
  int32_t* ord = malloc((n ? n : 1) * 4);
  for (int64_t i = 0; i < n; ++i) ord[i] = (int32_t)i;
  /* qsort comparator uses globals: serialize (the oracle is not a hot path) */
  pthread_mutex_lock(mu);
  g_sort_hi = ix->ehi;
  g_sort_lo = ix->elo;
  qsort(ord, n, 4, cmp_rows);
  pthread_mutex_unlock(mu);
  for (int64_t i = 0; i < n; ++i)
    table_push(out, S, ix->ehi[ord[i]], ix->elo[ord[i]], ix->st + (int64_t)ord[i] * S);
  free(ord);
  memset(ix->slot, 0xFF, ix->cap * 4);
  ix->resident = 0;
}

typedef struct {
  table_t out;
  int64_t rows_spilled, pages_written, runs;
  int64_t* cycles;
  int64_t ncycles, cap_cycles;
} result_part;

typedef struct oracle_result {
  int S;
  table_t out;
  int64_t ledger[8];  /* rows_spilled, rows_read_back, pages_written, pages_read, merge_steps, merge_levels, runs, n_groups */
  int64_t* cycles;
  int64_t ncycles;
} oracle_result;

static pthread_mutex_t g_mu = PTHREAD_MUTEX_INITIALIZER;

/* heap entry for the wide merge */
typedef struct { u64 h, l; int32_t run; } hent;
static inline int hless(const hent* a, const hent* b) {
  int c = key_cmp(a->h, a->l, b->h, b->l);
  return c < 0 || (c == 0 && a->run < b->run);
}
static void sift_down(hent* hp, int64_t n, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && hless(&hp[l], &hp[m])) m = l;
    if (r < n && hless(&hp[r], &hp[m])) m = r;
    if (m == i) return;
    hent t = hp[i]; hp[i] = hp[m]; hp[m] = t;
    i = m;
  }
}

/* one operator instance over the rows whose key lies in [lo_key, hi_key) */
static void run_operator(int64_t n, const u64* khi, const u64* klo, const u64* const* slots, const slots_t* sl,
                         int64_t M, int64_t P, int use_range, u64 rlo_h, u64 rlo_l, int has_hi, u64 rhi_h,
                         u64 rhi_l, result_part* res) {
  const int S = sl->S;
  index_t ix;
  index_init(&ix, M, S);
  table_t* runs = NULL;
  int64_t nruns = 0, cap_runs = 0;
  int64_t consumed = 0;
  u64 st[16];
  for (int64_t i = 0; i < n; ++i) {
    u64 h = khi ? khi[i] : 0, l = klo[i];
    if (use_range) {
      if (key_cmp(h, l, rlo_h, rlo_l) < 0) continue;
      if (has_hi && key_cmp(h, l, rhi_h, rhi_l) >= 0) continue;
    }
    for (int s = 0; s < S; ++s) st[s] = slots[s][i];
    consumed++;
    int o = index_insert(&ix, sl, h, l, st);
    while (o < 0) {
      /* read-sort-write flush of the whole index (sortagg.py:344-351) */
      if (res->ncycles == res->cap_cycles) {
        res->cap_cycles = res->cap_cycles ? res->cap_cycles * 2 : 64;
        res->cycles = realloc(res->cycles, res->cap_cycles * 8);
      }
      res->cycles[res->ncycles++] = consumed - 1;
      consumed = 1;
      if (nruns == cap_runs) {
        cap_runs = cap_runs ? cap_runs * 2 : 16;
        runs = realloc(runs, cap_runs * sizeof(table_t));
      }
      memset(&runs[nruns], 0, sizeof(table_t));
      index_drain(&ix, S, &runs[nruns], &g_mu);
      nruns++;
      o = index_insert(&ix, sl, h, l, st);
    }
  }
  if (nruns == 0) {
    index_drain(&ix, S, &res->out, &g_mu);
  } else {
    if (ix.resident) {
      if (nruns == cap_runs) {
        cap_runs = cap_runs ? cap_runs * 2 : 16;
        runs = realloc(runs, cap_runs * sizeof(table_t));
      }
      memset(&runs[nruns], 0, sizeof(table_t));
      index_drain(&ix, S, &runs[nruns], &g_mu);
      nruns++;
    }
    for (int64_t r = 0; r < nruns; ++r) {
      res->rows_spilled += runs[r].n;
      res->pages_written += (runs[r].n + P - 1) / P;
    }
    res->runs = nruns;
    /* wide merge: k-way merge, combining equal keys into one output row */
    hent* hp = malloc(nruns * sizeof(hent));
    int64_t* pos = calloc(nruns, 8);
    int64_t hn = 0;
    for (int64_t r = 0; r < nruns; ++r)
      if (runs[r].n) { hp[hn].h = runs[r].hi[0]; hp[hn].l = runs[r].lo[0]; hp[hn].run = (int32_t)r; hn++; }
    for (int64_t i = hn / 2 - 1; i >= 0; --i) sift_down(hp, hn, i);
    u64 acc[16];
    u64 ch = 0, cl = 0;
    int have = 0;
    while (hn) {
      hent top = hp[0];
      int32_t r = top.run;
      const u64* rs = runs[r].st + pos[r] * S;
      if (have && top.h == ch && top.l == cl) {
        for (int s = 0; s < S; ++s) acc[s] = combine(sl, s, acc[s], rs[s]);
      } else {
        if (have) table_push(&res->out, S, ch, cl, acc);
        have = 1; ch = top.h; cl = top.l;
        for (int s = 0; s < S; ++s) acc[s] = rs[s];
      }
      pos[r]++;
      if (pos[r] < runs[r].n) {
        hp[0].h = runs[r].hi[pos[r]];
        hp[0].l = runs[r].lo[pos[r]];
      } else {
        hp[0] = hp[--hn];
      }
      sift_down(hp, hn, 0);
    }
    if (have) table_push(&res->out, S, ch, cl, acc);
    free(hp);
    free(pos);
    for (int64_t r = 0; r < nruns; ++r) table_free(&runs[r]);
  }
  free(runs);
  index_free(&ix);
}

typedef struct {
  int64_t n; const u64 *khi, *klo; const u64* const* slots; const slots_t* sl; int64_t M, P;
  int use_range; u64 rlo_h, rlo_l; int has_hi; u64 rhi_h, rhi_l; result_part res;
} job_t;

static void* job_main(void* arg) {
  job_t* j = (job_t*)arg;
  run_operator(j->n, j->khi, j->klo, j->slots, j->sl, j->M, j->P, j->use_range, j->rlo_h, j->rlo_l, j->has_hi,
               j->rhi_h, j->rhi_l, &j->res);
  return NULL;
}

/* nthreads == 1: the reference algorithm exactly (ledger comparable).
 * nthreads > 1: one independent operator per key range (splitters taken from
 * `split_hi/split_lo`, nthreads-1 sorted normalized keys), outputs
 * concatenated in range order; ledger counters are summed. */
oracle_result* oracle_sortagg(int64_t n, const u64* khi, const u64* klo, int S, const u64* const* slots,
                              const int* op, const int* type, int64_t M, int64_t P, int nthreads,
                              const u64* split_hi, const u64* split_lo) {
  slots_t sl;
  memset(&sl, 0, sizeof(sl));
  sl.S = S;
  for (int s = 0; s < S && s < 16; ++s) { sl.op[s] = op[s]; sl.type[s] = type[s]; }
  if (nthreads < 1) nthreads = 1;
  job_t* jobs = calloc(nthreads, sizeof(job_t));
  for (int t = 0; t < nthreads; ++t) {
    job_t* j = &jobs[t];
    j->n = n; j->khi = khi; j->klo = klo; j->slots = slots; j->sl = &sl; j->M = M; j->P = P;
    j->use_range = nthreads > 1;
    if (t > 0) { j->rlo_h = split_hi ? split_hi[t - 1] : 0; j->rlo_l = split_lo[t - 1]; }
    j->has_hi = t < nthreads - 1;
    if (j->has_hi) { j->rhi_h = split_hi ? split_hi[t] : 0; j->rhi_l = split_lo[t]; }
  }
  if (nthreads == 1) {
    job_main(&jobs[0]);
  } else {
    pthread_t* th = malloc(nthreads * sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, job_main, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  oracle_result* r = calloc(1, sizeof(oracle_result));
  r->S = S;
  for (int t = 0; t < nthreads; ++t) {
    result_part* p = &jobs[t].res;
    for (int64_t i = 0; i < p->out.n; ++i) table_push(&r->out, S, p->out.hi[i], p->out.lo[i], p->out.st + i * S);
    r->ledger[0] += p->rows_spilled;
    r->ledger[1] += p->rows_spilled;
    r->ledger[2] += p->pages_written;
    r->ledger[3] += p->pages_written;
    if (p->runs) { r->ledger[4] += 1; r->ledger[5] += 1; }
    r->ledger[6] += p->runs;
    if (p->ncycles) {
      r->cycles = realloc(r->cycles, (r->ncycles + p->ncycles) * 8);
      memcpy(r->cycles + r->ncycles, p->cycles, p->ncycles * 8);
      r->ncycles += p->ncycles;
    }
    table_free(&p->out);
    free(p->cycles);
  }
  r->ledger[7] = r->out.n;
  free(jobs);
  return r;
}

int64_t oracle_n_groups(const oracle_result* r) { return r->out.n; }

void oracle_copy(const oracle_result* r, u64* hi, u64* lo, u64* const* slots_out) {
  int64_t n = r->out.n;
  if (hi) memcpy(hi, r->out.hi, n * 8);
  memcpy(lo, r->out.lo, n * 8);
  for (int s = 0; s < r->S; ++s)
    for (int64_t i = 0; i < n; ++i) slots_out[s][i] = r->out.st[i * r->S + s];
}

void oracle_ledger(const oracle_result* r, int64_t* out8) { memcpy(out8, r->ledger, 8 * 8); }

int64_t oracle_cycles(const oracle_result* r, int64_t* out, int64_t cap) {
  for (int64_t i = 0; i < r->ncycles && i < cap; ++i) out[i] = r->cycles[i];
  return r->ncycles;
}

void oracle_free(oracle_result* r) {
  if (!r) return;
  table_free(&r->out);
  free(r->cycles);
  free(r);
}
