/*
 * ORACLE -- test infrastructure only.  Never linked into or called by the
 * product path (paper_2605_10501_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs load it.
 *
 * Plain-C restatement of the reference wavefront scheduler
 * (/root/reference/pkg/src/maestro/scheduling.py) in IEEE fp64 with the
 * reference's exact operation order, so results are bit-identical to the
 * Python reference.  Pinned against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py -> the JSON fixtures under tests/golden).
 *
 * Times are phase-major: t[p*B + i] for phase p in (f_bc, f_c, f_ac, b_bc,
 * b_c, b_ac) and batch index i.  Orders are arrays of batch indices.
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -shared -fPIC (see Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define F_BC 0
#define F_C 1
#define F_AC 2
#define B_BC 3
#define B_C 4
#define B_AC 5
#define T(p, i) (t[(size_t)(p) * (size_t)B + (size_t)(i)])

/* Python max(a, b): returns b only when b > a (first maximal element). */
static inline double pmax(double a, double b) { return b > a ? b : a; }

typedef struct {
  double c, first, last, busy;
  int have_first;
} crit_clock;

static inline double run_critical(crit_clock* k, double floor_, double ready, double dur) {
  /* scheduling.py:104-113 */
  double start = pmax(floor_, ready);
  double end = start + dur;
  k->c = end;
  if (!k->have_first) {
    k->first = start;
    k->have_first = 1;
  }
  k->last = end;
  k->busy += dur;
  return end;
}

/* rank_metrics (scheduling.py:81-152).  policy 0 = interleaved, 1 = all-fwd-then-bwd.
 * scratch must hold 2*n doubles.  Returns makespan; busy/span optional. */
double oracle_rank_metrics(const double* t, int B, const int* order, int n, int policy,
                           double* busy_out, double* span_out, double* scratch) {
  if (n <= 0) {
    if (busy_out) *busy_out = 0.0;
    if (span_out) *span_out = 0.0;
    return 0.0;
  }
  double* ready_fc = scratch;
  double* after_fwd = scratch + n;
  double u = 0.0;
  for (int k = 0; k < n; ++k) {
    double f = T(F_BC, order[k]);
    if (f > 0) {
      u += f;
      ready_fc[k] = u;
    } else {
      ready_fc[k] = 0.0;
    }
  }
  double ub = u, d = 0.0, mk = 0.0, chain, start;
  crit_clock k0 = {0.0, 0.0, 0.0, 0.0, 0};
  if (policy == 0) {
    for (int k = 0; k < n; ++k) {
      int s = order[k];
      chain = run_critical(&k0, k0.c, ready_fc[k], T(F_C, s));
      if (T(F_AC, s) > 0) { start = pmax(d, chain); chain = d = start + T(F_AC, s); }
      if (T(B_BC, s) > 0) { start = pmax(d, chain); chain = d = start + T(B_BC, s); }
      if (T(B_C, s) > 0) chain = run_critical(&k0, k0.c, chain, T(B_C, s));
      if (T(B_AC, s) > 0) { start = pmax(ub, chain); chain = ub = start + T(B_AC, s); }
      mk = pmax(mk, chain);
    }
  } else {
    for (int k = 0; k < n; ++k) {
      int s = order[k];
      chain = run_critical(&k0, k0.c, ready_fc[k], T(F_C, s));
      if (T(F_AC, s) > 0) { start = pmax(d, chain); chain = d = start + T(F_AC, s); }
      after_fwd[k] = chain;
    }
    for (int k = 0; k < n; ++k) {
      int s = order[k];
      chain = after_fwd[k];
      if (T(B_BC, s) > 0) { start = pmax(d, chain); chain = d = start + T(B_BC, s); }
      if (T(B_C, s) > 0) chain = run_critical(&k0, k0.c, chain, T(B_C, s));
      if (T(B_AC, s) > 0) { start = pmax(ub, chain); chain = ub = start + T(B_AC, s); }
      mk = pmax(mk, chain);
    }
  }
  if (busy_out) *busy_out = k0.busy;
  if (span_out) *span_out = k0.last - (k0.have_first ? k0.first : 0.0);
  return mk;
}

/* schedule_rank (scheduling.py:162-199): stable sort by t_f_bc, seed with the
 * first, insert each next at the makespan-minimising position (strict <, so the
 * smallest index wins ties), then keep the input order if strictly better.
 * in/out are batch-index arrays of length n.  Returns evaluation count. */
long long oracle_schedule_rank(const double* t, int B, const int* in, int n, int policy, int* out) {
  if (n <= 1) {
    if (n == 1) out[0] = in[0];
    return 0;
  }
  int* init = (int*)malloc(sizeof(int) * (size_t)n);
  int* cand = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  double* scratch = (double*)malloc(sizeof(double) * 2 * (size_t)(n + 1));
  /* stable insertion sort by t_f_bc (sort_initial, scheduling.py:76-78) */
  for (int i = 0; i < n; ++i) {
    int v = in[i], j = i;
    while (j > 0 && T(F_BC, init[j - 1]) > T(F_BC, v)) {
      init[j] = init[j - 1];
      --j;
    }
    init[j] = v;
  }
  long long evals = 0;
  int len = 1;
  out[0] = init[0];
  double best = 0.0;
  for (int q = 1; q < n; ++q) {
    int x = init[q];
    int best_pos = 0;
    best = INFINITY;
    for (int p = 0; p <= len; ++p) {
      for (int i = 0, j = 0; i <= len; ++i) cand[i] = (i == p) ? x : out[j++];
      double m = oracle_rank_metrics(t, B, cand, len + 1, policy, NULL, NULL, scratch);
      ++evals;
      if (m < best) {
        best = m;
        best_pos = p;
      }
    }
    memmove(out + best_pos + 1, out + best_pos, sizeof(int) * (size_t)(len - best_pos));
    out[best_pos] = x;
    ++len;
  }
  double in_mk = oracle_rank_metrics(t, B, in, n, policy, NULL, NULL, scratch);
  ++evals;
  if (in_mk < best) memcpy(out, in, sizeof(int) * (size_t)n);
  free(init);
  free(cand);
  free(scratch);
  return evals;
}

/* ---- partition_batch (scheduling.py:202-264) ---------------------------- */
typedef struct {
  double crit, aux;
  int id, idx;
} lpt_key;

static int lpt_cmp(const void* a_, const void* b_) {
  const lpt_key* a = (const lpt_key*)a_;
  const lpt_key* b = (const lpt_key*)b_;
  /* key (-crit, -(up+down), id); Python sorted() is stable -> idx last */
  double ka = -a->crit, kb = -b->crit;
  if (ka < kb) return -1;
  if (ka > kb) return 1;
  ka = -a->aux;
  kb = -b->aux;
  if (ka < kb) return -1;
  if (ka > kb) return 1;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

#define MAX_SEC 16 /* MAESTRO_MAX_SECTIONS */
static int up_has(int u, int s) { return u == s || (u >= MAX_SEC && (((u - MAX_SEC) >> s) & 1)); }

/* up_sec/down_sec: resolved section index per sample or -1.  lists must hold B
 * ints (rank r's list starts at offsets[r]); counts[dp].  LPT order written to
 * lpt_out (optional).  aux load is tracked per (rank, section) in n_sec slots. */
int oracle_partition(const double* t, const int* ids, const int* up_sec, const int* down_sec,
                     int B, int dp, int n_sec, int* lists, int* offsets, int* counts,
                     int* lpt_out) {
  if (B <= 0) return 6;
  if (dp < 1) return 5;
  lpt_key* keys = (lpt_key*)malloc(sizeof(lpt_key) * (size_t)B);
  for (int i = 0; i < B; ++i) {
    keys[i].crit = T(F_C, i) + T(B_C, i);
    double up = T(F_BC, i) + T(B_AC, i);
    double down = T(F_AC, i) + T(B_BC, i);
    keys[i].aux = up + down;
    keys[i].id = ids[i];
    keys[i].idx = i;
  }
  qsort(keys, (size_t)B, sizeof(lpt_key), lpt_cmp);
  int base = B / dp, extra = B % dp;
  int off = 0;
  for (int r = 0; r < dp; ++r) {
    offsets[r] = off;
    counts[r] = 0;
    off += base + (r < extra ? 1 : 0);
  }
  double* crit_load = (double*)calloc((size_t)dp, sizeof(double));
  double* aux_load = (double*)calloc((size_t)dp * (size_t)n_sec, sizeof(double));
  for (int q = 0; q < B; ++q) {
    int i = keys[q].idx;
    if (lpt_out) lpt_out[q] = i;
    int nk = 0, ks[MAX_SEC + 1];
    double kt[MAX_SEC + 1];
    if (up_sec[i] >= MAX_SEC) {
      /* extension (parallel upstream sections, NOT IN REF): code MAX_SEC + section mask; the
       * sample's upstream time is charged to every activated upstream section, ascending */
      for (int s = 0; s < MAX_SEC; ++s)
        if (((up_sec[i] - MAX_SEC) >> s) & 1) { ks[nk] = s; kt[nk] = T(F_BC, i) + T(B_AC, i); ++nk; }
    } else if (up_sec[i] >= 0) { ks[nk] = up_sec[i]; kt[nk] = T(F_BC, i) + T(B_AC, i); ++nk; }
    if (down_sec[i] >= 0) { ks[nk] = down_sec[i]; kt[nk] = T(F_AC, i) + T(B_BC, i); ++nk; }
    int best = -1;
    double bc = 0.0, ba = 0.0;
    for (int r = 0; r < dp; ++r) {
      int cap = base + (r < extra ? 1 : 0);
      if (counts[r] >= cap) continue;
      double sa = 0.0; /* sum() starts from int 0: 0 + x == x exactly */
      for (int k = 0; k < nk; ++k) sa = sa + aux_load[(size_t)r * n_sec + ks[k]];
      if (best < 0 || crit_load[r] < bc || (crit_load[r] == bc && sa < ba)) {
        best = r;
        bc = crit_load[r];
        ba = sa;
      }
    }
    lists[offsets[best] + counts[best]++] = i;
    crit_load[best] += T(F_C, i) + T(B_C, i);
    for (int k = 0; k < nk; ++k) aux_load[(size_t)best * n_sec + ks[k]] += kt[k];
  }
  free(keys);
  free(crit_load);
  free(aux_load);
  return 0;
}

/* merge_fanout (scheduling.py:267-285): round-robin over `fanout` lists. */
int oracle_merge_fanout(const int* const* lists, const int* lens, int fanout, int* out) {
  int longest = 0, n = 0;
  for (int r = 0; r < fanout; ++r) longest = lens[r] > longest ? lens[r] : longest;
  for (int i = 0; i < longest; ++i)
    for (int r = 0; r < fanout; ++r)
      if (i < lens[r]) out[n++] = lists[r][i];
  return n;
}

/* build_schedule (scheduling.py:309-373) over resolved activations.
 * Section tables: dp[s], fanout[s], neighbor[s] (-1 for critical), merge_order
 * (n_aux auxiliaries by hop distance).  Output: for every section s and rank q,
 * the order is orders[s*B + sec_off[s*max_dp + q] ...] with length
 * sec_cnt[s*max_dp + q].  Returns 0 or an error code (8 = FanoutViolation,
 * with *bad_section set). */
int oracle_build_schedule(const double* t, const int* ids, const int* up_sec, const int* down_sec,
                          int B, int n_sec, int critical, const int* dp, const int* fanout,
                          const int* neighbor, const int* merge_order, int n_aux, int policy,
                          int max_dp, int* orders, int* sec_off, int* sec_cnt, long long* evals,
                          int* bad_section) {
  int dpc = dp[critical];
  int* lists = (int*)malloc(sizeof(int) * (size_t)B);
  int* offs = (int*)malloc(sizeof(int) * (size_t)dpc);
  int* cnts = (int*)malloc(sizeof(int) * (size_t)dpc);
  int rc = oracle_partition(t, ids, up_sec, down_sec, B, dpc, n_sec, lists, offs, cnts, NULL);
  if (rc) {
    free(lists); free(offs); free(cnts);
    return rc;
  }
  for (int s = 0; s < n_sec * max_dp; ++s) { sec_off[s] = 0; sec_cnt[s] = 0; }
  long long ev = 0;
  int* crit_out = orders + (size_t)critical * B;
  for (int r = 0; r < dpc; ++r) {
    ev += oracle_schedule_rank(t, B, lists + offs[r], cnts[r], policy, crit_out + offs[r]);
    sec_off[critical * max_dp + r] = offs[r];
    sec_cnt[critical * max_dp + r] = cnts[r];
  }
  if (evals) *evals = ev;
  int* filtered = (int*)malloc(sizeof(int) * (size_t)B);
  for (int a = 0; a < n_aux; ++a) {
    int s = merge_order[a], nb = neighbor[s];
    if (dp[s] * fanout[s] != dp[nb]) {
      if (bad_section) *bad_section = s;
      free(lists); free(offs); free(cnts); free(filtered);
      return 8;
    }
    int f = fanout[s];
    int pos = 0;
    for (int q = 0; q < dp[s]; ++q) {
      const int* sub[64];
      int lens[64];
      int fill = 0;
      for (int j = 0; j < f; ++j) {
        int r = q * f + j;
        const int* src = orders + (size_t)nb * B + sec_off[nb * max_dp + r];
        int n = sec_cnt[nb * max_dp + r];
        sub[j] = filtered + fill;
        lens[j] = 0;
        for (int k = 0; k < n; ++k) {
          int i = src[k];
          if (up_has(up_sec[i], s) || down_sec[i] == s) filtered[fill + lens[j]++] = i;
        }
        fill += lens[j];
      }
      int n = oracle_merge_fanout(sub, lens, f, orders + (size_t)s * B + pos);
      sec_off[s * max_dp + q] = pos;
      sec_cnt[s * max_dp + q] = n;
      pos += n;
    }
  }
  free(lists); free(offs); free(cnts); free(filtered);
  return 0;
}
