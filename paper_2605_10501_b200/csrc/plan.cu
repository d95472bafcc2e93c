// Device wavefront scheduler: K1 sample 6-tuples, K2 resolve + partition, K3 greedy
// insertion per critical rank, K4 fan-out merge, K5 varlen pack.
//
// Bit-exact with the reference's CPython fp64 arithmetic
// (/root/reference/pkg/src/maestro/scheduling.py, costs.py): this TU is compiled with
// --fmad=false, every max() is Python's first-maximal max (b > a ? b : a), sums follow
// the reference's left-to-right order, and ties break exactly like the reference's
// strict '<' scans and stable sorts.
#include "common.cuh"

namespace mb {
namespace {

enum { F_BC = 0, F_C = 1, F_AC = 2, B_BC = 3, B_C = 4, B_AC = 5 };

__device__ __forceinline__ double pmax(double a, double b) { return b > a ? b : a; }

// ---------------------------------------------------------------------------------------
// K1: per-sample 6-tuples from token counts.  costs.py:105-123 (estimate_step_time),
// costs.py:182-200 (per_sample_times), costs.py:264-286 (derive_batch per-side sums).
__device__ __forceinline__ void per_sample_times(const double* row, long long tokens, long long n,
                                                 double& fwd_out, double& bwd_out) {
  const double fpt = row[0], eff = row[1], ratio = row[2];
  const bool fwd_only = row[3] != 0.0;
  const long long mbs = (long long)row[4], pp = (long long)row[5];
  if (n <= 0) {
    fwd_out = 0.0;
    bwd_out = 0.0;
    return;
  }
  const double flops = (double)(mbs * tokens) * fpt;  // config.mbs * tokens * fpt
  const double fwd = flops / eff;                     // / (peak * tp * cp * eff), precomputed
  const double bwd = fwd_only ? 0.0 : fwd * ratio;
  const long long m = (n + mbs - 1) / mbs;            // ceil(samples / mbs)
  const double scale = (double)(m + pp - 1) / (double)(m * pp * mbs);
  fwd_out = fwd * scale;
  bwd_out = bwd * scale;
}

__global__ void __launch_bounds__(1024) sample_times_kernel(maestro_graph_t g, const double* __restrict__ cost,
                                                            const int32_t* __restrict__ tokens, int B,
                                                            double* __restrict__ times, uint32_t* __restrict__ act,
                                                            int64_t* err) {
  __shared__ int cnt[MAESTRO_MAX_SECTIONS];
  if (threadIdx.x < MAESTRO_MAX_SECTIONS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t crit_bits = g.sec_bits[g.critical];
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    uint32_t m = 0, secs = 0;
    for (int b = 0; b < g.n_bits; ++b) {
      if ((crit_bits >> b) & 1u) continue;
      if (tokens[(size_t)b * B + i] > 0) {
        m |= 1u << b;
        secs |= 1u << g.sub_owner[b];
      }
    }
    act[i] = m;
    while (secs) {  // activated-sample count per auxiliary (costs.py:262-263)
      int s = __ffs(secs) - 1;
      secs &= secs - 1;
      atomicAdd(&cnt[s], 1);
    }
  }
  __syncthreads();
  const double* crow = cost + (size_t)g.crit_bit * 8;
  const long long dpc = (long long)crow[6];
  const long long n_crit = ((long long)B + dpc - 1) / dpc;  // ceil(b / crit_cfg.dp)
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    double t[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const long long tc = tokens[(size_t)g.crit_bit * B + i];
    if (tc <= 0) {
      report(err, (uint32_t)i, MAESTRO_E_INVALID_DIMS, i);  // tokens_per_sample must be positive
      continue;
    }
    per_sample_times(crow, tc, n_crit, t[F_C], t[B_C]);
    uint32_t m = act[i];
    // parallel upstream sections (g.par_up): per-section upstream times, the sample's t_f_bc /
    // t_b_ac is the max over them (one activated bit per section, BothActivated otherwise, so
    // a single-section sample gets exactly the reference's 0 + fwd)
    double upf[MAESTRO_MAX_SECTIONS], upb[MAESTRO_MAX_SECTIONS];
    if (g.par_up)
      for (int s2 = 0; s2 < MAESTRO_MAX_SECTIONS; ++s2) upf[s2] = upb[s2] = 0.0;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int s = g.sub_owner[b];
      const double* row = cost + (size_t)b * 8;
      const long long dps = (long long)row[6];
      const long long n_aux = cnt[s] > 0 ? ((long long)cnt[s] + dps - 1) / dps : 0;
      double fwd, bwd;
      per_sample_times(row, tokens[(size_t)b * B + i], n_aux, fwd, bwd);
      if (g.side[s] == 0 && g.par_up) {
        upf[s] += fwd;
        upb[s] += bwd;
      } else if (g.side[s] == 0) {
        t[F_BC] += fwd;
        t[B_AC] += bwd;
      } else {
        t[F_AC] += fwd;
        t[B_BC] += bwd;
      }
    }
    if (g.par_up)
      for (int s2 = 0; s2 < g.n_sections; ++s2) {
        t[F_BC] = pmax(t[F_BC], upf[s2]);
        t[B_AC] = pmax(t[B_AC], upb[s2]);
      }
    bool bad = !(t[F_C] > 0.0);
    for (int p = 0; p < 6; ++p) bad |= !(t[p] >= 0.0) || isinf(t[p]);
    if (bad) report(err, (uint32_t)i, MAESTRO_E_NEGATIVE_TIME, i);
    for (int p = 0; p < 6; ++p) times[(size_t)p * B + i] = t[p] + 0.0;  // canonicalise -0.0
  }
}

// ---------------------------------------------------------------------------------------
// K2: resolve_activation (workload.py:297-355) + partition_batch (scheduling.py:202-264).
// One CTA.  Phase A resolves every sample and computes its LPT rank by counting (the sort
// key (-crit, -(up+down), id) plus batch index is a strict total order, so counting ranks
// reproduces Python's stable sorted()).  Phase B is the sequential greedy, run by warp 0 with
// one lane per pair of ranks and redux.sync argmins over the IEEE bit patterns
// (nonnegative doubles order like their bits).

struct LptSample {  // staged in smem in LPT order
  double crit, up, down;
  int up_sec, down_sec, idx;
};

__device__ __forceinline__ bool lpt_less(double ca, double aa, int ida, int ia, double cb, double ab, int idb,
                                         int ib) {
  const double ka = -ca, kb = -cb;
  if (ka != kb) return ka < kb;
  const double xa = -aa, xb = -ab;
  if (xa != xb) return xa < xb;
  if (ida != idb) return ida < idb;
  return ia < ib;
}

__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = __reduce_min_sync(kFull, (uint32_t)(v >> 32));
  const uint32_t lo = __reduce_min_sync(kFull, (uint32_t)(v >> 32) == hi ? (uint32_t)v : 0xffffffffu);
  return ((uint64_t)hi << 32) | lo;
}

__global__ void __launch_bounds__(1024) partition_kernel(maestro_graph_t g, const double* __restrict__ times,
                                                         const int32_t* __restrict__ ids,
                                                         const uint32_t* __restrict__ act, int B,
                                                         int32_t* __restrict__ up_out, int32_t* __restrict__ down_out,
                                                         int32_t* __restrict__ lpt_out, int32_t* __restrict__ part,
                                                         int32_t* __restrict__ part_off, int64_t* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LptSample* st = reinterpret_cast<LptSample*>(smem_raw);                       // [B]
  double* aux_load = reinterpret_cast<double*>(st + B);                          // [MAX_DP][n_sec]
  double* crit_load = aux_load + MAESTRO_MAX_DP * MAESTRO_MAX_SECTIONS;          // [MAX_DP]
  int* cnt = reinterpret_cast<int*>(crit_load + MAESTRO_MAX_DP);                 // [MAX_DP]
  int* cap = cnt + MAESTRO_MAX_DP;                                               // [MAX_DP]

  const int dp = g.dp[g.critical];
  const int n_sec = g.n_sections;
  const uint32_t prio_dup = (uint32_t)B, prio_act = (uint32_t)B + 1u;

  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const double fbc = times[(size_t)F_BC * B + i], fc = times[(size_t)F_C * B + i];
    const double fac = times[(size_t)F_AC * B + i], bbc = times[(size_t)B_BC * B + i];
    const double bc = times[(size_t)B_C * B + i], bac = times[(size_t)B_AC * B + i];
    const double crit = fc + bc, up_t = fbc + bac, down_t = fac + bbc;
    const double aux = up_t + down_t;
    const int id = ids[i];
    // LPT rank + duplicate ids (build_schedule checks duplicates first, scheduling.py:325-327)
    int rank = 0, dup = 0;
    for (int j = 0; j < B; ++j) {
      const double cj = times[(size_t)F_C * B + j] + times[(size_t)B_C * B + j];
      const double aj = (times[(size_t)F_BC * B + j] + times[(size_t)B_AC * B + j]) +
                        (times[(size_t)F_AC * B + j] + times[(size_t)B_BC * B + j]);
      const int idj = ids[j];
      rank += lpt_less(cj, aj, idj, j, crit, aux, id, i);
      dup += (idj == id) && (j != i);
    }
    if (dup) report(err, prio_dup, MAESTRO_E_INCONSISTENT, i);
    // resolve_activation: names walked in sorted order == ascending bits
    const uint32_t m = act[i];
    int code = 0;
    uint32_t up_secs = 0, down_secs = 0;
    for (int s = 0; s < n_sec; ++s) {
      const uint32_t bits = m & g.sec_bits[s];
      if (!bits) continue;
      if (__popc(bits) > 1) code = code ? code : MAESTRO_E_BOTH_ACTIVATED;
      if (g.side[s] == 0) up_secs |= 1u << s;
      if (g.side[s] == 2) down_secs |= 1u << s;
    }
    if (!code && ((__popc(up_secs) > 1 && !g.par_up) || __popc(down_secs) > 1)) code = MAESTRO_E_ACTIVATION;
    int up_sec = -1, down_sec = -1;
    if (!code && up_t > 0) {  // _attribute (workload.py:336-355)
      // several upstream sections (par_up): encoded MAESTRO_MAX_SECTIONS + section mask
      if (__popc(up_secs) > 1) up_sec = MAESTRO_MAX_SECTIONS + (int)up_secs;
      else if (up_secs) up_sec = __ffs(up_secs) - 1;
      else if (g.n_up == 1) up_sec = g.up_cand[0];
      else code = MAESTRO_E_ACTIVATION;
    }
    if (!code && down_t > 0) {
      if (down_secs) down_sec = __ffs(down_secs) - 1;
      else if (g.n_down == 1) down_sec = g.down_cand[0];
      else code = MAESTRO_E_ACTIVATION;
    }
    if (code) report(err, prio_act + (uint32_t)rank, code, i);
    up_out[i] = up_sec;
    down_out[i] = down_sec;
    lpt_out[rank] = i;
    LptSample s;
    s.crit = crit;
    s.up = up_t;
    s.down = down_t;
    s.up_sec = up_sec;
    s.down_sec = down_sec;
    s.idx = i;
    st[rank] = s;
  }
  for (int k = threadIdx.x; k < MAESTRO_MAX_DP * MAESTRO_MAX_SECTIONS; k += blockDim.x) aux_load[k] = 0.0;
  if (threadIdx.x < MAESTRO_MAX_DP) {
    const int r = threadIdx.x;
    crit_load[r] = 0.0;
    cnt[r] = 0;
    cap[r] = r < dp ? B / dp + (r < B % dp ? 1 : 0) : 0;  // equal-count capacities (:237-239)
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int off = 0;
    for (int r = 0; r < dp; ++r) {
      part_off[r] = off;
      off += cap[r];
    }
    part_off[dp] = off;
  }
  if (threadIdx.x >= 32) return;
  __syncwarp();
  const int lane = threadIdx.x;
  int off0 = 0, off1 = 0;
  for (int r = 0; r < lane; ++r) off0 += cap[r];
  for (int r = 0; r < lane + 32; ++r) off1 += cap[r];
  for (int q = 0; q < B; ++q) {
    const LptSample s = st[q];
    // lane owns ranks lane and lane+32; key (crit_load, sum of aux loads, r)  (:249-259)
    uint64_t kc = ~0ull, ka = ~0ull;
    int kr = 0x7fffffff;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (r >= dp || cnt[r] >= cap[r]) continue;
      double sa = 0.0;  // sum() starts from int 0; 0 + x == x
      if (s.up_sec >= MAESTRO_MAX_SECTIONS) {  // par_up: every activated upstream section, ascending
        for (uint32_t mm = (uint32_t)(s.up_sec - MAESTRO_MAX_SECTIONS); mm; mm &= mm - 1)
          sa = sa + aux_load[r * MAESTRO_MAX_SECTIONS + __ffs(mm) - 1];
      } else if (s.up_sec >= 0) {
        sa = sa + aux_load[r * MAESTRO_MAX_SECTIONS + s.up_sec];
      }
      if (s.down_sec >= 0) sa = sa + aux_load[r * MAESTRO_MAX_SECTIONS + s.down_sec];
      const uint64_t c = dbits(crit_load[r]), a = dbits(sa);
      if (c < kc || (c == kc && a < ka)) {  // r ascending: strict less keeps the smaller r
        kc = c;
        ka = a;
        kr = r;
      }
    }
    const uint64_t mc = warp_min_u64(kc);
    const uint64_t ma = warp_min_u64(kc == mc ? ka : ~0ull);
    const int best = (int)__reduce_min_sync(kFull, (kc == mc && ka == ma) ? (uint32_t)kr : 0xffffffffu);
    if (best == lane || best == lane + 32) {
      const int off = best == lane ? off0 : off1;
      part[off + cnt[best]] = s.idx;
      cnt[best] += 1;
      crit_load[best] += s.crit;
      if (s.up_sec >= MAESTRO_MAX_SECTIONS) {
        for (uint32_t mm = (uint32_t)(s.up_sec - MAESTRO_MAX_SECTIONS); mm; mm &= mm - 1)
          aux_load[best * MAESTRO_MAX_SECTIONS + __ffs(mm) - 1] += s.up;
      } else if (s.up_sec >= 0) {
        aux_load[best * MAESTRO_MAX_SECTIONS + s.up_sec] += s.up;
      }
      if (s.down_sec >= 0) aux_load[best * MAESTRO_MAX_SECTIONS + s.down_sec] += s.down;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------
// K3: schedule_rank (scheduling.py:162-199), one CTA per critical DP rank.
//
// Candidate p of an insertion step is res[:p] + [x] + res[p:]; thread p evaluates its
// makespan with the exact rank_metrics recurrence (scheduling.py:81-152).  The recurrence
// needs ub0 = the fp64 sum of all t_f_bc in candidate order before the main pass, so it is
// evaluated in passes over the candidate; all-fwd-then-bwd replays the forward pass as a
// shadow during the backward pass instead of storing per-sample chain values.
// Block argmin keeps the smallest p among equal makespans (Python's strict '<').

struct Sample6 {
  double fbc, fc, fac, bbc, bc, bac;
};

struct View {  // current partial order, SoA in smem
  const double* t[6];
  __device__ __forceinline__ Sample6 at(int j) const {
    Sample6 s;
    s.fbc = t[0][j];
    s.fc = t[1][j];
    s.fac = t[2][j];
    s.bbc = t[3][j];
    s.bc = t[4][j];
    s.bac = t[5][j];
    return s;
  }
};

// Visit candidate elements in order: view[0..p), x, view[p..len).  One loop of len + 1 steps
// with the element chosen by index (cur[j] before p, x at p, cur[j-1] after), so every thread of
// a warp runs the same trip count -- no divergent loop nests -- and the unrolled body issues the
// next elements' shared-memory loads ahead of the dependent fp64 recurrence.
template <class F>
__device__ __forceinline__ void for_candidate(const View& v, int len, int p, const Sample6& x, F&& f) {
#pragma unroll 4
  for (int j = 0; j <= len; ++j) {
    Sample6 s = v.at(j - (j > p ? 1 : 0));  // j == p reads a stale slot (< cap), replaced by x
    if (j == p) s = x;
    f(s);
  }
}

struct Metrics {
  double mk, busy, first, last;
  bool have_first;
};

// need_ub = false when no sample of the sequence has t_b_ac > 0 (e.g. a forward-only upstream
// section): ub is then never read, so the pass that computes its start value is skipped -- the
// makespan bits are unchanged.
template <int POLICY, bool WITH_METRICS, class Seq>
__device__ Metrics eval_order(Seq&& seq, bool need_ub = true) {
  // pass 1: u = sum of positive t_f_bc in order (ub starts there, scheduling.py:97)
  double u_total = 0.0;
  if (need_ub)
    seq([&](const Sample6& s) {
      if (s.fbc > 0) u_total += s.fbc;
    });
  Metrics m{0.0, 0.0, 0.0, 0.0, false};
  double c = 0.0, d = 0.0, ub = u_total, u = 0.0, mk = 0.0;
  auto crit = [&](double floor_, double ready, double dur) {
    const double start = pmax(floor_, ready);
    const double end = start + dur;
    c = end;
    if (WITH_METRICS) {
      if (!m.have_first) {
        m.first = start;
        m.have_first = true;
      }
      m.last = end;
      m.busy += dur;
    }
    return end;
  };
  if (POLICY == MAESTRO_POLICY_INTERLEAVED) {
    seq([&](const Sample6& s) {
      double ready = 0.0;
      if (s.fbc > 0) {
        u += s.fbc;
        ready = u;
      }
      double ch = crit(c, ready, s.fc);
      if (s.fac > 0) ch = d = pmax(d, ch) + s.fac;
      if (s.bbc > 0) ch = d = pmax(d, ch) + s.bbc;
      if (s.bc > 0) ch = crit(c, ch, s.bc);
      if (s.bac > 0) ch = ub = pmax(ub, ch) + s.bac;
      mk = pmax(mk, ch);
    });
  } else {
    // forward pass: critical + downstream forward stages
    seq([&](const Sample6& s) {
      double ready = 0.0;
      if (s.fbc > 0) {
        u += s.fbc;
        ready = u;
      }
      double ch = crit(c, ready, s.fc);
      if (s.fac > 0) ch = d = pmax(d, ch) + s.fac;
    });
    // backward pass; the shadow (us, cs, ds) replays the forward chain values
    double us = 0.0, cs = 0.0, ds = 0.0;
    seq([&](const Sample6& s) {
      double ready = 0.0;
      if (s.fbc > 0) {
        us += s.fbc;
        ready = us;
      }
      double ch = pmax(cs, ready) + s.fc;
      cs = ch;
      if (s.fac > 0) ch = ds = pmax(ds, ch) + s.fac;
      if (s.bbc > 0) ch = d = pmax(d, ch) + s.bbc;
      if (s.bc > 0) ch = crit(c, ch, s.bc);
      if (s.bac > 0) ch = ub = pmax(ub, ch) + s.bac;
      mk = pmax(mk, ch);
    });
  }
  m.mk = mk;
  return m;
}

// Interleaved policy, no downstream stage in the rank (no sample has t_f_ac or t_b_bc): the
// recurrence without branches.  Bit-exact with eval_order because, for these samples,
//  * u + 0.0 == u (so u is advanced unconditionally; ready = t_f_bc > 0 ? u : 0),
//  * the critical backward starts at pmax(c, ch) with ch == c, i.e. at c, and c + 0.0 == c,
//  * without a b_ac stage mk = pmax over a non-decreasing sequence of c = its last value.
// Candidate elements are {t_f_bc, t_f_c, t_b_c, t_b_ac} (AoS, two 16-byte loads per element).
template <bool UB>
__device__ __forceinline__ double eval_nodown(const double4* __restrict__ cur, int len, int p, const double4& x,
                                              double u_total) {
  double u = 0.0, c = 0.0, ub = u_total, mk = 0.0;
#pragma unroll 8
  for (int j = 0; j <= len; ++j) {
    double4 s = cur[j - (j > p ? 1 : 0)];
    if (j == p) s = x;
    u = u + s.x;
    const double ready = s.x > 0 ? u : 0.0;
    c = pmax(c, ready) + s.y;
    c = c + s.z;
    if (UB) {
      const double t = pmax(ub, c) + s.w;
      const bool has = s.w > 0;
      ub = has ? t : ub;
      mk = pmax(mk, has ? t : c);
    }
  }
  return UB ? mk : c;
}

__device__ __forceinline__ void argmin_combine(double& v, int& p, double ov, int op) {
  if (ov < v || (ov == v && op < p)) {
    v = ov;
    p = op;
  }
}

// MAXT: launch bound (256 for ranks of <= 255 samples: registers for the unrolled recurrence)
template <int POLICY, int MAXT>
__global__ void __launch_bounds__(MAXT) wavefront_kernel(const double* __restrict__ times, int B,
                                                         const int32_t* __restrict__ part,
                                                         const int32_t* __restrict__ part_off,
                                                         int32_t* __restrict__ orders, double* __restrict__ metrics,
                                                         int64_t* __restrict__ evals) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int r = blockIdx.x;
  const int base = part_off[r];
  const int n = part_off[r + 1] - base;
  const int32_t* in = part + base;
  const int cap = (int)blockDim.x;  // >= n + 1
  double* cur = reinterpret_cast<double*>(smem_raw);  // [6][cap]  current partial order
  double* stg = cur + 6 * cap;                        // [6][cap]  staged samples (init order)
  double4* cur4 = reinterpret_cast<double4*>(stg + 6 * cap);  // [cap] {fbc, fc, bc, bac} (fast path)
  int* ord = reinterpret_cast<int*>(cur4 + cap);      // [cap]     batch index per position
  int* init = ord + cap;                              // [cap]
  __shared__ double red_v[32];
  __shared__ int red_p[32];
  __shared__ int s_best;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (n <= 1) {  // scheduling.py:178-179
    if (tid == 0 && n == 1) {
      orders[base] = in[0];
      View v{{cur, cur + cap, cur + 2 * cap, cur + 3 * cap, cur + 4 * cap, cur + 5 * cap}};
      Sample6 s;
      const int i = in[0];
      s.fbc = times[i];
      s.fc = times[(size_t)B + i];
      s.fac = times[(size_t)2 * B + i];
      s.bbc = times[(size_t)3 * B + i];
      s.bc = times[(size_t)4 * B + i];
      s.bac = times[(size_t)5 * B + i];
      (void)v;
      Metrics m = eval_order<POLICY, true>([&](auto&& f) { f(s); });
      metrics[3 * r] = m.mk;
      metrics[3 * r + 1] = m.busy;
      metrics[3 * r + 2] = m.last - (m.have_first ? m.first : 0.0);
    }
    if (tid == 0) {
      evals[r] = 0;
      if (n == 0) {
        metrics[3 * r] = 0.0;
        metrics[3 * r + 1] = 0.0;
        metrics[3 * r + 2] = 0.0;
      }
    }
    return;
  }
  // sort_initial: stable ascending t_f_bc (scheduling.py:76-78), rank by counting
  if (tid < n) init[tid] = in[tid];
  __syncthreads();
  int my_rank = 0, my_idx = -1;
  if (tid < n) {
    my_idx = init[tid];
    const double f = times[my_idx];
    for (int j = 0; j < n; ++j) {
      const double fj = times[init[j]];
      my_rank += (fj < f) || (fj == f && j < tid);
    }
  }
  __syncthreads();
  if (tid < n) {
    init[my_rank] = my_idx;
    for (int p = 0; p < 6; ++p) stg[p * cap + my_rank] = times[(size_t)p * B + my_idx];
  }
  __syncthreads();
  View cv{{cur, cur + cap, cur + 2 * cap, cur + 3 * cap, cur + 4 * cap, cur + 5 * cap}};
  View sv{{stg, stg + cap, stg + 2 * cap, stg + 3 * cap, stg + 4 * cap, stg + 5 * cap}};
  // does any sample of this rank have a b_ac stage (the ub chain)?
  const bool need_ub = __syncthreads_or(tid < n && stg[5 * cap + tid] > 0.0) != 0;
  // no downstream stage anywhere in the rank: the branch-free interleaved recurrence (eval_nodown)
  const bool fast = POLICY == MAESTRO_POLICY_INTERLEAVED &&
                    __syncthreads_or(tid < n && (stg[2 * cap + tid] > 0.0 || stg[3 * cap + tid] > 0.0)) == 0;
  if (tid == 0) {
    ord[0] = init[0];
    for (int p = 0; p < 6; ++p) cur[p * cap] = stg[p * cap];
    cur4[0] = make_double4(stg[0], stg[cap], stg[4 * cap], stg[5 * cap]);
  }
  __syncthreads();
  double best_mk = 0.0;
  for (int len = 1; len < n; ++len) {
    const Sample6 x = sv.at(len);
    double v = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int pos = 0x7fffffff;
    if (tid <= len) {
      if (fast) {
        const double4 x4 = make_double4(x.fbc, x.fc, x.bc, x.bac);
        if (need_ub) {
          double u_total = 0.0;  // sum of t_f_bc in candidate order (ub starts there)
          for (int j = 0; j <= len; ++j) u_total = u_total + (j == tid ? x.fbc : cur4[j - (j > tid ? 1 : 0)].x);
          v = eval_nodown<true>(cur4, len, tid, x4, u_total);
        } else {
          v = eval_nodown<false>(cur4, len, tid, x4, 0.0);
        }
      } else {
        Metrics m = eval_order<POLICY, false>([&](auto&& f) { for_candidate(cv, len, tid, x, f); }, need_ub);
        v = m.mk;
      }
      pos = tid;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, v, o);
      const int op = __shfl_xor_sync(kFull, pos, o);
      argmin_combine(v, pos, ov, op);
    }
    if (lane == 0) {
      red_v[warp] = v;
      red_p[warp] = pos;
    }
    __syncthreads();
    if (warp == 0) {
      const int nw = (len + 1 + 31) >> 5;
      v = lane < nw ? red_v[lane] : __longlong_as_double(0x7ff0000000000000ll);
      pos = lane < nw ? red_p[lane] : 0x7fffffff;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, v, o);
        const int op = __shfl_xor_sync(kFull, pos, o);
        argmin_combine(v, pos, ov, op);
      }
      if (lane == 0) {
        s_best = pos;
        red_v[0] = v;
      }
    }
    __syncthreads();
    const int bp = s_best;
    best_mk = red_v[0];
    // res.insert(bp, x): shift [bp, len) right by one
    double keep[6];
    double4 keep4;
    int keep_idx = 0;
    const bool mover = tid >= bp && tid < len;
    if (mover) {
      for (int p = 0; p < 6; ++p) keep[p] = cur[p * cap + tid];
      keep4 = cur4[tid];
      keep_idx = ord[tid];
    }
    __syncthreads();
    if (mover) {
      for (int p = 0; p < 6; ++p) cur[p * cap + tid + 1] = keep[p];
      cur4[tid + 1] = keep4;
      ord[tid + 1] = keep_idx;
    }
    if (tid == 0) {
      cur4[bp] = make_double4(x.fbc, x.fc, x.bc, x.bac);
      cur[0 * cap + bp] = x.fbc;
      cur[1 * cap + bp] = x.fc;
      cur[2 * cap + bp] = x.fac;
      cur[3 * cap + bp] = x.bbc;
      cur[4 * cap + bp] = x.bc;
      cur[5 * cap + bp] = x.bac;
      ord[bp] = init[len];
    }
    __syncthreads();
  }
  // "return the input order if strictly better" (scheduling.py:197-199); stage input order
  if (tid < n) {
    const int i = in[tid];
    for (int p = 0; p < 6; ++p) stg[p * cap + tid] = times[(size_t)p * B + i];
  }
  __syncthreads();
  if (tid == 0) {
    Metrics mi = eval_order<POLICY, true>([&](auto&& f) {
      for (int j = 0; j < n; ++j) f(sv.at(j));
    });
    const bool use_input = mi.mk < best_mk;
    Metrics mo = mi;
    if (!use_input) {
      mo = eval_order<POLICY, true>([&](auto&& f) {
        for (int j = 0; j < n; ++j) f(cv.at(j));
      });
    }
    metrics[3 * r] = mo.mk;
    metrics[3 * r + 1] = mo.busy;
    metrics[3 * r + 2] = mo.last - (mo.have_first ? mo.first : 0.0);
    evals[r] = (int64_t)n * (n + 1) / 2;  // sum over steps of (len+1), plus the final check
    s_best = use_input;
  }
  __syncthreads();
  const bool use_input = s_best != 0;
  for (int k = tid; k < n; k += blockDim.x) orders[base + k] = use_input ? in[k] : ord[k];
}

// ---------------------------------------------------------------------------------------
// K4: auxiliary orders (scheduling.py:347-371).  One CTA.  For each auxiliary in merge
// order and each of its ranks q, the neighbour ranks q*f .. q*f+f-1 are one contiguous
// range of the neighbour's orders; each element is kept if the sample activates the
// auxiliary (ballot/popc compaction), and element c of list j lands at the round-robin
// position sum_j' min(len_j', c) + #{j' < j : len_j' > c}  (merge_fanout, :267-285).

__device__ int block_exclusive_scan(int flag, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(kFull, flag);
  const int pre = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int v = lane < nw ? warp_tot[lane] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane < nw) warp_tot[lane] = incl - v;
    if (lane == 31) warp_tot[32] = incl;
  }
  __syncthreads();
  const int res = warp_tot[warp] + pre;
  total = warp_tot[32];
  __syncthreads();
  return res;
}

// Does resolved upstream code u (section index, -1, or MAESTRO_MAX_SECTIONS + mask) include s?
__device__ __forceinline__ bool up_has(int u, int s) {
  return u == s || (u >= MAESTRO_MAX_SECTIONS && (((u - MAESTRO_MAX_SECTIONS) >> s) & 1));
}

__global__ void __launch_bounds__(1024) fanout_merge_kernel(maestro_graph_t g, int B,
                                                            const int32_t* __restrict__ up,
                                                            const int32_t* __restrict__ down,
                                                            const int32_t* __restrict__ part_off,
                                                            int32_t* __restrict__ orders,
                                                            int32_t* __restrict__ sec_off, int64_t* err) {
  __shared__ int warp_tot[33];
  __shared__ int list_len[MAESTRO_MAX_DP];
  __shared__ int list_base[MAESTRO_MAX_DP];  // compacted index of each list's first kept element
  constexpr int W = MAESTRO_MAX_DP + 1;
  const int tid = threadIdx.x;
  const int crit = g.critical;
  const int dpc = g.dp[crit];
  for (int r = tid; r <= dpc; r += blockDim.x) sec_off[crit * W + r] = part_off[r];
  __syncthreads();
  for (int a = 0; a < g.n_aux; ++a) {
    const int s = g.merge_order[a];
    const int nb = g.neighbor[s];
    const int f = g.fanout[s], dps = g.dp[s];
    if (dps * f != g.dp[nb]) {  // FanoutViolation (scheduling.py:361-365)
      if (tid == 0) report(err, 2u * (uint32_t)B + 2u + (uint32_t)a, MAESTRO_E_FANOUT_VIOLATION, s);
      return;
    }
    const int32_t* src = orders + (size_t)nb * B;
    int32_t* dst = orders + (size_t)s * B;
    int pos = 0;
    for (int q = 0; q < dps; ++q) {
      const int lo = sec_off[nb * W + q * f], hi = sec_off[nb * W + (q + 1) * f];
      if (tid < f) list_len[tid] = 0;
      __syncthreads();
      int carry = 0;
      // pass 1: list lengths
      for (int e0 = lo; e0 < hi; e0 += blockDim.x) {
        const int e = e0 + tid;
        int flag = 0, j = 0;
        if (e < hi) {
          const int i = src[e];
          flag = up_has(up[i], s) || (down[i] == s);
          while (j + 1 < f && sec_off[nb * W + q * f + j + 1] <= e) ++j;
        }
        if (flag) atomicAdd(&list_len[j], 1);
      }
      __syncthreads();
      if (tid == 0) {
        int acc = 0;
        for (int j = 0; j < f; ++j) {
          list_base[j] = acc;
          acc += list_len[j];
        }
      }
      __syncthreads();
      // pass 2: compacted index (block scan) -> round-robin position
      for (int e0 = lo; e0 < hi; e0 += blockDim.x) {
        const int e = e0 + tid;
        int flag = 0, j = 0, i = -1;
        if (e < hi) {
          i = src[e];
          flag = up_has(up[i], s) || (down[i] == s);
          while (j + 1 < f && sec_off[nb * W + q * f + j + 1] <= e) ++j;
        }
        int total;
        const int g_idx = carry + block_exclusive_scan(flag, warp_tot, total);
        carry += total;
        if (flag) {
          const int c = g_idx - list_base[j];
          int p = 0;
          for (int jj = 0; jj < f; ++jj) {
            const int L = list_len[jj];
            p += L < c ? L : c;
            p += (jj < j && L > c) ? 1 : 0;
          }
          dst[pos + p] = i;
        }
      }
      if (tid == 0) sec_off[s * W + q] = pos;
      int tot = 0;
      for (int j = 0; j < f; ++j) tot += list_len[j];
      pos += tot;
      __syncthreads();
    }
    if (tid == 0) sec_off[s * W + dps] = pos;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// K5: varlen pack of one rank's order.  Token offsets are an exclusive prefix scan of the
// sequence lengths in schedule order (one CTA, carry across 1024-sample chunks);
// consecutive groups of `mbs` samples form micro-batches with their own cu_seqlens.
__global__ void __launch_bounds__(1024) varlen_pack_kernel(const int32_t* __restrict__ order, int n,
                                                           const int32_t* __restrict__ len, int mbs,
                                                           int32_t* __restrict__ mb, int32_t* __restrict__ tok_off,
                                                           int32_t* __restrict__ mb_tokens, int32_t* __restrict__ cu,
                                                           int32_t* __restrict__ mb_start) {
  __shared__ int wsum[33];
  __shared__ int carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int k0 = 0; k0 < n; k0 += blockDim.x) {
    const int k = k0 + threadIdx.x;
    const int l = k < n ? len[order[k]] : 0;
    int incl = l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      const int v = lane < nw ? wsum[lane] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane < nw) wsum[lane] = x - v;
      if (lane == 31) wsum[32] = x;
    }
    __syncthreads();
    const int carry = carry_s;
    if (k < n) {
      tok_off[k] = carry + wsum[warp] + incl - l;
      mb[k] = k / mbs;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + wsum[32];
    __syncthreads();
  }
  const int n_mb = (n + mbs - 1) / mbs;
  for (int m = threadIdx.x; m < n_mb; m += blockDim.x) {
    const int k0 = m * mbs, k1 = min(n, k0 + mbs);
    const int base = tok_off[k0];
    mb_start[m] = base;
    cu[m * (mbs + 1)] = 0;
    for (int k = k0; k < k1; ++k) cu[m * (mbs + 1) + (k - k0) + 1] = tok_off[k] + len[order[k]] - base;
    for (int k = k1 - k0; k < mbs; ++k) cu[m * (mbs + 1) + k + 1] = cu[m * (mbs + 1) + (k1 - k0)];
    mb_tokens[m] = cu[m * (mbs + 1) + mbs];
  }
}

// Token ids of the ordered samples into one packed stream: out[tok_off[k] + j] = ids[order[k], j].
__global__ void pack_tokens_kernel(const int32_t* __restrict__ ids, int ld, const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ len, const int32_t* __restrict__ tok_off, int n,
                                   int32_t* __restrict__ out) {
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int i = order[k];
    const int32_t* src = ids + (size_t)i * ld;
    int32_t* dst = out + tok_off[k];
    for (int j = threadIdx.x; j < len[i]; j += blockDim.x) dst[j] = src[j];
  }
}

template <int POLICY>
__global__ void rank_metrics_kernel(const double* __restrict__ times, int B, const int32_t* __restrict__ order,
                                    int n, double* __restrict__ out) {
  Metrics m = eval_order<POLICY, true>([&](auto&& f) {
    for (int k = 0; k < n; ++k) {
      const int i = order[k];
      Sample6 s;
      s.fbc = times[i];
      s.fc = times[(size_t)B + i];
      s.fac = times[(size_t)2 * B + i];
      s.bbc = times[(size_t)3 * B + i];
      s.bc = times[(size_t)4 * B + i];
      s.bac = times[(size_t)5 * B + i];
      f(s);
    }
  });
  out[0] = n > 0 ? m.mk : 0.0;
  out[1] = m.busy;
  out[2] = m.last - (m.have_first ? m.first : 0.0);
}

__global__ void error_reset_kernel(int64_t* err) { *err = 0x7fffffffffffffffll; }

size_t partition_smem(int B) {
  return (size_t)B * sizeof(LptSample) + sizeof(double) * (MAESTRO_MAX_DP * MAESTRO_MAX_SECTIONS + MAESTRO_MAX_DP) +
         sizeof(int) * 2 * MAESTRO_MAX_DP;
}

int wavefront_threads(int max_n) { return ((max_n + 1 + 31) / 32) * 32; }

size_t wavefront_smem(int threads) { return (size_t)threads * (16 * sizeof(double) + 2 * sizeof(int)); }

}  // namespace
}  // namespace mb

using namespace mb;

MAESTRO_API int maestro_error_reset(int64_t* d_err, void* stream) {
  error_reset_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_err);
  return launch_status();
}

MAESTRO_API int maestro_rank_metrics(const double* d_times, int32_t B, const int32_t* d_order, int32_t n,
                                     int32_t policy, double* d_out, void* stream) {
  if (policy == MAESTRO_POLICY_INTERLEAVED)
    rank_metrics_kernel<0><<<1, 1, 0, (cudaStream_t)stream>>>(d_times, B, d_order, n, d_out);
  else
    rank_metrics_kernel<1><<<1, 1, 0, (cudaStream_t)stream>>>(d_times, B, d_order, n, d_out);
  return launch_status();
}

MAESTRO_API int maestro_sample_times(const maestro_graph_t* g, const double* d_cost, const int32_t* d_tokens,
                                     int32_t B, double* d_times, uint32_t* d_act, int64_t* d_err, void* stream) {
  if (B <= 0 || B > MAESTRO_MAX_BATCH) return (int)cudaErrorInvalidValue;
  sample_times_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(*g, d_cost, d_tokens, B, d_times, d_act, d_err);
  return launch_status();
}

MAESTRO_API int maestro_partition(const maestro_graph_t* g, const double* d_times, const int32_t* d_ids,
                                  const uint32_t* d_act, int32_t B, int32_t* d_up, int32_t* d_down,
                                  int32_t* d_lpt, int32_t* d_part, int32_t* d_part_off, int64_t* d_err,
                                  void* stream) {
  if (B <= 0 || B > MAESTRO_MAX_BATCH) return (int)cudaErrorInvalidValue;
  const int dp = g->dp[g->critical];
  if (dp < 1 || dp > MAESTRO_MAX_DP) return (int)cudaErrorInvalidValue;
  const size_t smem = partition_smem(B);
  if (ensure_smem<partition_kernel>(smem)) return launch_status();
  partition_kernel<<<1, 1024, smem, (cudaStream_t)stream>>>(*g, d_times, d_ids, d_act, B, d_up, d_down, d_lpt,
                                                            d_part, d_part_off, d_err);
  return launch_status();
}

MAESTRO_API int maestro_wavefront(const double* d_times, int32_t B, const int32_t* d_part,
                                  const int32_t* d_part_off, int32_t dp, int32_t policy, int32_t* d_orders,
                                  double* d_metrics, int64_t* d_evals, void* stream) {
  // blockDim must cover the largest rank (+1 insertion slot): ranks differ by at most one
  // sample, so ceil(B / dp) bounds them without reading part_off back.
  const int max_n = (B + dp - 1) / dp;
  if (max_n > MAESTRO_MAX_RANK_SAMPLES) return (int)cudaErrorInvalidValue;
  const int threads = wavefront_threads(max_n);
  const size_t smem = wavefront_smem(threads);
#define WF_LAUNCH(P, T)                                                                                  \
  do {                                                                                                   \
    if (ensure_smem<wavefront_kernel<P, T>>(smem)) return launch_status();                               \
    wavefront_kernel<P, T><<<dp, threads, smem, (cudaStream_t)stream>>>(d_times, B, d_part, d_part_off, \
                                                                       d_orders, d_metrics, d_evals);    \
  } while (0)
  const bool small = threads <= 256;
  if (policy == MAESTRO_POLICY_INTERLEAVED) {
    if (small) WF_LAUNCH(0, 256);
    else WF_LAUNCH(0, 1024);
  } else {
    if (small) WF_LAUNCH(1, 256);
    else WF_LAUNCH(1, 1024);
  }
#undef WF_LAUNCH
  return launch_status();
}

static int fanout_merge_impl(const maestro_graph_t* g, int32_t B, const int32_t* d_up, const int32_t* d_down,
                             const int32_t* d_part_off, int32_t* d_orders, int32_t* d_sec_off, int64_t* d_err,
                             void* stream) {
  fanout_merge_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(*g, B, d_up, d_down, d_part_off, d_orders,
                                                            d_sec_off, d_err);
  return launch_status();
}

MAESTRO_API int maestro_fanout_merge(const maestro_graph_t* g, int32_t B, const int32_t* d_up,
                                     const int32_t* d_down, int32_t* d_orders, int32_t* d_sec_off, int64_t* d_err,
                                     void* stream) {
  // critical offsets already in d_sec_off: pass them as part_off (kernel copies onto itself)
  const int W = MAESTRO_MAX_DP + 1;
  return fanout_merge_impl(g, B, d_up, d_down, d_sec_off + g->critical * W, d_orders, d_sec_off, d_err, stream);
}

MAESTRO_API int64_t maestro_schedule_workspace(int32_t B, int32_t dp_critical) {
  return (int64_t)sizeof(int32_t) * (4 * (int64_t)B + dp_critical + 1);
}

MAESTRO_API int maestro_build_schedule(const maestro_graph_t* g, const double* d_times, const int32_t* d_ids,
                                       const uint32_t* d_act, int32_t B, int32_t policy, int32_t* d_orders,
                                       int32_t* d_sec_off, double* d_metrics, int64_t* d_evals, void* d_work,
                                       int64_t* d_err, void* stream) {
  int32_t* w = (int32_t*)d_work;
  int32_t *up = w, *down = w + B, *lpt = w + 2 * B, *part = w + 3 * B, *part_off = w + 4 * B;
  int rc = maestro_partition(g, d_times, d_ids, d_act, B, up, down, lpt, part, part_off, d_err, stream);
  if (rc) return rc;
  const int crit = g->critical;
  rc = maestro_wavefront(d_times, B, part, part_off, g->dp[crit], policy, d_orders + (size_t)crit * B, d_metrics,
                         d_evals, stream);
  if (rc) return rc;
  return fanout_merge_impl(g, B, up, down, part_off, d_orders, d_sec_off, d_err, stream);
}

MAESTRO_API int maestro_varlen_pack(const int32_t* d_order, int32_t n, const int32_t* d_len, int32_t mbs,
                                    int32_t* d_mb, int32_t* d_tok_off, int32_t* d_mb_tokens, int32_t* d_cu,
                                    int32_t* d_mb_start, void* stream) {
  if (n <= 0) return 0;
  varlen_pack_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(d_order, n, d_len, mbs, d_mb, d_tok_off, d_mb_tokens, d_cu,
                                                            d_mb_start);
  return launch_status();
}

MAESTRO_API int maestro_pack_tokens(const int32_t* d_ids, int32_t ld, const int32_t* d_order, const int32_t* d_len,
                                    const int32_t* d_tok_off, int32_t n, int32_t* d_out, void* stream) {
  if (n <= 0) return 0;
  pack_tokens_kernel<<<n < 1024 ? n : 1024, 256, 0, (cudaStream_t)stream>>>(d_ids, ld, d_order, d_len, d_tok_off, n,
                                                                            d_out);
  return launch_status();
}
