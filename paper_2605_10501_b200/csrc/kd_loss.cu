// K9: fused knowledge-distillation loss over the full vocabulary.
//
// Per token row:  KL(p_t || p_s) = sum_v p_t (t - s) - lse(t) + lse(s),   p = softmax(logits / tau)
// and its gradient w.r.t. the student logits  ds = g / tau * (softmax(s/tau) - softmax(t/tau)).
// The teacher's output layer is colocated with the student (workload.py:471-514), so both
// logit rows are produced in the student section; no probabilities are ever materialised.
// Pass 1 streams both rows once keeping online (max, sum-exp) for t and s plus the running
// sum_v e^{t-m}(t - s); pass 2 re-reads the rows (L2-resident: a CTA's row is < 0.6 MB and
// just touched) and writes ds.  HBM traffic ~ 2 x V x 2 B read + V x 2 B written per token.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace mb {
namespace {

constexpr int KD_THREADS = 512;
#ifndef KD_EMU_BITS
#define KD_EMU_BITS 0x00  // elements j of each 8-vector whose exponential pair runs on the FMA pipe (measured: no gain, MUFU is not the bound)
#endif
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// 2^x on the MUFU unit without exp2f's range fix-ups (arguments here are <= 0 or bounded)
__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Stat {  // online stats in the log2 domain
  float mt, st, at, ms, ss;
};

__device__ __forceinline__ void merge(Stat& a, const Stat& b) {
  if (b.mt != -INFINITY) {
    if (a.mt == -INFINITY) {
      a.mt = b.mt;
      a.st = b.st;
      a.at = b.at;
    } else {
      const float mt = fmaxf(a.mt, b.mt);
      const float ca = ex2a(a.mt - mt), cb = ex2a(b.mt - mt);
      a.st = a.st * ca + b.st * cb;
      a.at = a.at * ca + b.at * cb;
      a.mt = mt;
    }
  }
  if (b.ms != -INFINITY) {
    if (a.ms == -INFINITY) {
      a.ms = b.ms;
      a.ss = b.ss;
    } else {
      const float ms = fmaxf(a.ms, b.ms);
      a.ss = a.ss * ex2a(a.ms - ms) + b.ss * ex2a(b.ms - ms);
      a.ms = ms;
    }
  }
}

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 x = __bfloat1622float2(h[j]);
    f[2 * j] = x.x;
    f[2 * j + 1] = x.y;
  }
}

template <int THREADS, int MIN_BLOCKS, int UNROLL>
__global__ void __launch_bounds__(THREADS, MIN_BLOCKS) kd_loss_kernel(const __nv_bfloat16* __restrict__ tl,
                                                             const __nv_bfloat16* sl,
                                                             __nv_bfloat16* ds,  // may alias sl
                                                             float* __restrict__ loss,
                                                             int T, int V, int ldt, int lds, int ldd, float scale2,
                                                             float grad_scale, float inv_tau) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  __shared__ Stat red[THREADS / 32];
  __shared__ Stat fin;
  const int nvec = V / 8;
  for (int row = blockIdx.x; row < T; row += gridDim.x) {
    const uint4* t4 = reinterpret_cast<const uint4*>(tl + (size_t)row * ldt);
    const uint4* s4 = reinterpret_cast<const uint4*>(sl + (size_t)row * lds);
    Stat a{-INFINITY, 0.f, 0.f, -INFINITY, 0.f};
    // four vectors per step (their loads are independent of the running stats, so they are all
    // in flight together); the running max is only rescaled when it grows, which after the first
    // few vectors of a row is rare -- the exponentials are what bounds this kernel next to HBM
    for (int v0 = threadIdx.x; v0 < nvec; v0 += UNROLL * THREADS) {
      uint4 rt[UNROLL], rs[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int v = v0 + u * THREADS;
        if (v < nvec) {
          rt[u] = t4[v];
          rs[u] = s4[v];
        }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (v0 + u * THREADS >= nvec) break;
        float ft[8], fs[8];
        unpack8(rt[u], ft);
        unpack8(rs[u], fs);
        // max of the raw logits, scaled once (scale2 > 0: exact)
        float rt = ft[0], rs = fs[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) {
          rt = fmaxf(rt, ft[j]);
          rs = fmaxf(rs, fs[j]);
        }
        const float mt = fmaxf(a.mt, rt * scale2), ms = fmaxf(a.ms, rs * scale2);
        if (mt > a.mt) {  // a.mt == -inf: st = at = 0, any finite factor is fine
          const float ct = a.mt == -INFINITY ? 0.f : ex2a(a.mt - mt);
          a.st *= ct;
          a.at *= ct;
          a.mt = mt;
        }
        if (ms > a.ms) {
          a.ss *= a.ms == -INFINITY ? 0.f : ex2a(a.ms - ms);
          a.ms = ms;
        }
        // teacher and student exponentials of element j as one pair: paired FMA/add, and
        // KD_EMU_BITS of the pairs on the FMA pipe (degree-5 polynomial, fp32-accurate)
        float2 sts = make_float2(a.st, a.ss);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 x = __ffma2_rn(make_float2(ft[j], fs[j]), make_float2(scale2, scale2), make_float2(-mt, -ms));
          const float2 e = ((KD_EMU_BITS >> j) & 1) ? ex2_fma2<5>(x) : make_float2(ex2a(x.x), ex2a(x.y));
          sts = __fadd2_rn(sts, e);
          a.at = fmaf(e.x, ft[j] - fs[j], a.at);
        }
        a.st = sts.x;
        a.ss = sts.y;
      }
    }
    // block reduction of the online stats
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Stat b{__shfl_xor_sync(kFull, a.mt, o), __shfl_xor_sync(kFull, a.st, o), __shfl_xor_sync(kFull, a.at, o),
             __shfl_xor_sync(kFull, a.ms, o), __shfl_xor_sync(kFull, a.ss, o)};
      merge(a, b);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
      a = threadIdx.x < THREADS / 32 ? red[threadIdx.x] : Stat{-INFINITY, 0.f, 0.f, -INFINITY, 0.f};
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Stat b{__shfl_xor_sync(kFull, a.mt, o), __shfl_xor_sync(kFull, a.st, o), __shfl_xor_sync(kFull, a.at, o),
               __shfl_xor_sync(kFull, a.ms, o), __shfl_xor_sync(kFull, a.ss, o)};
        merge(a, b);
      }
      if (threadIdx.x == 0) {
        fin = a;
        // lse in natural units of the tempered logits: (m2 + log2 S) * ln 2
        const float lse_t = (a.mt + log2f(a.st)) * LN2;
        const float lse_s = (a.ms + log2f(a.ss)) * LN2;
        // sum p_t (t - s)/tau - lse_t + lse_s
        loss[row] = a.at / a.st * inv_tau - lse_t + lse_s;
      }
    }
    __syncthreads();
    if (ds != nullptr) {
      const Stat f = fin;
      const float it = 1.f / f.st, is = 1.f / f.ss;
      const float g = grad_scale * inv_tau;
      uint4* d4 = reinterpret_cast<uint4*>(ds + (size_t)row * ldd);
      for (int v = threadIdx.x; v < nvec; v += THREADS) {
        float ft[8], fs[8];
        unpack8(t4[v], ft);
        unpack8(s4[v], fs);
        uint4 o;
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
        float gg[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 x = __ffma2_rn(make_float2(fs[j], ft[j]), make_float2(scale2, scale2), make_float2(-f.ms, -f.mt));
          const float2 e = __fmul2_rn(((KD_EMU_BITS >> j) & 1) ? ex2_fma2<5>(x) : make_float2(ex2a(x.x), ex2a(x.y)),
                                      make_float2(is, it));
          gg[j] = g * (e.x - e.y);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) oh[j] = __floats2bfloat162_rn(gg[2 * j], gg[2 * j + 1]);
        d4[v] = o;
      }
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------------------------
// Shared-memory-resident K9.  A token row is read from HBM exactly once: a cluster of C CTAs
// (three per SM, so row slices in different phases overlap) holds the row, CTA c owning columns
// [c*VC, c*VC + VC), VC <= 16384, as eight 2048-column chunks of (t, s) bf16 = 64 KB, filled by
// 1-D TMA bulk copies from a producer warp.
//   pass 1 (as chunks land): per thread one 8-column vector of t and s per chunk; online (max,
//          sum-exp) of both plus sum e^t (t - s); the exponentials are written back IN PLACE as
//          fp16 (relative to the thread's running max at that chunk, kept in registers), so
//          pass 2 needs no exponentials: MUFU work is 2 per column instead of 4.
//   stats: warp/CTA reduction, then each CTA pushes its partial into every cluster peer's
//          shared memory (st.shared::cluster + remote mbarrier arrive); every CTA merges the C
//          partials in rank order (identical bits everywhere).
//   pass 2: ds = g (e_s 2^(m_s,k - M_s)/S_s - e_t 2^(m_t,k - M_t)/S_t), bf16 stores; each chunk is
//          released to the producer as soon as it is consumed, so row r+1 streams in behind
//          row r's pass 2.
// HBM traffic is the algorithmic 2 x V x 2 B read + V x 2 B written per row.  fp16 storage of
// the exponentials (all <= 1) adds a relative error <= 2^-12 per probability to ds (which is then
// rounded to bf16, 2^-9); the loss uses the fp32 exponentials.
#ifndef KDS_CONS_T
#define KDS_CONS_T 256
#endif
#ifndef KDS_CTAS
#define KDS_CTAS 3
#endif
constexpr int KDS_CONS = KDS_CONS_T;       // consumer threads: one 8-column vector per chunk each
constexpr int KDS_CH = 8 * KDS_CONS;       // columns per chunk
constexpr int KDS_NCH = 8;                 // chunks per CTA slice
constexpr int KDS_VC_MAX = KDS_CH * KDS_NCH;  // 16384 columns = 64 KB of (t, s) per CTA
constexpr int KDS_THREADS = KDS_CONS + 32; // + producer warp
constexpr int KDS_SMEM = KDS_NCH * KDS_CH * 4 + 1024;
constexpr int KDS_CTAS_PER_SM = KDS_CTAS;  // row slices in flight per SM (different phases)
#ifndef KDS_SLEEP_NS
#define KDS_SLEEP_NS 20000
#endif

// Cluster-scope acquire wait with a suspend-time hint: the waiting threads sleep until the phase
// completes instead of re-polling (each poll at cluster scope also invalidates L1: CCTL).
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, "
      "0, p;\n}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "n"(KDS_SLEEP_NS)
      : "memory");
  return ok != 0;
}
// chunk barriers: sleep on the barrier rather than spin (the kernel is issue-bound; spinning
// consumer and producer warps took a third of the issue slots)
__device__ __forceinline__ void kds_wait(uint64_t* bar, uint32_t parity) { sm100::mbar_wait_sleep<KDS_SLEEP_NS>(bar, parity); }
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

template <int C>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(KDS_THREADS, KDS_CTAS_PER_SM)
    kd_loss_smem_kernel(const __nv_bfloat16* __restrict__ tl, const __nv_bfloat16* sl, __nv_bfloat16* ds,
                        float* __restrict__ loss, int T, int V, int VC, int ldt, int lds, int ldd, float scale2,
                        float grad_scale, float inv_tau) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  using namespace sm100;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  // chunk k: t at sm + k * 16 KB, s at + 8 KB
  __shared__ __align__(8) uint64_t full[KDS_NCH], empty[KDS_NCH], stats_bar[2];
  __shared__ Stat red[KDS_CONS / 32];
  __shared__ float slot[2][C][8];  // [row parity][source rank] partial stats
  const int rank = C > 1 ? (int)cluster_ctarank() : 0;
  const int n_clusters = gridDim.x / C, cid = blockIdx.x / C;
  const int c0 = rank * VC;
  const int cols = max(0, min(V - c0, VC));  // this CTA's slice width (multiple of 8)
  const int nch = (cols + KDS_CH - 1) / KDS_CH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int k = 0; k < KDS_NCH; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], KDS_CONS / 32);
    }
    mbar_init(&stats_bar[0], C);
    mbar_init(&stats_bar[1], C);
    fence_barrier_init();
  }
  if constexpr (C > 1) cluster_sync();  // peers' barriers initialised before any remote arrive
  else __syncthreads();

  if (warp == KDS_CONS / 32) {  // producer
    if (lane == 0) {
      int it = 0;
      for (int row = cid; row < T; row += n_clusters, ++it) {
        const __nv_bfloat16* tr = tl + (size_t)row * ldt + c0;
        const __nv_bfloat16* sr = sl + (size_t)row * lds + c0;
        for (int k = 0; k < nch; ++k) {
          const int w = min(KDS_CH, cols - k * KDS_CH);
          kds_wait(&empty[k], (it & 1) ^ 1);
          mbar_arrive_expect_tx(&full[k], 4u * (uint32_t)w);
          bulk_load_1d(sm + k * (KDS_CH * 4), tr + k * KDS_CH, 2u * (uint32_t)w, &full[k]);
          bulk_load_1d(sm + k * (KDS_CH * 4) + KDS_CH * 2, sr + k * KDS_CH, 2u * (uint32_t)w, &full[k]);
        }
      }
    }
  } else {
    const int tid = threadIdx.x;
    int it = 0;
    for (int row = cid; row < T; row += n_clusters, ++it) {
      const uint32_t ph = it & 1;
      Stat a{-INFINITY, 0.f, 0.f, -INFINITY, 0.f};
      float mh_t[KDS_NCH], mh_s[KDS_NCH];
      // ---- pass 1
#pragma unroll
      for (int k = 0; k < KDS_NCH; ++k) {
        mh_t[k] = mh_s[k] = 0.f;
        if (k >= nch) break;
        kds_wait(&full[k], ph);
        const bool mine = k * KDS_CH + 8 * tid < cols;
        uint4* pt = reinterpret_cast<uint4*>(sm + k * (KDS_CH * 4)) + tid;
        uint4* ps = reinterpret_cast<uint4*>(sm + k * (KDS_CH * 4) + KDS_CH * 2) + tid;
        if (mine) {
          float ft[8], fs[8];
          unpack8(*pt, ft);
          unpack8(*ps, fs);
          // max of the raw logits, scaled once (scale2 > 0); three-input max pairs
          float rt = fmaxf(fmaxf(ft[0], ft[1]), fmaxf(ft[2], ft[3]));
          float rs = fmaxf(fmaxf(fs[0], fs[1]), fmaxf(fs[2], fs[3]));
          rt = fmaxf(rt, fmaxf(fmaxf(ft[4], ft[5]), fmaxf(ft[6], ft[7])));
          rs = fmaxf(rs, fmaxf(fmaxf(fs[4], fs[5]), fmaxf(fs[6], fs[7])));
          const float mt = fmaxf(a.mt, rt * scale2), ms = fmaxf(a.ms, rs * scale2);
          if (mt > a.mt) {
            const float ct = a.mt == -INFINITY ? 0.f : ex2a(a.mt - mt);
            a.st *= ct;
            a.at *= ct;
            a.mt = mt;
          }
          if (ms > a.ms) {
            a.ss *= a.ms == -INFINITY ? 0.f : ex2a(a.ms - ms);
            a.ms = ms;
          }
          mh_t[k] = mt;
          mh_s[k] = ms;
          float2 sts = make_float2(a.st, a.ss);
          float2 at2 = make_float2(a.at, 0.f);  // sum e_t (t - s), two partial sums (paired FMA)
          uint32_t et[4], es[4];
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const float2 x0 = __ffma2_rn(make_float2(ft[j], fs[j]), make_float2(scale2, scale2), make_float2(-mt, -ms));
            const float2 x1 =
                __ffma2_rn(make_float2(ft[j + 1], fs[j + 1]), make_float2(scale2, scale2), make_float2(-mt, -ms));
            const float2 e0 = make_float2(ex2a(x0.x), ex2a(x0.y));
            const float2 e1 = make_float2(ex2a(x1.x), ex2a(x1.y));
            sts = __fadd2_rn(__fadd2_rn(sts, e0), e1);
            const float2 d = __fadd2_rn(make_float2(ft[j], ft[j + 1]), make_float2(-fs[j], -fs[j + 1]));
            at2 = __ffma2_rn(make_float2(e0.x, e1.x), d, at2);
            if (ds != nullptr) {
              const __half2 ht = __floats2half2_rn(e0.x, e1.x), hs = __floats2half2_rn(e0.y, e1.y);
              et[j >> 1] = *reinterpret_cast<const uint32_t*>(&ht);
              es[j >> 1] = *reinterpret_cast<const uint32_t*>(&hs);
            }
          }
          a.st = sts.x;
          a.ss = sts.y;
          a.at = at2.x + at2.y;
          if (ds != nullptr) {
            *pt = make_uint4(et[0], et[1], et[2], et[3]);
            *ps = make_uint4(es[0], es[1], es[2], es[3]);
          }
        }
        if (ds == nullptr) {  // loss only: the chunk is free once read
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[k]);
        }
      }
      // ---- row statistics: warp -> CTA -> cluster (every CTA merges the C partials in rank order)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Stat b{__shfl_xor_sync(kFull, a.mt, o), __shfl_xor_sync(kFull, a.st, o), __shfl_xor_sync(kFull, a.at, o),
               __shfl_xor_sync(kFull, a.ms, o), __shfl_xor_sync(kFull, a.ss, o)};
        merge(a, b);
      }
      if (lane == 0) red[warp] = a;
      named_barrier_sync(1, KDS_CONS);
      if (tid == 0) {
        Stat b = red[0];
        for (int w = 1; w < KDS_CONS / 32; ++w) merge(b, red[w]);
        const float v[5] = {b.mt, b.st, b.at, b.ms, b.ss};
        for (int q = 0; q < C; ++q) {
          const uint32_t dst = smem_u32(&slot[ph][rank][0]);
          const uint32_t bar = smem_u32(&stats_bar[ph]);
          if constexpr (C > 1) {
            for (int e = 0; e < 5; ++e) st_cluster_f32(mapa_shared(dst + 4 * e, q), v[e]);
            mbar_arrive_cluster(mapa_shared(bar, q));
          } else {
            for (int e = 0; e < 5; ++e) slot[ph][0][e] = v[e];
            mbar_arrive(&stats_bar[ph]);
          }
        }
      }
      {
        const uint32_t a_bar = smem_u32(&stats_bar[ph]);
        while (!mbar_try_wait_cluster(a_bar, (it >> 1) & 1)) {
        }
      }
      Stat f{slot[ph][0][0], slot[ph][0][1], slot[ph][0][2], slot[ph][0][3], slot[ph][0][4]};
#pragma unroll
      for (int q = 1; q < C; ++q) merge(f, Stat{slot[ph][q][0], slot[ph][q][1], slot[ph][q][2], slot[ph][q][3], slot[ph][q][4]});
      if (rank == 0 && tid == 0) {
        const float lse_t = (f.mt + log2f(f.st)) * LN2;
        const float lse_s = (f.ms + log2f(f.ss)) * LN2;
        loss[row] = f.at / f.st * inv_tau - lse_t + lse_s;
      }
      if (ds == nullptr) continue;
      // ---- pass 2: ds from the stored exponentials, chunk by chunk (each released when done)
      const float g = grad_scale * inv_tau;
      const float gt = g / f.st, gs = g / f.ss;
      __nv_bfloat16* drow = ds + (size_t)row * ldd + c0;
#pragma unroll
      for (int k = 0; k < KDS_NCH; ++k) {
        if (k >= nch) break;
        const int col = k * KDS_CH + 8 * tid;
        if (col < cols) {
          const uint4 ut = reinterpret_cast<const uint4*>(sm + k * (KDS_CH * 4))[tid];
          const uint4 us = reinterpret_cast<const uint4*>(sm + k * (KDS_CH * 4) + KDS_CH * 2)[tid];
          const float fct = gt * ex2a(mh_t[k] - f.mt), fcs = gs * ex2a(mh_s[k] - f.ms);
          const uint32_t* ht = reinterpret_cast<const uint32_t*>(&ut);
          const uint32_t* hs = reinterpret_cast<const uint32_t*>(&us);
          uint32_t o[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 et = __half22float2(*reinterpret_cast<const __half2*>(&ht[j]));
            const float2 es = __half22float2(*reinterpret_cast<const __half2*>(&hs[j]));
            const float2 d = __ffma2_rn(es, make_float2(fcs, fcs), __fmul2_rn(et, make_float2(-fct, -fct)));
            o[j] = pack_bf16(d.x, d.y);
          }
          *reinterpret_cast<uint4*>(drow + col) = make_uint4(o[0], o[1], o[2], o[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[k]);
      }
    }
  }
  __syncwarp();
  if constexpr (C > 1) cluster_sync();  // no CTA exits while peers may still write its slots
}

// Next-token cross entropy over the full vocabulary with ignore index (label < 0):
// loss[row] = lse(s) - s[label];  ds = grad_scale * (softmax(s) - onehot(label)).  Same
// single-pass online max/sum-exp + L2-resident second pass as the streaming KL kernel: four
// vectors in flight per thread, the max over the raw logits scaled once, MUFU exp2.
template <int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS, 4) ce_loss_kernel(const __nv_bfloat16* sl, const int32_t* __restrict__ labels,
                                                             __nv_bfloat16* ds, float* __restrict__ loss, int T, int V,
                                                             int lds, int ldd, float grad_scale) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  __shared__ float red_m[THREADS / 32], red_s[THREADS / 32];
  __shared__ float fin_m, fin_s;
  const int nvec = V / 8;
  auto combine = [](float& m, float& ss, float om, float os) {
    const float mx = fmaxf(m, om);
    ss = (m == -INFINITY ? 0.f : ss * ex2a(m - mx)) + (om == -INFINITY ? 0.f : os * ex2a(om - mx));
    m = mx;
  };
  for (int row = blockIdx.x; row < T; row += gridDim.x) {
    const int lab = labels[row];
    const uint4* s4 = reinterpret_cast<const uint4*>(sl + (size_t)row * lds);
    uint4* d4 = reinterpret_cast<uint4*>(ds + (size_t)row * ldd);
    if (lab < 0) {  // ignored position: zero loss and gradient
      for (int v = threadIdx.x; v < nvec; v += THREADS) d4[v] = make_uint4(0, 0, 0, 0);
      if (threadIdx.x == 0) loss[row] = 0.f;
      continue;
    }
    float m = -INFINITY, ss = 0.f;
    for (int v0 = threadIdx.x; v0 < nvec; v0 += UNROLL * THREADS) {
      uint4 rv[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (v0 + u * THREADS < nvec) rv[u] = s4[v0 + u * THREADS];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (v0 + u * THREADS >= nvec) break;
        float f[8];
        unpack8(rv[u], f);
        float r = f[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) r = fmaxf(r, f[j]);
        const float mx = fmaxf(m, r * LOG2E);
        if (mx > m) {
          ss *= m == -INFINITY ? 0.f : ex2a(m - mx);
          m = mx;
        }
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const float2 x = __ffma2_rn(make_float2(f[j], f[j + 1]), make_float2(LOG2E, LOG2E), make_float2(-m, -m));
          acc = __fadd2_rn(acc, make_float2(ex2a(x.x), ex2a(x.y)));
        }
        ss += acc.x + acc.y;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) combine(m, ss, __shfl_xor_sync(kFull, m, o), __shfl_xor_sync(kFull, ss, o));
    if ((threadIdx.x & 31) == 0) {
      red_m[threadIdx.x >> 5] = m;
      red_s[threadIdx.x >> 5] = ss;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      m = threadIdx.x < THREADS / 32 ? red_m[threadIdx.x] : -INFINITY;
      ss = threadIdx.x < THREADS / 32 ? red_s[threadIdx.x] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) combine(m, ss, __shfl_xor_sync(kFull, m, o), __shfl_xor_sync(kFull, ss, o));
      if (threadIdx.x == 0) {
        fin_m = m;
        fin_s = ss;
        const float lse = (m + log2f(ss)) * LN2;
        loss[row] = lse - __bfloat162float(sl[(size_t)row * lds + lab]);
      }
    }
    __syncthreads();
    const float fm = fin_m, g = grad_scale / fin_s;
    for (int v = threadIdx.x; v < nvec; v += THREADS) {
      float f[8];
      unpack8(s4[v], f);
      uint4 o;
      uint32_t* oh = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 x = __ffma2_rn(make_float2(f[2 * j], f[2 * j + 1]), make_float2(LOG2E, LOG2E), make_float2(-fm, -fm));
        float g0 = ex2a(x.x) * g, g1 = ex2a(x.y) * g;
        if (8 * v + 2 * j == lab) g0 -= grad_scale;
        if (8 * v + 2 * j + 1 == lab) g1 -= grad_scale;
        oh[j] = sm100::pack_bf16(g0, g1);
      }
      d4[v] = o;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace mb

using namespace mb;

// Clusters of `cs` CTAs that can be resident at once (a grid larger than this runs a second wave
// of whole clusters: GPCs do not all hold a multiple of the cluster size).
template <class K>
static int max_clusters(K kernel, int cs, int threads, int smem) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cs;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.gridDim = dim3(cs * 64, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)kernel, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = num_sms() * KDS_CTAS_PER_SM / cs;
  }
  return n;
}

// loss[T] (fp32, per token) and, if d_ds != null, ds = grad_scale * d loss / d s (bf16).
// ds may alias the student logits (in-place): every element is read before it is written
// by the same thread.
MAESTRO_API int maestro_kd_loss_fwd_bwd(const void* d_t, const void* d_s, void* d_ds, float* d_loss, int32_t T,
                                        int32_t V, int32_t ldt, int32_t lds, int32_t ldd, float grad_scale,
                                        float inv_tau, void* stream) {
  if (T <= 0) return 0;
  if (V % 8 || ldt % 8 || lds % 8 || ldd % 8) return (int)cudaErrorInvalidValue;
  // 256-thread blocks, 4 resident per SM (<= 64 registers), four 16-byte vector pairs in flight per
  // thread: rows in different phases (streaming pass / L2 re-read pass) overlap on each SM.
  // Measured at 16384 x 32000 (scripts/kd_bench.py): 512 x 1 block/SM 1.12 ms, 256 x 4 x 2 vectors
  // 0.84 ms, this (4 vectors in flight per thread) 0.82 ms.
#ifndef KD_TH
#define KD_TH 256
#define KD_MB 4
#define KD_UN 4
#endif
  constexpr int TH = KD_TH, MB = KD_MB, UN = KD_UN;
  // Experiment knob (MAESTRO_KD_ROWS_PER_SM=1): one row per SM at a time, 512 threads x 8 vector
  // pairs in flight, so the rows touched by the first pass stay L2-resident for the second at
  // V = 128256.  Measured slower (2840 vs 3612 GB/s at 8192 x 128256, 2936 vs 3870 at
  // 16384 x 32000): the kernel is bound by its exponentials (2 per element per pass) as much as
  // by HBM, and 4 rows per SM overlap them better.  Default: 4 rows per SM.
  // default: the shared-memory-resident kernel (one HBM read per row, 2 exponentials per column)
  static const int impl_env = [] {
    const char* e = getenv("MAESTRO_KD_IMPL");  // "stream": the L2 re-read kernel below; "smem": any C <= 8
    if (!e) return 0;
    return e[0] == 's' && e[1] == 't' ? 1 : (e[0] == 's' && e[1] == 'm' ? 2 : 0);
  }();
  const int C = (V + KDS_VC_MAX - 1) / KDS_VC_MAX;
  const bool aligned = (((uintptr_t)d_t | (uintptr_t)d_s | (uintptr_t)d_ds) & 15) == 0;
  // Cluster row slices pay a per-row stats exchange and cluster co-scheduling: measured (16384 x
  // 32000, C = 2) 3914 GB/s vs 3860 for the streaming kernel, but (8192 x 128256, C = 8) 2766 vs
  // 3609 -- so rows wider than two slices stay on the streaming kernel (MAESTRO_KD_IMPL=smem forces).
  const int c_max = (impl_env == 0) ? 2 : (impl_env == 2 ? 8 : 0);
  if (C <= c_max && aligned) {
    const int VC = ((V + C - 1) / C + 7) / 8 * 8;
    switch (C) {
#define KDS_LAUNCH(CC)                                                                                          \
  case CC: {                                                                                                    \
    if (ensure_smem<kd_loss_smem_kernel<CC>>(KDS_SMEM)) return launch_status();                                \
    static const int max_cl = max_clusters(kd_loss_smem_kernel<CC>, CC, KDS_THREADS, KDS_SMEM);                \
    const int n_cl = T < max_cl ? T : max_cl;                                                                   \
    launch_pdl(kd_loss_smem_kernel<CC>, dim3(n_cl * CC), dim3(KDS_THREADS), KDS_SMEM, (cudaStream_t)stream,                         \
        (const __nv_bfloat16*)d_t, (const __nv_bfloat16*)d_s, (__nv_bfloat16*)d_ds, d_loss, T, V, VC, ldt, lds, \
        ldd, inv_tau * LOG2E, grad_scale, inv_tau);                                                             \
    return launch_status();                                                                                     \
  }
      KDS_LAUNCH(1)
      KDS_LAUNCH(2)
      KDS_LAUNCH(3)
      KDS_LAUNCH(4)
      KDS_LAUNCH(5)
      KDS_LAUNCH(6)
      KDS_LAUNCH(7)
      KDS_LAUNCH(8)
#undef KDS_LAUNCH
    }
  }
  static const int rows_env = [] {
    const char* e = getenv("MAESTRO_KD_ROWS_PER_SM");
    return e ? atoi(e) : 0;
  }();
  const bool big = rows_env == 1;
  if (big) {
    const int grid = T < num_sms() ? T : num_sms();
    launch_pdl(kd_loss_kernel<512, 1, 8>, dim3(grid), dim3(512), 0, (cudaStream_t)stream, 
        (const __nv_bfloat16*)d_t, (const __nv_bfloat16*)d_s, (__nv_bfloat16*)d_ds, d_loss, T, V, ldt, lds, ldd,
        inv_tau * LOG2E, grad_scale, inv_tau);
    return launch_status();
  }
  const int grid = T < 148 * MB * 4 ? T : 148 * MB * 4;
  launch_pdl(kd_loss_kernel<TH, MB, UN>, dim3(grid), dim3(TH), 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)d_t, (const __nv_bfloat16*)d_s, (__nv_bfloat16*)d_ds, d_loss, T, V, ldt, lds, ldd,
      inv_tau * LOG2E, grad_scale, inv_tau);
  return launch_status();
}

// Cross entropy with ignore index (label < 0): loss[T], ds = grad_scale * dCE/ds (bf16, may alias s).
MAESTRO_API int maestro_ce_loss_fwd_bwd(const void* d_s, const int32_t* d_labels, void* d_ds, float* d_loss,
                                        int32_t T, int32_t V, int32_t lds, int32_t ldd, float grad_scale,
                                        void* stream) {
  if (T <= 0) return 0;
  if (V % 8 || lds % 8 || ldd % 8) return (int)cudaErrorInvalidValue;
  const int grid = T < num_sms() * 4 * 4 ? T : num_sms() * 4 * 4;
  launch_pdl(ce_loss_kernel<256, 4>, dim3(grid), dim3(256), 0, (cudaStream_t)stream, (const __nv_bfloat16*)d_s, d_labels,
                                                                 (__nv_bfloat16*)d_ds, d_loss, T, V, lds, ldd,
                                                                 grad_scale);
  return launch_status();
}
