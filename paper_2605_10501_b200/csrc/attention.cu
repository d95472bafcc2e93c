// K8: varlen (cu_seqlens) attention with GQA on tcgen05/TMEM, head_dim 64 or 128, causal or not.
//
// Both directions are persistent: one CTA per SM loops over heavy-first work items dealt in
// snake order; items come from a per-micro-batch plan (query-tile / KV-tile lists) built once by
// maestro_attn_plan and shared by every layer.
//
// Forward item = (128 queries, head), warp-specialised (320 threads):
//   w0     TMA producer: Q (double-buffered by item), K/V tiles through a 3-stage ring
//   w1     MMA issuer:   S_i = Q K_i^T into one of two TMEM score buffers (M=128, N=128, K=64);
//                        O += P_{i-1} V_{i-1} issued after S_i, keys 0-63 into O_a and 64-127
//                        into O_b (V as an MN-major operand), O double-buffered by item
//   w2..w9 softmax:      two warps per TMEM lane quadrant, each owning 64 key columns of a row
//                        with its own online softmax (max, sum, lazy rescale of its O half when
//                        the max grows by > 2^8); P written as a swizzled bf16 smem operand.
//                        The item epilogue (combine the halves, normalise, store O and LSE) runs
//                        after the next item's first tile, when the last PV has long completed.
// TMEM: S0 [0,128) S1 [128,256), O(item parity 0) [256,384), O(parity 1) [384,512).
//
// Backward item = (128 keys, KV head) over its GQA heads and visible query tiles: softmax work in
// two phases (P^T from S^T, then dS^T from dP^T) that overlap the MMAs of the neighbouring
// phases; dV/dK accumulate in TMEM across the item; dQ tiles are drained by a dedicated
// warpgroup through swizzled smem boxes and TMA reduce-add; inverse RoPE fused into the dQ/dK stores.
#include <cuda_bf16.h>
#include <stdlib.h>
#include <climits>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace mb {
namespace {

using namespace sm100;

constexpr int BQ = 128, BKV = 128;  // forward query tile, key tile (rows)
constexpr float LOG2E_F = 1.4426950408889634f;
constexpr float LN2_F = 0.6931471805599453f;

// Query-tile list (tiles of QT rows), heaviest (largest causal row count) first: tiles[i] = (seq, q0)
template <int QT = BQ>
__global__ void attn_tiles_kernel(const int32_t* __restrict__ cu, int nseq, int2* __restrict__ tiles,
                                  int* __restrict__ count) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  __shared__ int s_max, s_n;
  if (threadIdx.x == 0) {
    s_max = 0;
    s_n = 0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nseq; j += blockDim.x) atomicMax(&s_max, (cu[j + 1] - cu[j] + QT - 1) / QT);
  __syncthreads();
  for (int qb = s_max - 1; qb >= 0; --qb) {
    for (int j0 = 0; j0 < nseq; j0 += blockDim.x) {
      const int j = j0 + threadIdx.x;
      const bool has = j < nseq && (cu[j + 1] - cu[j] + QT - 1) / QT > qb;
      const unsigned bal = __ballot_sync(kFull, has);
      // warp-aggregated append (order inside a qb level is irrelevant)
      int base = 0;
      if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(&s_n, __popc(bal));
      base = __shfl_sync(kFull, base, 0);
      if (has) tiles[base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = make_int2(j, qb * QT);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = s_n;
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// One arrive per warp (barrier count = warps) instead of one per thread: each lane's tcgen05
// ld/st wait + fence::before_thread_sync precede the __syncwarp, so lane 0's release covers the
// whole warp -- 8 shared-memory arrives per tile-barrier instead of 256.
#ifndef ATTN_WARP_ARRIVE
#define ATTN_WARP_ARRIVE 0  // 1: one arrive per warp (measured: no consistent gain, r02_attn_arrive_ab.jsonl)
#endif
constexpr int ARRIVE_UNIT = ATTN_WARP_ARRIVE ? 32 : 1;  // threads per arrive
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  if (ATTN_WARP_ARRIVE) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
  } else {
    mbar_arrive(bar);
  }
}

// Barrier addresses as 32-bit shared-window offsets from one base computed once per kernel (kept
// in a uniform register), instead of a generic->shared conversion (S2R SR_CgaCtaId + LEA, which
// ptxas rematerialises under register pressure) at every wait/arrive of the softmax loop.
#ifndef ATTN_BAR_U32
#define ATTN_BAR_U32 0  // measured: +1.6-2 % at the KD shapes, -3-4 % at cfg 5 (r02_attn_bar_ab.jsonl)
#endif
struct Bars {
  uint64_t* base;
  uint32_t base_u;
  __device__ __forceinline__ uint32_t at(const uint64_t* p) const { return base_u + (uint32_t)(p - base) * 8u; }
};
__device__ __forceinline__ void bwait(const Bars& B, uint64_t* p, uint32_t parity) {
  if (ATTN_BAR_U32) {
    const uint32_t a = B.at(p);
    while (!mbar_try_wait(a, parity)) {
    }
  } else {
    mbar_wait(p, parity);
  }
}
__device__ __forceinline__ void barrive(const Bars& B, uint64_t* p) {
  if (ATTN_BAR_U32)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(B.at(p)) : "memory");
  else
    mbar_arrive(p);
}
__device__ __forceinline__ void warp_arrive(const Bars& B, uint64_t* p) {
  if (ATTN_WARP_ARRIVE) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) barrive(B, p);
  } else {
    barrive(B, p);
  }
}

#ifndef BWD_EMU_BITS
#define BWD_EMU_BITS 0x00  // backward P^T = exp2(S^T scale2 - lse2): not MUFU-bound, all on MUFU
#endif
#ifndef ATTN_SETMAXNREG
#define ATTN_SETMAXNREG 0
#endif
#ifndef ATTN_FWD_CG64
#define ATTN_FWD_CG64 2  // default column groups of the head_dim-64 forward (see FwdCfg)
#endif
#ifndef ATTN_FWD_VARIANT
#define ATTN_FWD_VARIANT -1  // forward: -1 by shape, 0 shared tile, 1 decoupled groups, 2 ping-pong (MAESTRO_ATTN_FWD=base|dec|pp)
#endif
#ifndef FWD_EMU_BITS
#define FWD_EMU_BITS 0x92  // pair p of a row's 32 goes to the FMA pipe if bit (p & 7) is set (3/8)
#endif
// SWIZZLE_128B smem descriptor from a 16-byte-unit address (addr >> 4; the CTA window is below
// 256 KB so it fits the 14-bit field unmasked): callers shift a stage base once and add per-K-step
// constants, so issuing an MMA costs one add per operand instead of a shift/mask/or chain.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr16, uint32_t lbo, uint32_t sbo) {
  return ((uint64_t)((sbo >> 4) | (1u << 14) | (2u << 29)) << 32) | (uint64_t)(addr16 + ((lbo >> 4) << 16));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t p_offset(int r, int c) {
  // (row r, col c) of a 128 x 128 bf16 operand stored as two K-major SWIZZLE_128B chunks
  const int chunk = c >> 6, cc = c & 63;
  return (uint32_t)(chunk * 16384 + r * 128 + ((((cc >> 3) ^ (r & 7)) << 4)) + ((cc & 7) << 1));
}

#ifndef ATTN_FWD_PRODUCER_SLEEP
#define ATTN_FWD_PRODUCER_SLEEP 0
#endif
// TMA / MMA warps of the forward kernels: sleep on the barrier (suspend hint) or poll
__device__ __forceinline__ void prod_wait(uint64_t* bar, uint32_t parity) {
  if constexpr (ATTN_FWD_PRODUCER_SLEEP) mbar_wait_sleep<20000>(bar, parity);
  else mbar_wait(bar, parity);
}

// Persistent forward: one CTA per SM loops over work items (query tile, head) in heavy-first
// order.  All pipeline counters run across items: K/V stream through the ring, S alternates
// between two TMEM buffers by global tile index, Q is double-buffered by item index, so the
// next item's Q load, first S MMAs and softmax overlap the current item's epilogue.
//
// The 128 key columns of a tile are split into CG column groups; each lane quadrant has one
// softmax warp per group, each group runs its own online softmax (max, sum, lazy rescale) into
// its own O accumulator (keys of its columns), and the groups combine once per item in the
// epilogue.  CG = 2: 8 softmax warps, 64 columns per thread.  CG = 4 (head_dim 64 only): 16
// softmax warps, 32 columns per thread -- twice the warps per SM sub-partition to hide the
// per-tile latency chain (TMEM load -> max -> exp -> sum -> pack -> TMEM store), at half the
// registers per thread.
// TMEM: S0 [0,128) S1 [128,256), then NOB x CG O accumulators of DH columns:
//   DH 64, CG 2: O double-buffered by item ([256,384), [384,512));
//   DH 64, CG 4 and DH 128, CG 2: one set of O accumulators ([256,512)), so the first PV of an
//   item waits for the previous item's (deferred) epilogue to have read them.
// A [128 rows][DH] bf16 tile is DH/64 SWIZZLE_128B chunks of 128 rows x 128 B (16 KB each).
template <int DH, int CG>
struct FwdCfg {
  // w0 TMA, w1 MMA, softmax warps from SW0 on (CG per lane quadrant).  CG = 4: warps 2-3 idle so
  // the softmax warps fill whole warpgroups and setmaxnreg can move registers to them
  static constexpr int SW0 = (CG == 4 && ATTN_SETMAXNREG) ? 4 : 2;
  static constexpr int THREADS = 32 * SW0 + 128 * CG;
  static constexpr int REG_LO = 88, REG_HI = 104;     // CG = 4: TMA/MMA warpgroup, softmax warpgroups
  static constexpr int SMX = 128 * CG;                // softmax threads
  static constexpr int CW = BKV / CG;                 // key columns per group
  static constexpr int TILE = 128 * DH * 2;           // bytes of a 128-row tile
  static constexpr int KVS = DH == 64 ? 3 : 2;        // K/V ring depth
  static constexpr int NOB = (256 + 2 * CG * DH <= 512) ? 2 : 1;  // O accumulator sets (by item)
  static constexpr int Q = 0;                         // 2 x TILE (by item parity)
  static constexpr int K = Q + 2 * TILE;
  static constexpr int V = K + KVS * TILE;
  static constexpr int XMAX = V + KVS * TILE;         // [2 items][CG groups][128] row maxima
  static constexpr int XSUM = XMAX + 2 * CG * 128 * 4; // [2 items][CG groups][128] row sums
  static constexpr int BAR = XSUM + 2 * CG * 128 * 4;
  static constexpr int TOTAL = BAR + 256;
  static_assert(TOTAL + 1024 <= 227 * 1024, "forward smem");
  static_assert(256 + NOB * CG * DH <= 512, "forward TMEM");
  static_assert(CW == 32 || CW == 64, "column group width");
};

struct FwdItem {
  int seq, q0, h, hk, s0, L, n_kv;
};

template <bool CAUSAL>
__device__ __forceinline__ FwdItem fwd_item(int w, int H, int Hk, const int32_t* cu, const int2* tiles) {
  FwdItem it;
  const int2 tq = tiles[w / H];
  it.seq = tq.x;
  it.q0 = tq.y;
  it.h = w % H;
  it.hk = it.h / (H / Hk);
  it.s0 = cu[it.seq];
  it.L = cu[it.seq + 1] - it.s0;
  const int n_all = (it.L + BKV - 1) / BKV;
  it.n_kv = CAUSAL ? min(n_all, it.q0 / BKV + 1) : n_all;
  return it;
}

// Item of round r for this CTA; rounds alternate direction so the heavy-first item list is
// dealt like LPT (the CTA that got the heaviest item of one round gets the lightest of the next).
__device__ __forceinline__ int snake_item(int r) {
  return r * (int)gridDim.x + ((r & 1) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x);
}

// TMA load of one 128-row tile: DH/64 boxes of 64 columns, one per SWIZZLE_128B chunk.
template <int DH>
__device__ __forceinline__ void load_tile(unsigned char* dst, const CUtensorMap* map, uint64_t* bar, int col, int row) {
#pragma unroll
  for (int c = 0; c < DH / 64; ++c) tma_load_2d(dst + c * 16384, map, bar, col + 64 * c, row);
}

template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 32) {
    tmem_ld_32x32b_x32(taddr, r);
  } else {
    static_assert(N == 16, "tmem_ld_cols");
    tmem_ld_32x32b_x16(taddr, r);
  }
}
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t (&r)[N]) {
  if constexpr (N == 32) {
    tmem_st_32x32b_x32(taddr, r);
  } else {
    static_assert(N == 16, "tmem_st_cols");
    tmem_st_32x32b_x16(taddr, r);
  }
}

template <int DH, int CG, bool CAUSAL>
__global__ void __launch_bounds__(FwdCfg<DH, CG>::THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ cu,
                    const int2* __restrict__ tiles, const int* __restrict__ n_tiles, __nv_bfloat16* __restrict__ out,
                    int ldo, float* __restrict__ lse, int T, int H, int Hk, float scale2, int stagger_ns) {
  using C = FwdCfg<DH, CG>;
  constexpr int KVS = C::KVS, NOB = C::NOB, TB = C::TILE, CW = C::CW, SMX = C::SMX;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR);
  uint64_t* q_full = bar;                  // [2]
  uint64_t* q_empty = bar + 2;             // [2]
  uint64_t* k_full = bar + 4;              // [KVS]
  uint64_t* k_empty = k_full + KVS;
  uint64_t* v_full = k_empty + KVS;
  uint64_t* v_empty = v_full + KVS;
  uint64_t* s_full = v_empty + KVS;        // [2]
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 2;
  uint64_t* o_full = p_empty + 2;          // [NOB]
  uint64_t* o_empty = o_full + 2;          // [NOB]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);
  const Bars BR{bar, smem_u32(bar)};

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], SMX / ARRIVE_UNIT);
      mbar_init(&p_full[b], SMX / ARRIVE_UNIT);
      mbar_init(&p_empty[b], 1);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], SMX / ARRIVE_UNIT);
    }
    for (int s = 0; s < KVS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above (barriers, TMEM, tensor-map prefetch)
  // overlapped the previous kernel; global memory (the tile list included) only from here
  pdl_trigger();
  pdl_wait();
  const int n_items = *n_tiles * H;
  if constexpr (CG == 4 && ATTN_SETMAXNREG) {  // registers from the TMA/MMA warpgroup to the 16 softmax warps
    if (warp < 4)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::REG_LO));
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::REG_HI));
  }

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;  // global KV tile counter (ring position)
      int j = 0;  // local item counter
      FwdItem it_n{};
      if (snake_item(0) < n_items) it_n = fwd_item<CAUSAL>(snake_item(0), H, Hk, cu, tiles);
      for (int w = snake_item(0); w < n_items; w = snake_item(j + 1), ++j) {
        const FwdItem it = it_n;
        if (snake_item(j + 1) < n_items) it_n = fwd_item<CAUSAL>(snake_item(j + 1), H, Hk, cu, tiles);  // prefetch
        const int qb = j & 1;
        bwait(BR, &q_empty[qb], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], TB);
        load_tile<DH>(sm + C::Q + qb * TB, &map_q, &q_full[qb], it.h * DH, it.s0 + it.q0);
        for (int i = 0; i < it.n_kv; ++i, ++g) {
          const int st = g % KVS;
          const uint32_t ph = (g / KVS) & 1;
          bwait(BR, &k_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&k_full[st], TB);
          load_tile<DH>(sm + C::K + st * TB, &map_k, &k_full[st], it.hk * DH, it.s0 + i * BKV);
          bwait(BR, &v_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&v_full[st], TB);
          load_tile<DH>(sm + C::V + st * TB, &map_v, &v_full[st], it.hk * DH, it.s0 + i * BKV);
        }
      }
    }
  } else if (warp == 1) {
    {
      constexpr uint32_t idesc_s = idesc_bf16_f32(BQ, BKV, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(BQ, DH, false, true);
      // PV of global tile gp (item-local index ip, item counter jp) into O set ob
      auto issue_pv = [&](int gp, int ip, int jp, int ob) {
        const int pb = gp & 1;
        if (ip == 0) bwait(BR, &o_empty[ob], ((jp / NOB) & 1) ^ 1);  // epilogue of the item that last used O set ob
        bwait(BR, &p_full[pb], (gp >> 1) & 1);
        bwait(BR, &v_full[gp % KVS], (gp / KVS) & 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(sm + C::V + (gp % KVS) * TB);
        // keys of column group c accumulate into O_c: each group keeps its own running max, so
        // the groups never synchronise inside the KV loop.  A = P from TMEM: group c's bf16
        // pairs sit in the first CW/2 of its CW score columns of S buffer pb.  B = V as an
        // MN-major operand: DH/64 swizzle atoms 16 KB apart (LBO), 8-key groups 1 KB (SBO).
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const int c = kk / (CW / 16), kc = kk % (CW / 16);
            umma_bf16_ts(tmem + 256 + (ob * CG + c) * DH, tmem + pb * BKV + c * CW + kc * 8,
                         sdesc((v_base >> 4) + kk * 128, DH == 64 ? 8192 : 16384, 1024), idesc_o,
                         (ip > 0 || kc > 0) ? 1u : 0u);
          }
          umma_commit(&v_empty[gp % KVS]);
          umma_commit(&p_empty[pb]);
        }
        __syncwarp();
      };
      int g = 0, j = 0;
      // the PV of each tile is issued after the NEXT tile's S (also across item boundaries), so
      // the tensor core computes S while the softmax warps work on the previous tile
      int pend_g = -1, pend_i = 0, pend_j = 0, pend_o = 0;
      bool pend_last = false;
      auto flush = [&]() {
        if (pend_g < 0) return;
        issue_pv(pend_g, pend_i, pend_j, pend_o);
        if (pend_last) {
          if (elect_one()) umma_commit(&o_full[pend_o]);
          __syncwarp();
        }
        pend_g = -1;
      };
      FwdItem it_n{};
      if (snake_item(0) < n_items) it_n = fwd_item<CAUSAL>(snake_item(0), H, Hk, cu, tiles);
      for (int w = snake_item(0); w < n_items; w = snake_item(j + 1), ++j) {
        const FwdItem it = it_n;
        if (snake_item(j + 1) < n_items) it_n = fwd_item<CAUSAL>(snake_item(j + 1), H, Hk, cu, tiles);  // prefetch
        const int qb = j & 1, ob = j % NOB;
        bwait(BR, &q_full[qb], (j >> 1) & 1);
        const uint32_t q_base = smem_u32(sm + C::Q + qb * TB);
        for (int i = 0; i < it.n_kv; ++i, ++g) {
          const int b = g & 1;
          const int st = g % KVS;
          bwait(BR, &k_full[st], (g / KVS) & 1);
          bwait(BR, &s_empty[b], ((g >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(sm + C::K + st * TB);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)  // chunk kk/4 (16 KB apart), 32 B per K step inside it
              umma_bf16(tmem + b * BKV, sdesc((q_base >> 4) + (kk >> 2) * 1024 + (kk & 3) * 2, 16, 1024),
                        sdesc((k_base >> 4) + (kk >> 2) * 1024 + (kk & 3) * 2, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
            umma_commit(&k_empty[st]);
            umma_commit(&s_full[b]);
            if (i == it.n_kv - 1) umma_commit(&q_empty[qb]);  // last S of the item: Q buffer free
          }
          __syncwarp();
          flush();
          pend_g = g;
          pend_i = i;
          pend_j = j;
          pend_o = ob;
          pend_last = i == it.n_kv - 1;
        }
      }
      flush();
    }
  } else if (warp >= C::SW0) {
    // Softmax: warp (SW0 + 4 grp + q) owns TMEM lane quadrant q (rows 32q..32q+31) and key columns
    // [grp*CW, grp*CW + CW) of every tile.  The groups combine once per item in the epilogue
    // (named barrier per quadrant), each normalising and storing DH/CG of the DH output columns.
    const int q = warp & 3;
    const int grp = (warp - C::SW0) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int quad_bar = 2 + q;
    float* xmax = reinterpret_cast<float*>(sm + C::XMAX);
    float* xsum = reinterpret_cast<float*>(sm + C::XSUM);
    // Epilogue of item jj (final m / l), deferred until after the next item's first tile: by
    // then the item's last PV has completed, so O is read without waiting on it.
    auto epilogue = [&](const FwdItem& it, int jj, float m, float l) {
      const int ob = jj % NOB;
      const int qpos = it.q0 + r;
      float* xm = xmax + (jj & 1) * CG * 128;  // by item parity: the groups read it before the next item's barrier
      float* xs = xsum + (jj & 1) * CG * 128;
      xm[grp * 128 + r] = m;
      xs[grp * 128 + r] = l;
      bwait(BR, &o_full[ob], (jj / NOB) & 1);
      tc_fence_after();
      named_bar(quad_bar, 32 * CG);
      float mg[CG], lg[CG];
      float M = -INFINITY;
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        mg[c] = xm[c * 128 + r];
        lg[c] = xs[c * 128 + r];
        M = fmaxf(M, mg[c]);
      }
      float l_all = 0.f, fct[CG];
#pragma unroll
      for (int c = 0; c < CG; ++c) {
        fct[c] = mg[c] == -INFINITY ? 0.f : ex2(mg[c] - M);
        l_all += lg[c] * fct[c];
      }
      const float rl = __frcp_rn(l_all);
#pragma unroll
      for (int c = 0; c < CG; ++c) fct[c] *= rl;
      // this group's DH/CG output columns, in chunks of 16 or 32
      constexpr int OC = DH / CG;                      // 32 (DH 64, CG 2 / DH 128 ... ) or 16 (DH 64, CG 4)
      constexpr int CH = OC >= 32 ? 32 : OC;           // columns per TMEM load
#pragma unroll
      for (int sub = 0; sub < OC / CH; ++sub) {
        const int c0 = grp * OC + sub * CH;
        float acc[CH];
#pragma unroll
        for (int e = 0; e < CH; ++e) acc[e] = 0.f;
#pragma unroll
        for (int c = 0; c < CG; ++c) {
          uint32_t ra[CH];
          tmem_ld_cols<CH>(tmem + lane_base + 256 + (ob * CG + c) * DH + c0, ra);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < CH; ++e) acc[e] = fmaf(__uint_as_float(ra[e]), fct[c], acc[e]);
        }
        if (sub == OC / CH - 1) {
          tc_fence_before();
          warp_arrive(BR, &o_empty[ob]);
        }
        if (qpos < it.L) {
          uint32_t o[CH / 2];
#pragma unroll
          for (int e = 0; e < CH / 2; ++e) o[e] = pack_bf16(acc[2 * e], acc[2 * e + 1]);
          uint4* dst = reinterpret_cast<uint4*>(out + (size_t)(it.s0 + qpos) * ldo + it.h * DH + c0);
#pragma unroll
          for (int u = 0; u < CH / 8; ++u) dst[u] = make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
        }
      }
      if (grp == 0 && qpos < it.L) lse[(size_t)it.h * T + it.s0 + qpos] = (M + log2f(l_all)) * LN2_F;
    };
    // experiment knob (MAESTRO_ATTN_STAGGER_NS): start the second column group late so the two
    // softmax warps of an SM sub-partition run their phases (max / exp / pack) out of step
    if (grp == 1 && stagger_ns > 0) __nanosleep(stagger_ns);
    int g = 0, j = 0;
    bool pend = false;
    FwdItem pit{};
    int pj = 0;
    float pm = 0.f, pl = 0.f;
    int w = snake_item(0);
    FwdItem it{};
    if (w < n_items) it = fwd_item<CAUSAL>(w, H, Hk, cu, tiles);
    for (; w < n_items; ++j) {
      const int w_next = snake_item(j + 1);
      FwdItem nxt{};
      if (w_next < n_items) nxt = fwd_item<CAUSAL>(w_next, H, Hk, cu, tiles);  // prefetch the next item
      const int ob = j % NOB;
      const int qpos = it.q0 + r;
      float m = -INFINITY, l = 0.f;
      for (int i = 0; i < it.n_kv; ++i, ++g) {
        const int b = g & 1;
        bwait(BR, &s_full[b], (g >> 1) & 1);
        tc_fence_after();
        float s[CW];
        {
          uint32_t raw[CW / 32][32];
#pragma unroll
          for (int c = 0; c < CW / 32; ++c) tmem_ld_32x32b_x32(tmem + lane_base + b * BKV + grp * CW + 32 * c, raw[c]);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < CW / 32; ++c)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) s[c * 32 + jj] = __uint_as_float(raw[c][jj]);
        }
        tc_fence_before();
        warp_arrive(BR, &s_empty[b]);
        const int kv0 = i * BKV + grp * CW;
        const bool need_mask = (CAUSAL && kv0 + CW - 1 > it.q0) || (kv0 + CW > it.L);
        // valid key columns of this row: c < lim (causal: key <= query; key inside the sequence)
        const int lim = CAUSAL ? min(qpos - kv0 + 1, it.L - kv0) : it.L - kv0;
        if (need_mask && __all_sync(kFull, lim <= 0)) {
          // every row of this warp sees only masked keys in this group's columns (upper triangle
          // of the diagonal tile): P = 0, running max and sum unchanged
          uint32_t zero[CW / 2];
#pragma unroll
          for (int e = 0; e < CW / 2; ++e) zero[e] = 0u;
          tmem_st_cols<CW / 2>(tmem + lane_base + b * BKV + grp * CW, zero);
          tmem_st_wait();
          tc_fence_before();
          warp_arrive(BR, &p_full[b]);
          if (i == 0 && pend) {
            epilogue(pit, pj, pm, pl);
            pend = false;
          }
          continue;
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (need_mask) {
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            s[c] = c < lim ? s[c] : -INFINITY;
            mx4[c & 3] = fmaxf(mx4[c & 3], s[c]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < CW; ++c) mx4[c & 3] = fmaxf(mx4[c & 3], s[c]);
        }
        const float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * scale2;
        bool rescale = false;
        float alpha = 1.f;
        if (m_new > m + 8.0f) {
          alpha = ex2(m - m_new);
          m = m_new;
          rescale = i > 0;
        }
        const float neg_m = m == -INFINITY ? 0.f : -m;  // group fully masked so far: P = 0
        // paired fp32 FMA/add (FFMA2/FADD2): half the issue slots of the scalar forms
        const float2 sc2 = make_float2(scale2, scale2), nm2 = make_float2(neg_m, neg_m);
        float2 sum2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
        for (int c = 0; c < CW; c += 2) {
          const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), sc2, nm2);
          if ((FWD_EMU_BITS >> ((c >> 1) & 7)) & 1) {
            const float2 e = ex2_fma2<3>(x);
            s[c] = e.x;
            s[c + 1] = e.y;
          } else {
            s[c] = ex2(x.x);
            s[c + 1] = ex2(x.y);
          }
          sum2[(c >> 1) & 3] = __fadd2_rn(sum2[(c >> 1) & 3], make_float2(s[c], s[c + 1]));
        }
        const float2 t01 = __fadd2_rn(sum2[0], sum2[1]), t23 = __fadd2_rn(sum2[2], sum2[3]);
        const float2 t = __fadd2_rn(t01, t23);
        l = l * alpha + (t.x + t.y);
        // the rescale decision is per row; the TMEM load/store are warp-collective (.sync.aligned),
        // so the whole warp takes the branch when any lane needs it (the others scale by 1, exact)
        if (__any_sync(kFull, rescale)) {
          if (!rescale) alpha = 1.f;
          bwait(BR, &p_empty[(g - 1) & 1], ((g - 1) >> 1) & 1);  // PV_{g-1} retired: O is final
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tmem + lane_base + 256 + (ob * CG + grp) * DH + c * 32, rr);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) rr[jj] = __float_as_uint(__uint_as_float(rr[jj]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_base + 256 + (ob * CG + grp) * DH + c * 32, rr);
          }
          tmem_st_wait();
        }
        // P (bf16 pairs) over the first CW/2 of this group's score columns: S_{g+2} is issued
        // after PV_g, so the buffer is not rewritten before the tensor core has read P
        {
          uint32_t pk[CW / 2];
#pragma unroll
          for (int e = 0; e < CW / 2; ++e) pk[e] = pack_bf16(s[2 * e], s[2 * e + 1]);
          tmem_st_cols<CW / 2>(tmem + lane_base + b * BKV + grp * CW, pk);
        }
        tmem_st_wait();
        tc_fence_before();
        warp_arrive(BR, &p_full[b]);
        if (i == 0 && pend) {
          epilogue(pit, pj, pm, pl);
          pend = false;
        }
      }
      pend = true;
      pit = it;
      pj = j;
      pm = m;
      pl = l;
      it = nxt;
      w = w_next;
    }
    if (pend) epilogue(pit, pj, pm, pl);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------------------------------
// Forward, decoupled column groups.  The two 64-key column groups of a tile get independent
// pipelines: each has its own MMA-issuing warp (S_g = Q K_g^T with N = 64 into its own
// double-buffered score columns, O_g += P_g V_g), its own barriers and its own O accumulator;
// they share only the Q buffers and the K/V ring (stages released after both groups' MMAs).
// With one shared S tile (attn_fwd_kernel) the two softmax warps of an SM sub-partition wait
// on the same barriers and run the same phase (TMEM load -> max -> exponentials -> pack ->
// TMEM store) at the same time, so the exponential unit idles through the other phases.  Here
// group 1 starts `stagger_ns` late and nothing re-synchronises the groups inside an item, so the
// two warps of a sub-partition work on different phases.  The item epilogue is done by whichever
// group's warp of a lane quadrant arrives second (shared-memory counter): it combines both O
// halves and stores O and the LSE; the first arriver moves on to the next item.
// Warps: w0 TMA, w1 / w2 MMA for groups 0 / 1, w3..w10 softmax (group (w - 3) / 4, quadrant w & 3).
// TMEM: S_g buffer b at g * 128 + b * 64; O_g at 256 + (ob * 2 + g) * 64 (head_dim 64, two sets by
// item) or 256 + g * 128 (head_dim 128, one set).
template <int DH, int NG = 2>
struct FwdDecCfg {
  static constexpr int CW = BKV / NG;           // key columns per group
  // w0 TMA, w1..wNG MMA (one per group), then softmax; NG = 4: softmax from warp 8 so the two
  // producer warpgroups can hand registers to the four softmax warpgroups (setmaxnreg)
  static constexpr bool REG_SPLIT = false;  // NG == 4 with setmaxnreg: ptxas still compiles the softmax at 80 registers (spills)
  static constexpr int SW0 = REG_SPLIT ? 8 : 1 + NG;
  static constexpr int REG_PROD = 40, REG_SMX = 104;  // REG_SPLIT: 8 x 32 x 40 + 16 x 32 x 104 <= 64 K
  static constexpr int THREADS = 32 * SW0 + 128 * NG;
  static constexpr int TILE = 128 * DH * 2;
  static constexpr int KVS = DH == 64 ? 3 : 2;
  static constexpr int NOB = (256 + 2 * NG * DH <= 512) ? 2 : 1;  // O sets (by item)
  static constexpr int Q = 0;
  static constexpr int K = Q + 2 * TILE;
  static constexpr int V = K + KVS * TILE;
  // epilogue exchange slots by item % 4: a group can run up to two items ahead of the other (a
  // one-tile item's S is issued before the PV that waits for the item-before-last's epilogue),
  // so three items can have an epilogue in flight
  static constexpr int XS = 4;
  static constexpr int XMAX = V + KVS * TILE;  // [XS items][NG groups][128]
  static constexpr int XSUM = XMAX + XS * NG * 128 * 4;
  static constexpr int CNT = XSUM + XS * NG * 128 * 4;  // [XS items][4 quadrants] arrivals
  static constexpr int BAR = CNT + 64;
  static constexpr int TOTAL = BAR + 1024;
  static_assert(TOTAL + 1024 <= 227 * 1024, "forward smem");
  static_assert(2 * NG * CW + NOB * NG * DH <= 512, "forward TMEM");
  __device__ static constexpr uint32_t s_col(int g, int b) { return g * 2 * CW + b * CW; }
  __device__ static constexpr uint32_t o_col(int ob, int g) { return 256 + (ob * NG + g) * DH; }
};

template <int DH, bool CAUSAL, int NG = 2>
__global__ void __launch_bounds__(FwdDecCfg<DH, NG>::THREADS, 1)
    attn_fwd_dec_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                        const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ cu,
                        const int2* __restrict__ tiles, const int* __restrict__ n_tiles,
                        __nv_bfloat16* __restrict__ out, int ldo, float* __restrict__ lse, int T, int H, int Hk,
                        float scale2, int stagger_ns) {
  using C = FwdDecCfg<DH, NG>;
  constexpr int KVS = C::KVS, NOB = C::NOB, TB = C::TILE, CW = C::CW;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR);
  uint64_t* q_full = bar;          // [2]
  uint64_t* q_empty = bar + 2;     // [2]
  uint64_t* k_full = bar + 4;      // [KVS]
  uint64_t* k_empty = k_full + KVS;
  uint64_t* v_full = k_empty + KVS;
  uint64_t* v_empty = v_full + KVS;
  uint64_t* gb = v_empty + KVS;    // per group: s_full[2] s_empty[2] p_full[2] p_empty[2] o_full[2] o_empty[2]
  auto s_full = [&](int g) { return gb + 12 * g; };
  auto s_empty = [&](int g) { return gb + 12 * g + 2; };
  auto p_full = [&](int g) { return gb + 12 * g + 4; };
  auto p_empty = [&](int g) { return gb + 12 * g + 6; };
  auto o_full = [&](int g) { return gb + 12 * g + 8; };
  auto o_empty = [&](int g) { return gb + 12 * g + 10; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gb + 12 * NG);
  int* cnt = reinterpret_cast<int*>(sm + C::CNT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], NG);
    }
    for (int s = 0; s < KVS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], NG);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], NG);
    }
    for (int g = 0; g < NG; ++g)
      for (int b = 0; b < 2; ++b) {
        mbar_init(&s_full(g)[b], 1);
        mbar_init(&s_empty(g)[b], 128);
        mbar_init(&p_full(g)[b], 128);
        mbar_init(&p_empty(g)[b], 1);
        mbar_init(&o_full(g)[b], 1);
        mbar_init(&o_empty(g)[b], 128);
      }
    for (int k = 0; k < 4 * C::XS; ++k) cnt[k] = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above (barriers, TMEM, tensor-map prefetch)
  // overlapped the previous kernel; global memory (the tile list included) only from here
  pdl_trigger();
  pdl_wait();
  const int n_items = *n_tiles * H;
  if constexpr (C::REG_SPLIT) {
    if (warp < C::SW0)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::REG_PROD));
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::REG_SMX));
  }

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, j = 0;
      FwdItem it_n{};
      if (snake_item(0) < n_items) it_n = fwd_item<CAUSAL>(snake_item(0), H, Hk, cu, tiles);
      for (int w = snake_item(0); w < n_items; w = snake_item(j + 1), ++j) {
        const FwdItem it = it_n;
        if (snake_item(j + 1) < n_items) it_n = fwd_item<CAUSAL>(snake_item(j + 1), H, Hk, cu, tiles);
        const int qb = j & 1;
        prod_wait(&q_empty[qb], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], TB);
        load_tile<DH>(sm + C::Q + qb * TB, &map_q, &q_full[qb], it.h * DH, it.s0 + it.q0);
        for (int i = 0; i < it.n_kv; ++i, ++g) {
          const int st = g % KVS;
          const uint32_t ph = (g / KVS) & 1;
          prod_wait(&k_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&k_full[st], TB);
          load_tile<DH>(sm + C::K + st * TB, &map_k, &k_full[st], it.hk * DH, it.s0 + i * BKV);
          prod_wait(&v_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&v_full[st], TB);
          load_tile<DH>(sm + C::V + st * TB, &map_v, &v_full[st], it.hk * DH, it.s0 + i * BKV);
        }
      }
    }
  } else if (warp <= NG) {
    const int mg = warp - 1;  // column group served by this MMA warp
    if (mg > 0 && stagger_ns > 0) __nanosleep(stagger_ns * mg / (NG - 1));
    constexpr uint32_t idesc_s = idesc_bf16_f32(BQ, CW, false, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BQ, DH, false, true);
    uint64_t *sf = s_full(mg), *se = s_empty(mg), *pf = p_full(mg), *pe = p_empty(mg), *of = o_full(mg),
             *oe = o_empty(mg);
    auto issue_pv = [&](int gp, int ip, int jp, int ob) {
      const int pb = gp & 1;
      if (ip == 0) prod_wait(&oe[ob], ((jp / NOB) & 1) ^ 1);
      prod_wait(&pf[pb], (gp >> 1) & 1);
      prod_wait(&v_full[gp % KVS], (gp / KVS) & 1);
      tc_fence_after();
      const uint32_t v_base = smem_u32(sm + C::V + (gp % KVS) * TB);
      if (elect_one()) {
#pragma unroll
        for (int kc = 0; kc < CW / 16; ++kc)  // keys CW mg + 16 kc (V as an MN-major operand)
          umma_bf16_ts(tmem + C::o_col(ob, mg), tmem + C::s_col(mg, pb) + kc * 8,
                       sdesc((v_base >> 4) + ((CW / 16) * mg + kc) * 128, DH == 64 ? 8192 : 16384, 1024), idesc_o,
                       (ip > 0 || kc > 0) ? 1u : 0u);
        umma_commit(&v_empty[gp % KVS]);
        umma_commit(&pe[pb]);
      }
      __syncwarp();
    };
    int g = 0, j = 0;
    int pend_g = -1, pend_i = 0, pend_j = 0, pend_o = 0;
    bool pend_last = false;
    auto flush = [&]() {
      if (pend_g < 0) return;
      issue_pv(pend_g, pend_i, pend_j, pend_o);
      if (pend_last) {
        if (elect_one()) umma_commit(&of[pend_o]);
        __syncwarp();
      }
      pend_g = -1;
    };
    FwdItem it_n{};
    if (snake_item(0) < n_items) it_n = fwd_item<CAUSAL>(snake_item(0), H, Hk, cu, tiles);
    for (int w = snake_item(0); w < n_items; w = snake_item(j + 1), ++j) {
      const FwdItem it = it_n;
      if (snake_item(j + 1) < n_items) it_n = fwd_item<CAUSAL>(snake_item(j + 1), H, Hk, cu, tiles);
      const int qb = j & 1, ob = j % NOB;
      prod_wait(&q_full[qb], (j >> 1) & 1);
      const uint32_t q_base = smem_u32(sm + C::Q + qb * TB);
      for (int i = 0; i < it.n_kv; ++i, ++g) {
        const int b = g & 1;
        const int st = g % KVS;
        prod_wait(&k_full[st], (g / KVS) & 1);
        prod_wait(&se[b], ((g >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sm + C::K + st * TB);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)  // B = keys CW mg .. CW mg + CW - 1 (CW x 128 B into each chunk)
            umma_bf16(tmem + C::s_col(mg, b), sdesc((q_base >> 4) + (kk >> 2) * 1024 + (kk & 3) * 2, 16, 1024),
                      sdesc((k_base >> 4) + (kk >> 2) * 1024 + (kk & 3) * 2 + 8 * CW * mg, 16, 1024), idesc_s,
                      kk > 0 ? 1u : 0u);
          umma_commit(&k_empty[st]);
          umma_commit(&sf[b]);
          if (i == it.n_kv - 1) umma_commit(&q_empty[qb]);
        }
        __syncwarp();
        flush();
        pend_g = g;
        pend_i = i;
        pend_j = j;
        pend_o = ob;
        pend_last = i == it.n_kv - 1;
      }
    }
    flush();
  } else if (warp >= C::SW0) {
    const int q = warp & 3;
    const int grp = (warp - C::SW0) >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float* xmax = reinterpret_cast<float*>(sm + C::XMAX);
    float* xsum = reinterpret_cast<float*>(sm + C::XSUM);
    uint64_t *sf = s_full(grp), *se = s_empty(grp), *pf = p_full(grp), *pe = p_empty(grp);
    // Item jj is finished by whichever group's warp of this quadrant arrives second.
    auto epilogue = [&](const FwdItem& it, int jj, float m, float l) {
      const int ob = jj % NOB, par = jj % C::XS;
      xmax[(par * NG + grp) * 128 + r] = m;
      xsum[(par * NG + grp) * 128 + r] = l;
      __threadfence_block();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(&cnt[par * 4 + q], 1);
      old = __shfl_sync(kFull, old, 0);
      if (old != NG - 1) return;
      __threadfence_block();
      const uint32_t ph = (jj / NOB) & 1;
#pragma unroll
      for (int c = 0; c < NG; ++c) mbar_wait(&o_full(c)[ob], ph);
      tc_fence_after();
      float fc[NG], M = -INFINITY, l_all = 0.f;
#pragma unroll
      for (int c = 0; c < NG; ++c) M = fmaxf(M, xmax[(par * NG + c) * 128 + r]);
#pragma unroll
      for (int c = 0; c < NG; ++c) {
        const float mc = xmax[(par * NG + c) * 128 + r];
        fc[c] = mc == -INFINITY ? 0.f : ex2(mc - M);
        l_all += xsum[(par * NG + c) * 128 + r] * fc[c];
      }
      const float rl = __frcp_rn(l_all);
#pragma unroll
      for (int c = 0; c < NG; ++c) fc[c] *= rl;
      const int qpos = it.q0 + r;
#pragma unroll
      for (int sub = 0; sub < DH / 32; ++sub) {
        float acc[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[e] = 0.f;
#pragma unroll
        for (int c = 0; c < NG; ++c) {
          uint32_t ra[32];
          tmem_ld_32x32b_x32(tmem + lane_base + C::o_col(ob, c) + sub * 32, ra);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) acc[e] = fmaf(__uint_as_float(ra[e]), fc[c], acc[e]);
        }
        if (sub == DH / 32 - 1) {  // every group's O read: the slot's counter is reset before release
          if (lane == 0) cnt[par * 4 + q] = 0;
          __threadfence_block();
          tc_fence_before();
#pragma unroll
          for (int c = 0; c < NG; ++c) mbar_arrive(&o_empty(c)[ob]);
        }
        if (qpos < it.L) {
          uint32_t o[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) o[e] = pack_bf16(acc[2 * e], acc[2 * e + 1]);
          uint4* dst = reinterpret_cast<uint4*>(out + (size_t)(it.s0 + qpos) * ldo + it.h * DH + sub * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u) dst[u] = make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
        }
      }
      if (qpos < it.L) lse[(size_t)it.h * T + it.s0 + qpos] = (M + log2f(l_all)) * LN2_F;
    };
    int g = 0, j = 0;
    bool pend = false;
    FwdItem pit{};
    int pj = 0;
    float pm = 0.f, pl = 0.f;
    int w = snake_item(0);
    FwdItem it{};
    if (w < n_items) it = fwd_item<CAUSAL>(w, H, Hk, cu, tiles);
    for (; w < n_items; ++j) {
      const int w_next = snake_item(j + 1);
      FwdItem nxt{};
      if (w_next < n_items) nxt = fwd_item<CAUSAL>(w_next, H, Hk, cu, tiles);
      const int ob = j % NOB;
      const int qpos = it.q0 + r;
      float m = -INFINITY, l = 0.f;
      for (int i = 0; i < it.n_kv; ++i, ++g) {
        const int b = g & 1;
        mbar_wait(&sf[b], (g >> 1) & 1);
        tc_fence_after();
        const uint32_t s_col = tmem + lane_base + C::s_col(grp, b);
        float s[CW];
        {
          uint32_t raw[CW / 32][32];
#pragma unroll
          for (int c = 0; c < CW / 32; ++c) tmem_ld_32x32b_x32(s_col + 32 * c, raw[c]);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < CW / 32; ++c)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) s[c * 32 + jj] = __uint_as_float(raw[c][jj]);
        }
        tc_fence_before();
        mbar_arrive(&se[b]);
        const int kv0 = i * BKV + grp * CW;
        const bool need_mask = (CAUSAL && kv0 + CW - 1 > it.q0) || (kv0 + CW > it.L);
        const int lim = CAUSAL ? min(qpos - kv0 + 1, it.L - kv0) : it.L - kv0;
        if (need_mask && __all_sync(kFull, lim <= 0)) {
          uint32_t zero[CW / 2];
#pragma unroll
          for (int e = 0; e < CW / 2; ++e) zero[e] = 0u;
          tmem_st_cols<CW / 2>(s_col, zero);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&pf[b]);
          if (i == 0 && pend) {
            epilogue(pit, pj, pm, pl);
            pend = false;
          }
          continue;
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (need_mask) {
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            s[c] = c < lim ? s[c] : -INFINITY;
            mx4[c & 3] = fmaxf(mx4[c & 3], s[c]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < CW; ++c) mx4[c & 3] = fmaxf(mx4[c & 3], s[c]);
        }
        const float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * scale2;
        bool rescale = false;
        float alpha = 1.f;
        if (m_new > m + 8.0f) {
          alpha = ex2(m - m_new);
          m = m_new;
          rescale = i > 0;
        }
        const float neg_m = m == -INFINITY ? 0.f : -m;
        const float2 sc2 = make_float2(scale2, scale2), nm2 = make_float2(neg_m, neg_m);
        float2 sum2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
        for (int c = 0; c < CW; c += 2) {
          const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), sc2, nm2);
          if ((FWD_EMU_BITS >> ((c >> 1) & 7)) & 1) {
            const float2 e = ex2_fma2<3>(x);
            s[c] = e.x;
            s[c + 1] = e.y;
          } else {
            s[c] = ex2(x.x);
            s[c + 1] = ex2(x.y);
          }
          sum2[(c >> 1) & 3] = __fadd2_rn(sum2[(c >> 1) & 3], make_float2(s[c], s[c + 1]));
        }
        const float2 t01 = __fadd2_rn(sum2[0], sum2[1]), t23 = __fadd2_rn(sum2[2], sum2[3]);
        const float2 t = __fadd2_rn(t01, t23);
        l = l * alpha + (t.x + t.y);
        if (__any_sync(kFull, rescale)) {  // warp-collective TMEM access (see attn_fwd_kernel)
          if (!rescale) alpha = 1.f;
          mbar_wait(&pe[(g - 1) & 1], ((g - 1) >> 1) & 1);  // PV_{g-1} of this group retired
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tmem + lane_base + C::o_col(ob, grp) + c * 32, rr);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) rr[jj] = __float_as_uint(__uint_as_float(rr[jj]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_base + C::o_col(ob, grp) + c * 32, rr);
          }
          tmem_st_wait();
        }
        {
          uint32_t pk[CW / 2];
#pragma unroll
          for (int e = 0; e < CW / 2; ++e) pk[e] = pack_bf16(s[2 * e], s[2 * e + 1]);
          tmem_st_cols<CW / 2>(s_col, pk);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&pf[b]);
        if (i == 0 && pend) {
          epilogue(pit, pj, pm, pl);
          pend = false;
        }
      }
      pend = true;
      pit = it;
      pj = j;
      pm = m;
      pl = l;
      it = nxt;
      w = w_next;
    }
    if (pend) epilogue(pit, pj, pm, pl);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------------------------------
// Forward, ping-pong (FA4-style): one CTA item = 256 queries (two 128-row Q tiles A and B) of
// one head, sharing every K/V tile.  Each Q tile has its own softmax warpgroup (thread = row, all
// 128 key columns, read from TMEM in two 64-column halves: row max, then exponentials), its own
// S buffer and O accumulator.  The MMA warp issues S_A(0) S_B(0), then per KV tile
// PV_A(i) S_A(i+1) PV_B(i) S_B(i+1), so while warpgroup A turns S_A(i) into P_A(i) the tensor core
// works on tile B and vice versa: the two softmax warps of an SM sub-partition (one per Q tile)
// are half a period apart instead of running the same phase at the same time.  S_t(i+1) is issued
// after PV_t(i), so its completion barrier also covers O_t (lazy rescale without another wait).
// Warps: w0 TMA, w1 MMA, w2-3 idle, w4-7 softmax A, w8-11 softmax B (quadrant = warp & 3).
// TMEM: S_A [0,128) S_B [128,256); O_t at 256 + (ob * 2 + t) * DH (head_dim 64: two sets by item)
// or 256 + t * 128 (head_dim 128).
template <int DH>
struct FwdPPCfg {
  static constexpr int THREADS = 384;
  static constexpr int TILE = 128 * DH * 2;
  static constexpr int QB = DH == 64 ? 2 : 1;  // Q-pair buffers (by item)
  static constexpr int KVS = DH == 64 ? 3 : 2;
  static constexpr int NOB = DH == 64 ? 2 : 1;
  static constexpr int Q = 0;  // [QB][2] tiles
  static constexpr int K = Q + QB * 2 * TILE;
  static constexpr int V = K + KVS * TILE;
  static constexpr int BAR = V + KVS * TILE;
  static constexpr int TOTAL = BAR + 512;
  static_assert(TOTAL + 1024 <= 227 * 1024, "forward smem");
  __device__ static constexpr uint32_t o_col(int ob, int t) { return 256 + (ob * 2 + t) * DH; }
};

struct PPItem {
  int seq, q0, h, hk, s0, L, n[2], nk;
};

template <bool CAUSAL>
__device__ __forceinline__ PPItem pp_item(int w, int H, int Hk, const int32_t* cu, const int2* tiles) {
  PPItem it;
  const int2 tq = tiles[w / H];
  it.seq = tq.x;
  it.q0 = tq.y;
  it.h = w % H;
  it.hk = it.h / (H / Hk);
  it.s0 = cu[it.seq];
  it.L = cu[it.seq + 1] - it.s0;
  const int n_all = (it.L + BKV - 1) / BKV;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int q0t = it.q0 + t * BQ;
    it.n[t] = q0t >= it.L ? 0 : (CAUSAL ? min(n_all, q0t / BKV + 1) : n_all);
  }
  it.nk = max(it.n[0], it.n[1]);
  return it;
}

template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(FwdPPCfg<DH>::THREADS, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, const int32_t* __restrict__ cu,
                       const int2* __restrict__ tiles, const int* __restrict__ n_tiles,
                       __nv_bfloat16* __restrict__ out, int ldo, float* __restrict__ lse, int T, int H, int Hk,
                       float scale2) {
  using C = FwdPPCfg<DH>;
  constexpr int KVS = C::KVS, NOB = C::NOB, QB = C::QB, TB = C::TILE;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR);
  uint64_t* q_full = bar;           // [QB]
  uint64_t* q_empty = bar + 2;      // [QB]
  uint64_t* k_full = bar + 4;       // [KVS]
  uint64_t* k_empty = k_full + KVS;
  uint64_t* v_full = k_empty + KVS;
  uint64_t* v_empty = v_full + KVS;
  uint64_t* s_full = v_empty + KVS;  // [2 tiles]
  uint64_t* p_full = s_full + 2;     // [2 tiles]
  uint64_t* o_full = p_full + 2;     // [2 tiles][2 sets]
  uint64_t* o_empty = o_full + 4;    // [2 tiles][2 sets]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 128);
    }
    for (int s = 0; s < KVS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above (barriers, TMEM, tensor-map prefetch)
  // overlapped the previous kernel; global memory (the tile list included) only from here
  pdl_trigger();
  pdl_wait();
  const int n_items = *n_tiles * H;

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, j = 0;
      for (int w = snake_item(0); w < n_items; w = snake_item(++j)) {
        const PPItem it = pp_item<CAUSAL>(w, H, Hk, cu, tiles);
        const int qb = j % QB;
        prod_wait(&q_empty[qb], ((j / QB) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], TB * (it.n[1] > 0 ? 2 : 1));
        load_tile<DH>(sm + C::Q + qb * 2 * TB, &map_q, &q_full[qb], it.h * DH, it.s0 + it.q0);
        if (it.n[1] > 0) load_tile<DH>(sm + C::Q + (qb * 2 + 1) * TB, &map_q, &q_full[qb], it.h * DH, it.s0 + it.q0 + BQ);
        for (int i = 0; i < it.nk; ++i, ++g) {
          const int st = g % KVS;
          const uint32_t ph = (g / KVS) & 1;
          prod_wait(&k_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&k_full[st], TB);
          load_tile<DH>(sm + C::K + st * TB, &map_k, &k_full[st], it.hk * DH, it.s0 + i * BKV);
          prod_wait(&v_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&v_full[st], TB);
          load_tile<DH>(sm + C::V + st * TB, &map_v, &v_full[st], it.hk * DH, it.s0 + i * BKV);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = idesc_bf16_f32(BQ, BKV, false, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BQ, DH, false, true);
    int g = 0, j = 0;
    int np[2] = {0, 0};   // PVs issued per tile (p_full parity)
    int nw[2] = {0, 0};   // items with work per tile (O set, o_empty parity)
    for (int w = snake_item(0); w < n_items; w = snake_item(++j)) {
      const PPItem it = pp_item<CAUSAL>(w, H, Hk, cu, tiles);
      const int qb = j % QB;
      prod_wait(&q_full[qb], (j / QB) & 1);
      const uint32_t q_base = smem_u32(sm + C::Q + qb * 2 * TB);
      const int n_s = it.n[0] + it.n[1];
      int s_done = 0;
      auto issue_s = [&](int t, int kst) {  // S_t = Q_t K^T (K tile in ring stage kst)
        const uint32_t k_base = smem_u32(sm + C::K + kst * TB);
        const uint32_t qt = q_base + t * TB;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            umma_bf16(tmem + t * BKV, sdesc((qt >> 4) + (kk >> 2) * 1024 + (kk & 3) * 2, 16, 1024),
                      sdesc((k_base >> 4) + (kk >> 2) * 1024 + (kk & 3) * 2, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
          umma_commit(&s_full[t]);
          if (++s_done == n_s) umma_commit(&q_empty[qb]);  // last S of the item: Q pair free
        } else {
          ++s_done;
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int i, int vst) {  // O_t += P_t V (V tile in ring stage vst)
        const int ob = nw[t] % NOB;
        if (i == 0) prod_wait(&o_empty[t * 2 + ob], ((nw[t] / NOB) & 1) ^ 1);
        prod_wait(&p_full[t], np[t] & 1);
        ++np[t];
        tc_fence_after();
        const uint32_t v_base = smem_u32(sm + C::V + vst * TB);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            umma_bf16_ts(tmem + C::o_col(ob, t), tmem + t * BKV + kk * 8,
                         sdesc((v_base >> 4) + kk * 128, DH == 64 ? 8192 : 16384, 1024), idesc_o,
                         (i > 0 || kk > 0) ? 1u : 0u);
          if (i == it.n[t] - 1) umma_commit(&o_full[t * 2 + ob]);
        }
        __syncwarp();
        if (i == it.n[t] - 1) ++nw[t];
      };
      // prologue: S_A(0), S_B(0)
      {
        const int st = g % KVS;
        prod_wait(&k_full[st], (g / KVS) & 1);
        tc_fence_after();
        for (int t = 0; t < 2; ++t)
          if (it.n[t] > 0) issue_s(t, st);
        if (elect_one()) umma_commit(&k_empty[st]);
        __syncwarp();
      }
      for (int i = 0; i < it.nk; ++i) {
        const int st = (g + i) % KVS, st1 = (g + i + 1) % KVS;
        prod_wait(&v_full[st], ((g + i) / KVS) & 1);
        const bool more = i + 1 < it.nk;
        if (more) prod_wait(&k_full[st1], ((g + i + 1) / KVS) & 1);
        for (int t = 0; t < 2; ++t) {
          if (i < it.n[t]) issue_pv(t, i, st);
          if (i + 1 < it.n[t]) {
            tc_fence_after();
            issue_s(t, st1);
          }
        }
        if (elect_one()) {
          umma_commit(&v_empty[st]);
          if (more) umma_commit(&k_empty[st1]);
        }
        __syncwarp();
      }
      g += it.nk;
    }
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;  // Q tile of this warpgroup
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t s_col = tmem + lane_base + t * BKV;
    int c = 0;                       // S tiles consumed (s_full parity)
    int nw = 0;                      // items with work for this tile
    auto epilogue = [&](const PPItem& it, int wi, float m, float l) {
      const int ob = wi % NOB;
      mbar_wait(&o_full[t * 2 + ob], (wi / NOB) & 1);
      tc_fence_after();
      const int qpos = it.q0 + t * BQ + r;
      const float rl = __frcp_rn(l);
#pragma unroll
      for (int sub = 0; sub < DH / 32; ++sub) {
        uint32_t ra[32];
        tmem_ld_32x32b_x32(tmem + lane_base + C::o_col(ob, t) + sub * 32, ra);
        tmem_ld_wait();
        if (sub == DH / 32 - 1) {
          tc_fence_before();
          mbar_arrive(&o_empty[t * 2 + ob]);
        }
        if (qpos < it.L) {
          uint32_t o[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            o[e] = pack_bf16(__uint_as_float(ra[2 * e]) * rl, __uint_as_float(ra[2 * e + 1]) * rl);
          uint4* dst = reinterpret_cast<uint4*>(out + (size_t)(it.s0 + qpos) * ldo + it.h * DH + sub * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u) dst[u] = make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
        }
      }
      if (qpos < it.L) lse[(size_t)it.h * T + it.s0 + qpos] = (m + log2f(l)) * LN2_F;
    };
    bool pend = false;
    PPItem pit{};
    int pw = 0;
    float pm = 0.f, pl = 0.f;
    int j = 0;
    for (int w = snake_item(0); w < n_items; w = snake_item(++j)) {
      const PPItem it = pp_item<CAUSAL>(w, H, Hk, cu, tiles);
      const int n_t = it.n[t];
      if (n_t == 0) {  // no rows of this tile in the sequence: nothing to compute
        if (pend) {
          epilogue(pit, pw, pm, pl);
          pend = false;
        }
        continue;
      }
      const int ob = nw % NOB;
      const int q0t = it.q0 + t * BQ;
      const int qpos = q0t + r;
      float m = -INFINITY, l = 0.f;
      for (int i = 0; i < n_t; ++i, ++c) {
        mbar_wait(&s_full[t], c & 1);
        tc_fence_after();
        const int kv0 = i * BKV;
        const bool need_mask = (CAUSAL && kv0 + BKV - 1 > q0t) || (kv0 + BKV > it.L);
        const int lim = CAUSAL ? min(qpos - kv0 + 1, it.L - kv0) : it.L - kv0;
        // pass 1: row max over both 64-column halves
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t raw[2][32];
          tmem_ld_32x32b_x32(s_col + h * 64, raw[0]);
          tmem_ld_32x32b_x32(s_col + h * 64 + 32, raw[1]);
          tmem_ld_wait();
          if (need_mask) {
#pragma unroll
            for (int e = 0; e < 64; ++e)
              mx4[e & 3] = fmaxf(mx4[e & 3], h * 64 + e < lim ? __uint_as_float(raw[e >> 5][e & 31]) : -INFINITY);
          } else {
#pragma unroll
            for (int e = 0; e < 64; ++e) mx4[e & 3] = fmaxf(mx4[e & 3], __uint_as_float(raw[e >> 5][e & 31]));
          }
        }
        const float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * scale2;
        bool rescale = false;
        float alpha = 1.f;
        if (m_new > m + 8.0f) {
          alpha = ex2(m - m_new);
          m = m_new;
          rescale = i > 0;
        }
        // O_t is final for the previous tiles: S_t(i) was issued after PV_t(i-1)
        if (__any_sync(kFull, rescale)) {
          if (!rescale) alpha = 1.f;
#pragma unroll
          for (int cc = 0; cc < DH / 32; ++cc) {
            uint32_t rr[32];
            tmem_ld_32x32b_x32(tmem + lane_base + C::o_col(ob, t) + cc * 32, rr);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) rr[e] = __float_as_uint(__uint_as_float(rr[e]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_base + C::o_col(ob, t) + cc * 32, rr);
          }
        }
        const float neg_m = m == -INFINITY ? 0.f : -m;
        const float2 sc2 = make_float2(scale2, scale2), nm2 = make_float2(neg_m, neg_m);
        float2 sum2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
        // pass 2: exponentials of each half, packed to bf16 P over the first 64 columns of S_t
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float s[64];
          {
            uint32_t raw[2][32];
            tmem_ld_32x32b_x32(s_col + h * 64, raw[0]);
            tmem_ld_32x32b_x32(s_col + h * 64 + 32, raw[1]);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 64; ++e) {
              const float x = __uint_as_float(raw[e >> 5][e & 31]);
              s[e] = (!need_mask || h * 64 + e < lim) ? x : -INFINITY;
            }
          }
#pragma unroll
          for (int e = 0; e < 64; e += 2) {
            const float2 x = __ffma2_rn(make_float2(s[e], s[e + 1]), sc2, nm2);
            if ((FWD_EMU_BITS >> ((e >> 1) & 7)) & 1) {
              const float2 y = ex2_fma2<3>(x);
              s[e] = y.x;
              s[e + 1] = y.y;
            } else {
              s[e] = ex2(x.x);
              s[e + 1] = ex2(x.y);
            }
            sum2[(e >> 1) & 3] = __fadd2_rn(sum2[(e >> 1) & 3], make_float2(s[e], s[e + 1]));
          }
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) pk[e] = pack_bf16(s[2 * e], s[2 * e + 1]);
          tmem_st_32x32b_x32(s_col + h * 32, pk);
        }
        const float2 t01 = __fadd2_rn(sum2[0], sum2[1]), t23 = __fadd2_rn(sum2[2], sum2[3]);
        const float2 tt = __fadd2_rn(t01, t23);
        l = l * alpha + (tt.x + tt.y);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[t]);
        if (i == 0 && pend) {
          epilogue(pit, pw, pm, pl);
          pend = false;
        }
      }
      pend = true;
      pit = it;
      pw = nw;
      pm = m;
      pl = l;
      ++nw;
    }
    if (pend) epilogue(pit, pw, pm, pl);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ==========================================================================================
// Backward, persistent: one CTA per SM loops over items (128-row KV tile, KV head) in
// heavy-first order; an item loops over the query heads of its GQA group and the query tiles
// (BQB rows) its keys can see.  Thread r of the 4 softmax warps owns KV row r:
//   S^T = K Q^T, dP^T = V dO^T                      (TMEM, M = kv, N = q)
//   P1: P^T = exp2(S^T * scale2 - lse2[q])            -> bf16 TMEM operand     (p_ready)
//   P2: dS^T = P^T (dP^T - D[q])                      -> bf16 TMEM + smem      (ds_ready)
//   dV += P^T dO, dK += dS^T Q                      (TMEM accumulators across the item)
//   dQ_tile = dS K  (head_dim 64)  or  dQ^T_tile = K^T dS^T (head_dim 128)   (TMEM, drained by
//                                                    TMA reduce-add into an fp32 accumulator)
// P^T and dS^T go back to TMEM as bf16 pairs (thread = kv row = TMEM lane), so dV and dK are
// TS-MMAs with A from TMEM (no shared-memory operand traffic; dS^T also goes to smem as the dQ
// operand).  P1 pulls S^T into registers first and releases it (s_empty), so S(i+1) runs while
// P1/P2(i) compute; dS^T reuses the dP^T columns, so dP(i+1) is issued after dK(i).
// Two softmax warps share each TMEM lane quadrant and split the BQB query columns (the backward
// needs no row reductions), so every SM sub-partition interleaves two softmax warps.
//
// head_dim 64:  BQB = 128; TMEM S^T [0,128), dP^T [128,256), dV [256,320), dK [320,384),
//               dQ [384,448) (M = q, N = dh), P^T [448,512); K/V double-buffered by item.
// head_dim 128: BQB = 64 (the dV / dK accumulators take 256 columns); TMEM S^T [0,64),
//               dP^T [64,128), dV [128,256), dK [256,384), dQ^T [384,448) (M = dh, N = q: its
//               A operand is K read as an MN-major view, B = dS^T), P^T [448,480); K/V single-
//               buffered (smem), so the next item's K/V load waits for the item's last MMAs.
// Backward barrier waits sleep on the barrier (suspend hint) instead of polling: +5-8 % at
// head_dim 128, neutral at 64 (r02_attn_suspend_ab.jsonl); the forward keeps polling (-1 %).
__device__ __forceinline__ void bwd_wait(uint64_t* bar, uint32_t parity) { mbar_wait_sleep<20000>(bar, parity); }

constexpr int BWD_THREADS = 448;  // w0 TMA, w1 MMA, w2-9 softmax (2 per lane quadrant), w10-13 dQ drain

template <int DH>
struct BwdCfg {
  static constexpr int BQB = DH == 64 ? 128 : 64;     // query rows per iteration
  static constexpr int QH = BQB / 2;                  // query columns per softmax half
  static constexpr int KV_TILE = 128 * DH * 2;        // K or V tile (128 kv rows)
  static constexpr int Q_TILE = BQB * DH * 2;         // Q or dO tile
  static constexpr int Q_CHUNK = BQB * 128;           // bytes per 64-column chunk of a Q/dO tile
  static constexpr int KVB = DH == 64 ? 2 : 1;        // K/V buffers (by item)
  static constexpr int QD_STAGES = 3;                 // Q/dO ring (two expose the TMA latency)
  static constexpr int KV = 0;
  static constexpr int QD = KV + KVB * 2 * KV_TILE;
  static constexpr int DST = QD + QD_STAGES * 2 * Q_TILE;  // dS^T [kv][q] bf16 (dQ operand)
  static constexpr int LSE = DST + 128 * BQB * 2;           // 2 x BQB fp32 (double-buffered by tile)
  static constexpr int DD = LSE + 1024;
  static constexpr int DQS = DD + 1024;                     // dQ staging, 4 drain warps
  static constexpr int DQS_WARP = DH == 64 ? 4096 : 8192;   // 32 x 32 fp32 | 64 q x 32 dh fp32
  static constexpr int BAR = DQS + 4 * DQS_WARP;
  static constexpr int TOTAL = BAR + 256;
  // TMEM columns
  static constexpr uint32_t T_ST = 0, T_DPT = BQB, T_DV = 2 * BQB, T_DK = 2 * BQB + DH, T_DQ = 2 * BQB + 2 * DH,
                            T_PT = 448;
  static_assert(TOTAL + 1024 <= 227 * 1024, "backward smem");
  static_assert(T_DQ + (DH == 64 ? DH : BQB) <= T_PT && T_PT + BQB / 2 <= 512, "backward TMEM");
};

struct BwdItem {
  int kv0, hk, s0, L, qt_first, n_q, n_it;
};

template <int BQB, bool CAUSAL>
__device__ __forceinline__ BwdItem bwd_item(int w, int Hk, int G, const int32_t* cu, const int2* tiles) {
  BwdItem it;
  const int2 tk = tiles[w / Hk];
  it.kv0 = tk.y;
  it.hk = w % Hk;
  it.s0 = cu[tk.x];
  it.L = cu[tk.x + 1] - it.s0;
  const int n_q_all = (it.L + BQB - 1) / BQB;
  it.qt_first = CAUSAL ? it.kv0 / BQB : 0;
  it.n_q = n_q_all - it.qt_first;
  it.n_it = G * it.n_q;
  return it;
}

// Flat cursor over (item, iteration) for the MMA warp's one-iteration lookahead.
template <int BQB, bool CAUSAL>
struct BwdCursor {
  int j, w, it;
  bool valid;
  BwdItem item;
  __device__ __forceinline__ void load(int n_items, int Hk, int G, const int32_t* cu, const int2* tiles) {
    w = snake_item(j);
    valid = w < n_items;
    if (valid) item = bwd_item<BQB, CAUSAL>(w, Hk, G, cu, tiles);
  }
  __device__ __forceinline__ void next(int n_items, int Hk, int G, const int32_t* cu, const int2* tiles) {
    if (++it == item.n_it) {
      ++j;
      it = 0;
      load(n_items, Hk, G, cu, tiles);
    }
  }
};

template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do,
                    const __grid_constant__ CUtensorMap map_dq, const int32_t* __restrict__ cu,
                    const int2* __restrict__ tiles, const int* __restrict__ n_tiles,
                    const float* __restrict__ lse, const float* __restrict__ Dvec,
                    __nv_bfloat16* __restrict__ dk, int lddk, __nv_bfloat16* __restrict__ dv, int lddv, int T, int H,
                    int Hk, float scale2, float scale, const float2* __restrict__ rope_cs) {
  using C = BwdCfg<DH>;
  constexpr int BQB = C::BQB, QH = C::QH, QDS = C::QD_STAGES, KVB = C::KVB;
  constexpr int KVT = C::KV_TILE, QT = C::Q_TILE;
  constexpr uint32_t T_ST = C::T_ST, T_DPT = C::T_DPT, T_DV = C::T_DV, T_DK = C::T_DK, T_DQ = C::T_DQ,
                     T_PT = C::T_PT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR);
  uint64_t* kv_full = bar;          // [2]
  uint64_t* kv_empty = bar + 2;     // [2]
  uint64_t* qd_full = bar + 4;      // [QDS]
  uint64_t* qd_empty = bar + 7;     // [QDS]
  uint64_t* s_full = bar + 10;
  uint64_t* dp_full = bar + 11;
  uint64_t* p_ready = bar + 12;
  uint64_t* p_free = bar + 13;
  uint64_t* ds_ready = bar + 14;
  uint64_t* ds_free = bar + 15;
  uint64_t* dq_full = bar + 16;
  uint64_t* dq_empty = bar + 17;
  uint64_t* dkv_full = bar + 18;
  uint64_t* dkv_empty = bar + 19;
  uint64_t* s_empty = bar + 20;   // S^T TMEM loaded by the softmax warps (the next S may overwrite it)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 21);
  float* s_lse = reinterpret_cast<float*>(sm + C::LSE);
  float* s_D = reinterpret_cast<float*>(sm + C::DD);

  const int G = H / Hk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    tma_prefetch(&map_do);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&kv_full[b], 1);
      mbar_init(&kv_empty[b], 1);
    }
    for (int b = 0; b < QDS; ++b) {
      mbar_init(&qd_full[b], 1);
      mbar_init(&qd_empty[b], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_ready, 256 / ARRIVE_UNIT);
    mbar_init(p_free, 1);
    mbar_init(ds_ready, 256 / ARRIVE_UNIT);
    mbar_init(ds_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128 / ARRIVE_UNIT);
    mbar_init(dkv_full, 1);
    mbar_init(dkv_empty, 256 / ARRIVE_UNIT);
    mbar_init(s_empty, 256 / ARRIVE_UNIT);  // arrive counts: see warp_arrive
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above (barriers, TMEM, tensor-map prefetch)
  // overlapped the previous kernel; global memory (the tile list included) only from here
  pdl_trigger();
  pdl_wait();
  const int n_items = *n_tiles * Hk;

  if (warp == 0) {
    if (lane == 0) {
      int gi = 0, j = 0;
      BwdItem itm_n{};
      if (snake_item(0) < n_items) itm_n = bwd_item<BQB, CAUSAL>(snake_item(0), Hk, G, cu, tiles);
      for (int w = snake_item(0); w < n_items; w = snake_item(j + 1), ++j) {
        const BwdItem itm = itm_n;
        if (snake_item(j + 1) < n_items) itm_n = bwd_item<BQB, CAUSAL>(snake_item(j + 1), Hk, G, cu, tiles);  // prefetch
        const int kb = j % KVB;
        bwd_wait(&kv_empty[kb], ((j / KVB) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[kb], 2 * KVT);
        unsigned char* kvd = sm + C::KV + kb * 2 * KVT;
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          tma_load_2d(kvd + c * 16384, &map_k, &kv_full[kb], itm.hk * DH + 64 * c, itm.s0 + itm.kv0);
          tma_load_2d(kvd + KVT + c * 16384, &map_v, &kv_full[kb], itm.hk * DH + 64 * c, itm.s0 + itm.kv0);
        }
        for (int it = 0; it < itm.n_it; ++it, ++gi) {
          const int g = it / itm.n_q, qt = itm.qt_first + it % itm.n_q;
          const int h = itm.hk * G + g;
          const int st = gi % QDS;
          bwd_wait(&qd_empty[st], ((gi / QDS) & 1) ^ 1);
          mbar_arrive_expect_tx(&qd_full[st], 2 * QT);
          unsigned char* dst = sm + C::QD + st * 2 * QT;
#pragma unroll
          for (int c = 0; c < DH / 64; ++c) {
            tma_load_2d(dst + c * C::Q_CHUNK, &map_q, &qd_full[st], h * DH + 64 * c, itm.s0 + qt * BQB);
            tma_load_2d(dst + QT + c * C::Q_CHUNK, &map_do, &qd_full[st], h * DH + 64 * c, itm.s0 + qt * BQB);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the loop; MMAs and commits are issued by one elected lane
      constexpr uint32_t id_sp = idesc_bf16_f32(BKV, BQB, false, false);  // M = kv, N = q
      constexpr uint32_t id_kv = idesc_bf16_f32(BKV, DH, false, true);    // dV, dK: A K-major, B MN-major
      // dQ (dh 64): M = q, N = dh, A = dS (MN-major view of dS^T), B = K (MN-major)
      // dQ^T (dh 128): M = dh, N = q, A = K^T (MN-major view of K), B = dS^T (MN-major)
      constexpr uint32_t id_dq = DH == 64 ? idesc_bf16_f32(BQB, DH, true, true) : idesc_bf16_f32(DH, BQB, true, true);
      const uint32_t ds_base = smem_u32(sm + C::DST);
      auto kv_base = [&](int j) { return smem_u32(sm + C::KV + (j % KVB) * 2 * KVT); };
      auto qd_base = [&](int gi) { return smem_u32(sm + C::QD + (gi % QDS) * 2 * QT); };
      // K-major descriptor of K-step kk over a [rows][DH] tile whose 64-column chunks are `cs` bytes apart
      auto kdesc = [&](uint32_t base, int kk, uint32_t cs) {
        return sdesc((base >> 4) + (kk >> 2) * (cs >> 4) + (kk & 3) * 2, 16, 1024);
      };
      // S^T(gi) = K Q^T and dP^T(gi) = V dO^T of the cursor's iteration
      auto issue_s = [&](const BwdCursor<BQB, CAUSAL>& c, int gi) {
        bwd_wait(&qd_full[gi % QDS], (gi / QDS) & 1);
        if (c.it == 0) bwd_wait(&kv_full[c.j % KVB], (c.j / KVB) & 1);
        if (gi >= 1) bwd_wait(s_empty, (gi - 1) & 1);  // S^T(gi-1) is in the softmax registers
        tc_fence_after();
        const uint32_t kb = kv_base(c.j), qb = qd_base(gi);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            umma_bf16(tmem + T_ST, kdesc(kb, kk, 16384), kdesc(qb, kk, C::Q_CHUNK), id_sp, kk > 0);
          umma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_dp = [&](const BwdCursor<BQB, CAUSAL>& c, int gi) {
        const uint32_t vb = kv_base(c.j) + KVT, db = qd_base(gi) + QT;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            umma_bf16(tmem + T_DPT, kdesc(vb, kk, 16384), kdesc(db, kk, C::Q_CHUNK), id_sp, kk > 0);
          umma_commit(dp_full);
        }
        __syncwarp();
      };
      BwdCursor<BQB, CAUSAL> cur;
      cur.j = 0;
      cur.it = 0;
      cur.load(n_items, Hk, G, cu, tiles);
      int gi = 0;
      if (cur.valid) {
        issue_s(cur, 0);
        issue_dp(cur, 0);
      }
      while (cur.valid) {
        BwdCursor<BQB, CAUSAL> nxt = cur;
        nxt.next(n_items, Hk, G, cu, tiles);
        const uint32_t qb = qd_base(gi), kb = kv_base(cur.j);
        // S^T(gi+1) as soon as P1(gi) has pulled S^T(gi) into registers: it runs while P1/P2(gi) compute
        // (head_dim 128: a new item's S also waits for its K/V, i.e. for the previous item's last MMAs)
        if (nxt.valid && (KVB == 2 || nxt.it > 0)) issue_s(nxt, gi + 1);
        // dV += P^T dO   (B = dO, MN-major: N = dh over DH/64 atoms Q_CHUNK apart, K = q rows)
        bwd_wait(p_ready, gi & 1);
        if (cur.it == 0) bwd_wait(dkv_empty, (cur.j & 1) ^ 1);  // previous item's epilogue read dK/dV
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BQB / 16; ++kk)  // reduction over the BQB queries; A = P^T from TMEM
            umma_bf16_ts(tmem + T_DV, tmem + T_PT + kk * 8, sdesc(((qb + QT) >> 4) + kk * 128, C::Q_CHUNK, 1024),
                         id_kv, (cur.it > 0 || kk > 0) ? 1u : 0u);
          umma_commit(p_free);
        }
        __syncwarp();
        // dK += dS^T Q (A = dS^T from TMEM) ; dQ from the dS^T smem operand
        bwd_wait(ds_ready, gi & 1);
        bwd_wait(dq_empty, (gi & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BQB / 16; ++kk)  // half kk / (QH/16) holds dS^T in the first QH/2 of its QH dP^T columns
            umma_bf16_ts(tmem + T_DK, tmem + T_DPT + (kk / (QH / 16)) * QH + (kk % (QH / 16)) * 8,
                         sdesc((qb >> 4) + kk * 128, C::Q_CHUNK, 1024), id_kv, (cur.it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {  // reduction over the 128 keys (16 kv rows = 2 KB per step)
            if constexpr (DH == 64)
              umma_bf16(tmem + T_DQ, sdesc((ds_base >> 4) + kk * 128, 16384, 1024),
                        sdesc((kb >> 4) + kk * 128, 8192, 1024), id_dq, kk > 0 ? 1u : 0u);
            else
              umma_bf16(tmem + T_DQ, sdesc((kb >> 4) + kk * 128, 16384, 1024),
                        sdesc((ds_base >> 4) + kk * 128, 8192, 1024), id_dq, kk > 0 ? 1u : 0u);
          }
          umma_commit(dq_full);
          umma_commit(&qd_empty[gi % QDS]);
          umma_commit(ds_free);
          if (cur.it == cur.item.n_it - 1) {
            umma_commit(dkv_full);
            umma_commit(&kv_empty[cur.j % KVB]);
          }
        }
        __syncwarp();
        // head_dim 128: the first S of the next item once its K/V (single buffer) has landed
        if (nxt.valid && KVB == 1 && nxt.it == 0) issue_s(nxt, gi + 1);
        // dP^T(gi+1) after dK(gi) (in issue order) has read dS^T out of the dP^T columns
        if (nxt.valid) issue_dp(nxt, gi + 1);
        cur = nxt;
        ++gi;
      }
    }
  } else if (warp >= 10) {
    // ---------------- dQ drain: TMEM -> smem (SWIZZLE_128B boxes of 32 fp32 columns) -> TMA
    // reduce-add into the fp32 accumulator.  Rows past the sequence end are exact zeros (their
    // dS columns were masked), so whole boxes are added; the map clips rows past T.
    const int q4 = warp & 3;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    unsigned char* stage = sm + C::DQS + q4 * C::DQS_WARP;
    bool staged = false;
    int gi = 0, j = 0;
    BwdItem itm_n{};
    if (snake_item(0) < n_items) itm_n = bwd_item<BQB, CAUSAL>(snake_item(0), Hk, G, cu, tiles);
    for (int w = snake_item(0); w < n_items; w = snake_item(j + 1), ++j) {
      const BwdItem itm = itm_n;
      if (snake_item(j + 1) < n_items) itm_n = bwd_item<BQB, CAUSAL>(snake_item(j + 1), Hk, G, cu, tiles);  // prefetch
      for (int it = 0; it < itm.n_it; ++it, ++gi) {
        const int g = it / itm.n_q, qt = itm.qt_first + it % itm.n_q;
        const int h = itm.hk * G + g;
        bwd_wait(dq_full, gi & 1);
        tc_fence_after();
        uint32_t qa[32], qb[32];
        tmem_ld_32x32b_x32(tmem + lane_base + T_DQ, qa);
        tmem_ld_32x32b_x32(tmem + lane_base + T_DQ + 32, qb);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive(dq_empty);  // TMEM free as soon as it is in registers
        if constexpr (DH == 64) {
          // lane = query row q4*32 + lane, registers = dh columns [0,32) and [32,64)
#pragma unroll
          for (int hc = 0; hc < 2; ++hc) {
            const uint32_t* x = hc == 0 ? qa : qb;
            if (staged) {  // the previous box has been read out of the staging buffer
              if (lane == 0) bulk_wait_read<0>();
              __syncwarp();
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<uint4*>(stage + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                  make_uint4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_2d(&map_dq, stage, h * DH + hc * 32, itm.s0 + qt * BQB + q4 * 32);
              bulk_commit();
            }
            staged = true;
          }
        } else {
          // dQ^T: lane = dh column q4*32 + lane, registers = the 64 query rows; one [64 q][32 dh]
          // box per warp (each row's 32 floats are one swizzled 128-byte line)
          if (staged) {
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
          }
#pragma unroll
          for (int r = 0; r < 64; ++r) {
            const uint32_t v = r < 32 ? qa[r] : qb[r - 32];
            *reinterpret_cast<uint32_t*>(stage + r * 128 + ((((lane >> 2) ^ (r & 7))) << 4) + (lane & 3) * 4) = v;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_reduce_add_2d(&map_dq, stage, h * DH + q4 * 32, itm.s0 + qt * BQB);
            bulk_commit();
          }
          staged = true;
        }
      }
    }
    if (lane == 0) bulk_wait<0>();
  } else {
    const int q4 = warp & 3;
    const int half = (warp - 2) >> 2;  // query columns [QH * half, QH * half + QH)
    const int r = q4 * 32 + lane;      // kv row (S^T, dP^T, dK, dV)
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const int tid = threadIdx.x - 64;  // 0..255
    unsigned char* dst = sm + C::DST;
    // This thread's -lse2 (tid < 128) or -D (tid >= 128) entry of iteration `it` of item `im`; loaded
    // one iteration ahead so the global-load latency stays off the per-tile path.
    auto fetch_row = [&](const BwdItem& im, int it) -> float {
      const int hh = im.hk * G + it / im.n_q;
      const int qi = (im.qt_first + it % im.n_q) * BQB + (tid & 127);
      if ((tid & 127) >= BQB || qi >= im.L) return tid < 128 ? -INFINITY : 0.f;  // stored negated: -lse2, -D
      return tid < 128 ? -lse[(size_t)hh * T + im.s0 + qi] * LOG2E_F : -Dvec[(size_t)hh * T + im.s0 + qi];
    };
    int gi = 0, j = 0;
    BwdItem itm_n{};
    float row_next = 0.f;
    if (snake_item(0) < n_items) {
      itm_n = bwd_item<BQB, CAUSAL>(snake_item(0), Hk, G, cu, tiles);
      row_next = fetch_row(itm_n, 0);
    }
    for (int w = snake_item(0); w < n_items; w = snake_item(j + 1), ++j) {
      const BwdItem itm = itm_n;
      const bool has_next = snake_item(j + 1) < n_items;
      if (has_next) itm_n = bwd_item<BQB, CAUSAL>(snake_item(j + 1), Hk, G, cu, tiles);  // prefetch
      const int kvpos = itm.kv0 + r;
      for (int it = 0; it < itm.n_it; ++it, ++gi) {
        const int q0 = (itm.qt_first + it % itm.n_q) * BQB;
        float* lse_t = s_lse + (gi & 1) * 128;  // double-buffered: one barrier per tile suffices
        float* D_t = s_D + (gi & 1) * 128;
        if ((tid & 127) < BQB) (tid < 128 ? lse_t : D_t)[tid & 127] = row_next;
        if (it + 1 < itm.n_it)
          row_next = fetch_row(itm, it + 1);
        else if (has_next)
          row_next = fetch_row(itm_n, 0);
        named_bar(1, 256);
        const bool need_mask =
            (CAUSAL && q0 < itm.kv0 + BKV - 1) || (q0 + BQB > itm.L) || (itm.kv0 + BKV > itm.L);
        // ---- P1: S^T -> P^T
        bwd_wait(s_full, gi & 1);
        tc_fence_after();
        uint32_t sr2[QH / 32][32];
#pragma unroll
        for (int c = 0; c < QH / 32; ++c) tmem_ld_32x32b_x32(tmem + lane_base + T_ST + half * QH + 32 * c, sr2[c]);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive(s_empty);
        if (gi >= 1) bwd_wait(p_free, (gi - 1) & 1);  // dV(gi-1) has read P^T
        uint32_t pk[QH / 2];  // this row's P^T as bf16 pairs: the dV operand, and P for phase 2
        // Two instantiations so that interior tiles carry no per-element mask code (if-converted
        // compares and selects otherwise cost more issue slots than the exponentials).
        auto phase1 = [&](auto masked) {
#pragma unroll
          for (int cc = 0; cc < QH; cc += 32) {
            const int c0 = half * QH + cc;
            const uint32_t* sr = sr2[cc >> 5];
            // valid columns c0 + i: i >= lo (causal: query not before the key), i < hi (inside the sequence)
            const int lo = CAUSAL ? kvpos - (q0 + c0) : INT_MIN;
            const int hi = kvpos >= itm.L ? INT_MIN : itm.L - (q0 + c0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float4 la = *reinterpret_cast<const float4*>(lse_t + c0 + 8 * u);
              const float4 lb = *reinterpret_cast<const float4*>(lse_t + c0 + 8 * u + 4);
              const float lv[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
              float pv[8];
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[8 * u + e]), __uint_as_float(sr[8 * u + e + 1])),
                                            make_float2(scale2, scale2), make_float2(lv[e], lv[e + 1]));
                if ((BWD_EMU_BITS >> (((cc + 8 * u + e) >> 1) & 7)) & 1) {
                  const float2 y = ex2_fma2<3>(x);
                  pv[e] = y.x;
                  pv[e + 1] = y.y;
                } else {
                  pv[e] = ex2(x.x);
                  pv[e + 1] = ex2(x.y);
                }
              }
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                if constexpr (decltype(masked)::value) {
                  const int i = 8 * u + e;
                  if (i < lo || i >= hi) pv[e] = 0.f;
                }
              }
#pragma unroll
              for (int e = 0; e < 4; ++e) pk[cc / 2 + 4 * u + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
            }
          }
        };
        if (need_mask)
          phase1(std::true_type{});
        else
          phase1(std::false_type{});
        if constexpr (QH == 64)
          tmem_st_32x32b_x32(tmem + lane_base + T_PT + half * 32, pk);
        else
          tmem_st_32x32b_x16(tmem + lane_base + T_PT + half * 16, pk);
        tmem_st_wait();
        tc_fence_before();
        warp_arrive(p_ready);
        // ---- P2: dP^T -> dS^T
        bwd_wait(dp_full, gi & 1);
        tc_fence_after();
        if (gi >= 1) bwd_wait(ds_free, (gi - 1) & 1);  // dQ(gi-1) has read the dS^T smem operand
        uint32_t dk2[QH / 2];  // dS^T as bf16 pairs
#pragma unroll
        for (int cc = 0; cc < QH; cc += 32) {
          const int c0 = half * QH + cc;
          uint32_t pr[32];
          tmem_ld_32x32b_x32(tmem + lane_base + T_DPT + c0, pr);
          tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 da = *reinterpret_cast<const float4*>(D_t + c0 + 8 * u);
            const float4 db = *reinterpret_cast<const float4*>(D_t + c0 + 8 * u + 4);
            const float dv8[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
              const float2 pp = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[cc / 2 + 4 * u + k / 2]));
              const float2 d = __fmul2_rn(pp, __fadd2_rn(make_float2(__uint_as_float(pr[8 * u + k]),
                                                                     __uint_as_float(pr[8 * u + k + 1])),
                                                         make_float2(dv8[k], dv8[k + 1])));
              dk2[cc / 2 + 4 * u + k / 2] = pack_bf16(d.x, d.y);
            }
            *reinterpret_cast<uint4*>(dst + p_offset(r, c0 + 8 * u)) =
                make_uint4(dk2[cc / 2 + 4 * u], dk2[cc / 2 + 4 * u + 1], dk2[cc / 2 + 4 * u + 2], dk2[cc / 2 + 4 * u + 3]);
          }
        }
        // dS^T into the first QH/2 of this half's QH dP^T columns (already in registers)
        if constexpr (QH == 64)
          tmem_st_32x32b_x32(tmem + lane_base + T_DPT + half * QH, dk2);
        else
          tmem_st_32x32b_x16(tmem + lane_base + T_DPT + half * QH, dk2);
        tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        warp_arrive(ds_ready);
      }
      // ---- item epilogue: dK (scaled, inverse RoPE), then dV -> bf16; TMEM is released after
      // the loads so the next item's first dV MMA can start while the stores drain
      bwd_wait(dkv_full, j & 1);
      tc_fence_after();
      {
        const int which = half;  // half 0 drains dK, half 1 dV
        const uint32_t tbase = tmem + lane_base + (which == 0 ? T_DK : T_DV);
        const float f = which == 0 ? scale : 1.f;
        __nv_bfloat16* base = which == 0 ? dk + (size_t)(itm.s0 + kvpos) * lddk : dv + (size_t)(itm.s0 + kvpos) * lddv;
        uint4* d4 = reinterpret_cast<uint4*>(base + itm.hk * DH);
        // DH/64 passes over the rotate-half column pairs (c, c + DH/2), 32 columns each side, so
        // only 64 accumulator registers are live (head_dim 128 would otherwise spill)
#pragma unroll
        for (int cp = 0; cp < DH / 64; ++cp) {
          uint32_t lo[32], hi[32];
          tmem_ld_32x32b_x32(tbase + 32 * cp, lo);
          tmem_ld_32x32b_x32(tbase + DH / 2 + 32 * cp, hi);
          tmem_ld_wait();
          if (cp == DH / 64 - 1) {
            tc_fence_before();
            warp_arrive(dkv_empty);
          }
          if (kvpos < itm.L) {
            if (which == 0 && rope_cs != nullptr) {
              // K was rotated by RoPE in the forward: dK_pre = R(pos)^T dK  (rotate by -theta)
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const float2 cs = rope_cs_at(rope_cs, kvpos, 32 * cp + k, DH / 2);
                const float a = __uint_as_float(lo[k]), b = __uint_as_float(hi[k]);
                lo[k] = __float_as_uint(a * cs.x + b * cs.y);
                hi[k] = __float_as_uint(b * cs.x - a * cs.y);
              }
            }
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const uint32_t* acc = h2 == 0 ? lo : hi;
              const int c0 = h2 * (DH / 2) + 32 * cp;  // first column of this 32-column chunk
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint32_t* x = acc + 8 * u;
                d4[c0 / 8 + u] = make_uint4(pack_bf16(__uint_as_float(x[0]) * f, __uint_as_float(x[1]) * f),
                                            pack_bf16(__uint_as_float(x[2]) * f, __uint_as_float(x[3]) * f),
                                            pack_bf16(__uint_as_float(x[4]) * f, __uint_as_float(x[5]) * f),
                                            pack_bf16(__uint_as_float(x[6]) * f, __uint_as_float(x[7]) * f));
              }
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// D[h][t] = sum_d dO[t,h,d] * O[t,h,d]; zero the fp32 dQ accumulator row.  One warp per (t, h).
template <int DH>
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ o, int ldo, const __nv_bfloat16* __restrict__ dout,
                                    int lddo, float* __restrict__ Dvec, float* __restrict__ dq_acc, int T, int H) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= T * H) return;
  const int t = w / H, h = w - t * H;
  float v = 0.f;
#pragma unroll
  for (int c = 0; c < DH / 64; ++c) {
    const __nv_bfloat162 a = reinterpret_cast<const __nv_bfloat162*>(o + (size_t)t * ldo + h * DH + 64 * c)[lane];
    const __nv_bfloat162 b = reinterpret_cast<const __nv_bfloat162*>(dout + (size_t)t * lddo + h * DH + 64 * c)[lane];
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    v += fa.x * fb.x + fa.y * fb.y;
    reinterpret_cast<float2*>(dq_acc + ((size_t)t * H + h) * DH + 64 * c)[lane] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  if (lane == 0) Dvec[(size_t)h * T + t] = v;
}

// dq[t, h, :] (bf16, pitched) = scale * dq_acc[t, h, :], then the inverse RoPE rotation at
// the token's sequence position (cs == null: no rotation; rotate-half pairs (k, k + DH/2)).
// Thread per (t, h, group of 8 rotation pairs).
template <int DH>
__global__ void attn_bwd_post_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dq, int lddq, int T,
                                     int H, float scale, const int32_t* __restrict__ pos,
                                     const float2* __restrict__ cs) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  constexpr int GROUPS = DH / 16;  // groups of 8 pairs per head
  const long long n = (long long)T * H * GROUPS;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long th = i / GROUPS;
    const int g = (int)(i % GROUPS);
    const long long t = th / H;
    const int h = (int)(th - t * H);
    const float* src = dq_acc + th * DH + 8 * g;
    float a[8], b[8];
    *reinterpret_cast<float4*>(a) = reinterpret_cast<const float4*>(src)[0];
    *reinterpret_cast<float4*>(a + 4) = reinterpret_cast<const float4*>(src)[1];
    *reinterpret_cast<float4*>(b) = reinterpret_cast<const float4*>(src + DH / 2)[0];
    *reinterpret_cast<float4*>(b + 4) = reinterpret_cast<const float4*>(src + DH / 2)[1];
    if (cs != nullptr) {
      const int pt = pos[t];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 v = rope_cs_at(cs, pt, 8 * g + k, DH / 2);
        const float x = a[k], y = b[k];
        a[k] = x * v.x + y * v.y;
        b[k] = y * v.x - x * v.y;
      }
    }
    uint4 va, vb;
    va.x = pack_bf16(a[0] * scale, a[1] * scale);
    va.y = pack_bf16(a[2] * scale, a[3] * scale);
    va.z = pack_bf16(a[4] * scale, a[5] * scale);
    va.w = pack_bf16(a[6] * scale, a[7] * scale);
    vb.x = pack_bf16(b[0] * scale, b[1] * scale);
    vb.y = pack_bf16(b[2] * scale, b[3] * scale);
    vb.z = pack_bf16(b[4] * scale, b[5] * scale);
    vb.w = pack_bf16(b[6] * scale, b[7] * scale);
    __nv_bfloat16* d = dq + t * lddq + h * DH + 8 * g;
    *reinterpret_cast<uint4*>(d) = va;
    *reinterpret_cast<uint4*>(d + DH / 2) = vb;
  }
}

// KV-tile list for the backward, lightest-first inversion of the query list: causal work of
// a KV tile shrinks with kv0, so ascending kv0 puts the heaviest tiles first.
__global__ void attn_kv_tiles_kernel(const int32_t* __restrict__ cu, int nseq, int2* __restrict__ tiles,
                                     int* __restrict__ count) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  __shared__ int s_max, s_n;
  if (threadIdx.x == 0) {
    s_max = 0;
    s_n = 0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nseq; j += blockDim.x) atomicMax(&s_max, (cu[j + 1] - cu[j] + BKV - 1) / BKV);
  __syncthreads();
  for (int kb = 0; kb < s_max; ++kb) {
    for (int j0 = 0; j0 < nseq; j0 += blockDim.x) {
      const int j = j0 + threadIdx.x;
      const bool has = j < nseq && (cu[j + 1] - cu[j] + BKV - 1) / BKV > kb;
      const unsigned bal = __ballot_sync(kFull, has);
      int base = 0;
      if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(&s_n, __popc(bal));
      base = __shfl_sync(kFull, base, 0);
      if (has) tiles[base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = make_int2(j, kb * BKV);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = s_n;
}

}  // namespace
}  // namespace mb

using namespace mb;

// Workspace for the tile list: (ceil(T/128) + nseq) int2 + one int.
MAESTRO_API int64_t maestro_attn_workspace(int32_t T, int32_t nseq) {
  return (int64_t)sizeof(int2) * ((T + BQ - 1) / BQ + nseq) + 16;
}

// q [T, H, 64] (row pitch ldq elements), k/v [T, Hk, 64] (pitch ldk/ldv), cu [nseq+1];
// out [T, H, 64] (pitch ldo), lse [H, T] fp32 (natural log-sum-exp of the scaled scores).
// Plan = [query-tile list | count] [KV-tile list | count] [256-row query-tile list | count], each
// maestro_attn_workspace bytes (the last one for the ping-pong forward).
MAESTRO_API int64_t maestro_attn_plan_size(int32_t T, int32_t nseq) { return 3 * maestro_attn_workspace(T, nseq); }

MAESTRO_API int maestro_attn_plan(const int32_t* cu, int32_t nseq, int32_t T, void* plan, void* stream) {
  if (T <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int max_tiles = (T + BQ - 1) / BQ + nseq;
  int2* fw = reinterpret_cast<int2*>(plan);
  int2* bw = reinterpret_cast<int2*>(reinterpret_cast<unsigned char*>(plan) + maestro_attn_workspace(T, nseq));
  launch_pdl(attn_tiles_kernel<>, dim3(1), dim3(1024), 0, st, cu, nseq, fw, reinterpret_cast<int*>(fw + max_tiles));
  launch_pdl(attn_kv_tiles_kernel, dim3(1), dim3(1024), 0, st, cu, nseq, bw, reinterpret_cast<int*>(bw + max_tiles));
  int2* pw = reinterpret_cast<int2*>(reinterpret_cast<unsigned char*>(plan) + 2 * maestro_attn_workspace(T, nseq));
  launch_pdl(attn_tiles_kernel<2 * BQ>, dim3(1), dim3(1024), 0, st, cu, nseq, pw, reinterpret_cast<int*>(pw + max_tiles));
  return launch_status();
}

MAESTRO_API int maestro_attn_fwd(const void* q, const void* k, const void* v, const int32_t* cu, int32_t nseq,
                                 int32_t T, int32_t H, int32_t Hk, int32_t head_dim, int32_t ldq, int32_t ldk,
                                 int32_t ldv, void* out, int32_t ldo, float* lse, float softmax_scale, int32_t causal,
                                 const void* plan, void* workspace, void* stream) {
  if (T <= 0) return 0;
  if ((head_dim != 64 && head_dim != 128) || H % Hk) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  const int max_tiles = (T + BQ - 1) / BQ + nseq;
  int2* tiles = reinterpret_cast<int2*>(plan != nullptr ? const_cast<void*>(plan) : workspace);
  int* count = reinterpret_cast<int*>(tiles + max_tiles);
  // forward variant: "pp" = ping-pong Q-tile pairs, "dec" = decoupled column groups, "base"
  // Default by shape (scripts/attn_quick.py A/B on one B200, r02_attn_fwd_variants.jsonl): head_dim 64
  // -> decoupled groups (+3 % over the shared tile at the KD / cfg 5 student shapes); head_dim 128
  // bidirectional -> ping-pong (+17 % at the cfg 3 ViT shape); head_dim 128 causal -> shared tile
  // (ping-pong +2 % at 8k, -5 % at 4k).
  static const int env_variant = [] {
    const char* e = getenv("MAESTRO_ATTN_FWD");
    if (!e) return ATTN_FWD_VARIANT;
    if (e[0] == 'd') return e[3] == '4' ? 3 : 1;  // "dec" / "dec4"
    return e[0] == 'p' ? 2 : (e[0] == 'b' ? 0 : ATTN_FWD_VARIANT);
  }();
  // causal head_dim 128: ping-pong for long sequences (cfg 5 teacher, 8k: +2 %), shared tile below
  // (cfg 3 backbone, 4k: ping-pong -5 %)
  const bool long_seq = nseq > 0 && T / nseq >= 6144;
  const int variant = env_variant >= 0 ? env_variant : (head_dim == 64 ? 1 : ((causal && !long_seq) ? 0 : 2));
  if (variant == 2) {  // 256-row items: the plan's third list, or built into the workspace
    int2* t2 = plan != nullptr ? reinterpret_cast<int2*>(reinterpret_cast<unsigned char*>(const_cast<void*>(plan)) +
                                                         2 * maestro_attn_workspace(T, nseq))
                               : reinterpret_cast<int2*>(workspace);
    int* c2 = reinterpret_cast<int*>(t2 + max_tiles);
    if (plan == nullptr) launch_pdl(attn_tiles_kernel<2 * BQ>, dim3(1), dim3(1024), 0, st, cu, nseq, t2, c2);
    CUtensorMap mq, mk, mv;
    bool ok = make_map_2d(&mq, q, (uint64_t)H * head_dim, T, ldq, 64, 128);
    ok = ok && make_map_2d(&mk, k, (uint64_t)Hk * head_dim, T, ldk, 64, 128);
    ok = ok && make_map_2d(&mv, v, (uint64_t)Hk * head_dim, T, ldv, 64, 128);
    if (!ok) return (int)cudaErrorInvalidValue;
    const int items = ((T + 2 * BQ - 1) / (2 * BQ) + nseq) * H;
    dim3 grid(items < num_sms() ? items : num_sms());
    const float scale2 = softmax_scale * LOG2E_F;
#define MB_ATTN_PP(D, CZ)                                                                                   \
  {                                                                                                         \
    const int smem = FwdPPCfg<D>::TOTAL + 1024;                                                             \
    if (ensure_smem<attn_fwd_pp_kernel<D, CZ>>(smem)) return launch_status();                               \
    launch_pdl(attn_fwd_pp_kernel<D, CZ>, dim3(grid), dim3(FwdPPCfg<D>::THREADS), smem, st, mq, mk, mv, cu, t2, c2,              \
                                                                         (__nv_bfloat16*)out, ldo, lse, T, H, \
                                                                         Hk, scale2);                        \
  }
    if (head_dim == 64) {
      if (causal) MB_ATTN_PP(64, true) else MB_ATTN_PP(64, false)
    } else {
      if (causal) MB_ATTN_PP(128, true) else MB_ATTN_PP(128, false)
    }
#undef MB_ATTN_PP
    return launch_status();
  }
  if (plan == nullptr) launch_pdl(attn_tiles_kernel<>, dim3(1), dim3(1024), 0, st, cu, nseq, tiles, count);
  CUtensorMap mq, mk, mv;
  bool ok = make_map_2d(&mq, q, (uint64_t)H * head_dim, T, ldq, 64, 128);
  ok = ok && make_map_2d(&mk, k, (uint64_t)Hk * head_dim, T, ldk, 64, 128);
  ok = ok && make_map_2d(&mv, v, (uint64_t)Hk * head_dim, T, ldv, 64, 128);
  if (!ok) return (int)cudaErrorInvalidValue;
  const int items = max_tiles * H;  // upper bound; the kernel reads the true count
  dim3 grid(items < num_sms() ? items : num_sms());
  const float scale2 = softmax_scale * LOG2E_F;
#define MB_ATTN_FWD(D, G, CZ)                                                                             \
  {                                                                                                       \
    using CF = FwdCfg<D, G>;                                                                              \
    const int smem = CF::TOTAL + 1024;                                                                    \
    if (ensure_smem<attn_fwd_kernel<D, G, CZ>>(smem)) return launch_status();                             \
    launch_pdl(attn_fwd_kernel<D, G, CZ>, dim3(grid), dim3(CF::THREADS), smem, st, mq, mk, mv, cu, tiles, count,               \
                                                              (__nv_bfloat16*)out, ldo, lse, T, H, Hk, scale2,   \
                                                              stagger);                                         \
  }
  static const int stagger = [] {
    const char* e = getenv("MAESTRO_ATTN_STAGGER_NS");
    return e ? atoi(e) : 0;
  }();
  static const int dec_stagger = [] {  // group 1's late start in the decoupled forward
    const char* e = getenv("MAESTRO_ATTN_DEC_STAGGER_NS");
    return e ? atoi(e) : 400;
  }();
  // column groups per tile (head_dim 64): 4 (16 softmax warps) or 2 (8); MAESTRO_ATTN_CG overrides
  static const int cg_env = [] {
    const char* e = getenv("MAESTRO_ATTN_CG");
    return e ? atoi(e) : 0;
  }();
  const int cg = cg_env == 2 || cg_env == 4 ? cg_env : ATTN_FWD_CG64;
  if (variant == 1 || (variant == 3 && head_dim == 64)) {
#define MB_ATTN_DEC(D, CZ, NGR)                                                                              \
  {                                                                                                          \
    using CF = FwdDecCfg<D, NGR>;                                                                            \
    const int smem = CF::TOTAL + 1024;                                                                       \
    if (ensure_smem<attn_fwd_dec_kernel<D, CZ, NGR>>(smem)) return launch_status();                          \
    launch_pdl(attn_fwd_dec_kernel<D, CZ, NGR>, dim3(grid), dim3(CF::THREADS), smem, st, mq, mk, mv, cu, tiles, count,            \
                                                                      (__nv_bfloat16*)out, ldo, lse, T, H,     \
                                                                      Hk, scale2, dec_stagger);              \
  }
    if (variant == 3) {  // four 32-column groups: four softmax warps per SM sub-partition
      if (causal) MB_ATTN_DEC(64, true, 4) else MB_ATTN_DEC(64, false, 4)
    } else if (head_dim == 64) {
      if (causal) MB_ATTN_DEC(64, true, 2) else MB_ATTN_DEC(64, false, 2)
    } else {
      if (causal) MB_ATTN_DEC(128, true, 2) else MB_ATTN_DEC(128, false, 2)
    }
#undef MB_ATTN_DEC
    return launch_status();
  }
  if (head_dim == 64 && cg == 4) {
    if (causal) MB_ATTN_FWD(64, 4, true) else MB_ATTN_FWD(64, 4, false)
  } else if (head_dim == 64) {
    if (causal) MB_ATTN_FWD(64, 2, true) else MB_ATTN_FWD(64, 2, false)
  } else {
    if (causal) MB_ATTN_FWD(128, 2, true) else MB_ATTN_FWD(128, 2, false)
  }
#undef MB_ATTN_FWD
  return launch_status();
}

// Backward workspace: tile list + D [H, T] fp32 + dQ accumulator [T, H, head_dim] fp32.
MAESTRO_API int64_t maestro_attn_bwd_workspace(int32_t T, int32_t nseq, int32_t H, int32_t head_dim) {
  return maestro_attn_workspace(T, nseq) + 256 + (int64_t)4 * H * T + (int64_t)4 * T * H * head_dim + 256;
}

MAESTRO_API int maestro_attn_bwd(const void* dout, int32_t lddo, const void* q, const void* k, const void* v,
                                 const void* o, int32_t ldo, const float* lse, const int32_t* cu, int32_t nseq,
                                 int32_t T, int32_t H, int32_t Hk, int32_t head_dim, int32_t ldq, int32_t ldk,
                                 int32_t ldv, void* dq, int32_t lddq, void* dk, int32_t lddk, void* dv, int32_t lddv,
                                 float softmax_scale, int32_t causal, const int32_t* rope_pos, const void* rope_cs,
                                 const void* plan, void* workspace, void* stream) {
  if (T <= 0) return 0;
  if ((head_dim != 64 && head_dim != 128) || H % Hk) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char* w = reinterpret_cast<unsigned char*>(workspace);
  const int max_tiles = (T + BKV - 1) / BKV + nseq;
  int2* tiles = plan != nullptr
                    ? reinterpret_cast<int2*>(const_cast<unsigned char*>(reinterpret_cast<const unsigned char*>(plan)) +
                                              maestro_attn_workspace(T, nseq))
                    : reinterpret_cast<int2*>(w);
  int* count = reinterpret_cast<int*>(tiles + max_tiles);
  const size_t off_d = ((size_t)maestro_attn_workspace(T, nseq) + 255) / 256 * 256;
  float* Dvec = reinterpret_cast<float*>(w + off_d);
  const size_t off_acc = (off_d + (size_t)4 * H * T + 255) / 256 * 256;
  float* dq_acc = reinterpret_cast<float*>(w + off_acc);
  if (plan == nullptr) launch_pdl(attn_kv_tiles_kernel, dim3(1), dim3(1024), 0, st, cu, nseq, tiles, count);
  const long long warps = (long long)T * H;
  const unsigned pre_grid = (unsigned)((warps * 32 + 255) / 256);
  if (head_dim == 64)
    launch_pdl(attn_bwd_pre_kernel<64>, dim3(pre_grid), dim3(256), 0, st, (const __nv_bfloat16*)o, ldo, (const __nv_bfloat16*)dout, lddo,
                                                     Dvec, dq_acc, T, H);
  else
    launch_pdl(attn_bwd_pre_kernel<128>, dim3(pre_grid), dim3(256), 0, st, (const __nv_bfloat16*)o, ldo, (const __nv_bfloat16*)dout, lddo,
                                                      Dvec, dq_acc, T, H);
  const int bqb = head_dim == 64 ? 128 : 64;
  CUtensorMap mq, mk, mv, mdo, mdq;
  bool ok = make_map_2d(&mq, q, (uint64_t)H * head_dim, T, ldq, 64, bqb);
  ok = ok && make_map_2d(&mk, k, (uint64_t)Hk * head_dim, T, ldk, 64, 128);
  ok = ok && make_map_2d(&mv, v, (uint64_t)Hk * head_dim, T, ldv, 64, 128);
  ok = ok && make_map_2d(&mdo, dout, (uint64_t)H * head_dim, T, lddo, 64, bqb);
  // dQ accumulator boxes: 32 fp32 columns x (32 query rows | 64 query rows)
  ok = ok && make_map_2d(&mdq, dq_acc, (uint64_t)H * head_dim, T, (uint64_t)H * head_dim, 32, head_dim == 64 ? 32 : 64,
                         CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4);
  if (!ok) return (int)cudaErrorInvalidValue;
  const int items = max_tiles * Hk;  // upper bound; the kernel reads the true count
  dim3 grid(items < num_sms() ? items : num_sms());
  const float scale2 = softmax_scale * LOG2E_F;
#define MB_ATTN_BWD(D, CZ)                                                                                  \
  {                                                                                                         \
    const int smem = BwdCfg<D>::TOTAL + 1024;                                                               \
    if (ensure_smem<attn_bwd_kernel<D, CZ>>(smem)) return launch_status();                                  \
    launch_pdl(attn_bwd_kernel<D, CZ>, dim3(grid), dim3(BWD_THREADS), smem, st, mq, mk, mv, mdo, mdq, cu, tiles, count, lse, Dvec, \
                                                           (__nv_bfloat16*)dk, lddk, (__nv_bfloat16*)dv, lddv, T, \
                                                           H, Hk, scale2, softmax_scale, (const float2*)rope_cs); \
  }
  if (head_dim == 64) {
    if (causal) MB_ATTN_BWD(64, true) else MB_ATTN_BWD(64, false)
  } else {
    if (causal) MB_ATTN_BWD(128, true) else MB_ATTN_BWD(128, false)
  }
#undef MB_ATTN_BWD
  const long long ng = (long long)T * H * (head_dim / 16);
  const unsigned post_grid = (unsigned)((ng + 255) / 256 < 148 * 16 ? (ng + 255) / 256 : 148 * 16);
  if (head_dim == 64)
    launch_pdl(attn_bwd_post_kernel<64>, dim3(post_grid), dim3(256), 0, st, dq_acc, (__nv_bfloat16*)dq, lddq, T, H, softmax_scale, rope_pos,
                                                       (const float2*)rope_cs);
  else
    launch_pdl(attn_bwd_post_kernel<128>, dim3(post_grid), dim3(256), 0, st, dq_acc, (__nv_bfloat16*)dq, lddq, T, H, softmax_scale,
                                                        rope_pos, (const float2*)rope_cs);
  return launch_status();
}
