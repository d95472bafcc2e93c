// K7: persistent warp-specialised tcgen05 GEMM for the dense section compute.
//
//   C[m, n] (+)= sum_k A(m, k) * B(n, k)      bf16 operands, fp32 accumulation in TMEM
//
// A and B are each K-major (row-major [rows][K]) or MN-major ([K][rows]), which covers the
// three training GEMMs without transposes:  fwd  Y = X W^T      (A K-major,  B K-major)
//                                            dgrad dX = dY W     (A K-major,  B MN-major)
//                                            wgrad dW = dY^T X   (A MN-major, B MN-major)
// A cluster of two CTAs (cta_group::2) computes a 256 x BN tile, BN in {256, 192, 128} picked
// per shape from the per-pair cost ceil(tiles / 74) x tile cost; each CTA TMA-loads its 128 rows
// of A and BN/2 rows of B into a 6-8-stage SWIZZLE_128B ring, one elected thread of the leader
// issues tcgen05.mma (M=256, N=BN, K=16) into a double-buffered TMEM accumulator, and four
// epilogue warps per CTA drain TMEM (tcgen05.ld) while the next tile's MMAs run.  The grid is
// min(work units, SM budget); tiles are visited in grouped-M raster order for L2 reuse.  Epilogues:
// bf16 through swizzled smem staging + TMA store, with fused RoPE / SwiGLU / residual add; fp32
// store or accumulate; split-K (weight gradients whose tile count cannot fill the pairs) with
// red.global.add.v4.f32.
//
// Warp roles (192 threads per CTA): w0 TMA producer, w1 MMA issuer + TMEM owner, w2..w5 epilogue.
#include <cuda_bf16.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace mb {
namespace {

using namespace sm100;

constexpr int BM = 128, BK = 64;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int GROUP_M = 8;
constexpr int THREADS = 192;

enum Epi { EPI_BF16 = 0, EPI_F32 = 1, EPI_F32_ACC = 2, EPI_F32_ATOMIC = 3 };


struct TileSched {
  int num_m, num_n;
  __device__ __forceinline__ void coords(int t, int& m, int& n) const {
    const int per_group = GROUP_M * num_n;
    const int g = t / per_group;
    const int first_m = g * GROUP_M;
    const int gsize = min(GROUP_M, num_m - first_m);
    const int r = t - g * per_group;
    m = first_m + r % gsize;
    n = r / gsize;
  }
};

// CTA-pair variant (cta_group::2): a cluster of 2 CTAs computes a 256 x BN2 tile.  Each CTA
// TMA-loads its 128 rows of A and BN2/2 rows of B; completion of both halves is counted on the
// leader's mbarrier; the leader alone issues tcgen05.mma (M=256, N=BN2), whose accumulator
// rows 0-127 land in the leader's TMEM and 128-255 in the peer's.  Commits are multicast to
// both CTAs (smem slot free / accumulator ready); both epilogues drain their own TMEM and
// arrive on the leader's TMEM-empty barrier.  Per SM this halves B traffic and smem operand
// bandwidth relative to the 1-CTA 128 x 256 tile.
template <int BN2>
struct Cfg2 {
  static constexpr int B_ROWS = BN2 / 2;  // B rows per CTA
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN2 == 128 ? 8 : 6;
  static constexpr int EPI_BUF = 128 * 64 * 2;  // one 128 x 64 bf16 SWIZZLE_128B staging tile
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * EPI_BUF + 1024 + 256;
};

template <int BN2, bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_r, void* C, int M,
                 int N, int K, int ldc, int splits,
                 const int32_t* __restrict__ rope_pos, const float2* __restrict__ rope_cs, int rope_cols, int rope_hd,
                 __nv_bfloat16* __restrict__ swiglu_out, int ld_swiglu, const __nv_bfloat16* __restrict__ resid,
                 int ldr, int l2hint) {
  using CF = Cfg2<BN2>;
  constexpr int STAGES = CF::STAGES, B_BYTES = CF::B_BYTES, STAGE_BYTES = CF::STAGE_BYTES, B_ROWS = CF::B_ROWS;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = align_smem_1024(smem_raw);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * A_BYTES;
  unsigned char* sC = smem + STAGES * STAGE_BYTES;  // 2 x 16 KB epilogue staging (bf16 path)
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + 2 * CF::EPI_BUF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // [2] residual chunk landed in staging buffer b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const TileSched sched{(M + 255) / 256, (N + BN2 - 1) / BN2};
  const int num_units = sched.num_m * sched.num_n * splits;
  const int kb_total = (K + BK - 1) / BK;
  const int kb_per = (kb_total + splits - 1) / splits;
  auto unit = [&](int u, int& mb_, int& nb_, int& kb0, int& kb1) {
    sched.coords(u / splits, mb_, nb_);
    const int ks = u % splits;
    kb0 = ks * kb_per;
    kb1 = min(kb_total, kb0 + kb_per);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 256);
      mbar_init(&rbar[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above overlapped the previous kernel's tail; every
  // global access below waits for it.  The next GEMM may start its own prologue once all of this
  // grid's CTAs are running.
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      // l2hint: B (swept once per grouped-M band, re-read by every band) is kept in L2
      const uint64_t pol_b = l2_policy_evict_last();
      for (int t = pair; t < num_units; t += npairs) {
        int mb_, nb_, kb0, kb1;
        unit(t, mb_, nb_, kb0, kb1);
        const int m0 = mb_ * 256 + (int)rank * 128, n0 = nb_ * BN2 + (int)rank * B_ROWS;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * STAGE_BYTES);
          const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
          const int k0 = kb * BK;
          unsigned char* a = sA + s * A_BYTES;
          unsigned char* b = sB + s * B_BYTES;
          if (!A_MN) {
            tma_load_2d_2sm(a, &map_a, fb, k0, m0);
          } else {
            tma_load_2d_2sm(a, &map_a, fb, m0, k0);
            tma_load_2d_2sm(a + 8192, &map_a, fb, m0 + 64, k0);
          }
          if (!B_MN) {
            if (l2hint)
              tma_load_2d_2sm_hint(b, &map_b, fb, k0, n0, pol_b);
            else
              tma_load_2d_2sm(b, &map_b, fb, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < B_ROWS / 64; ++j) tma_load_2d_2sm(b + 8192 * j, &map_b, fb, n0 + 64 * j, k0);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN2, A_MN, B_MN);
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int t = pair; t < num_units; t += npairs, ++local) {
        int mb_, nb_, kb0, kb1;
        unit(t, mb_, nb_, kb0, kb1);
        const int as = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&tempty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + as * BN2;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? smem_desc_sw128(a_base + k * 2048, 8192, 1024)
                                     : smem_desc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(b_base + k * 2048, 8192, 1024)
                                     : smem_desc_sw128(b_base + k * 32, 16, 1024);
            umma_bf16_2sm(d, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit_2sm(&empty[s], 0x3);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit_2sm(&tfull[as], 0x3);
      }
    }
  } else {
    const int q = warp & 3;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const int et = threadIdx.x - 64;  // 0..127 over the four epilogue warps
    int local = 0, chunk_ctr = 0;
    for (int t = pair; t < num_units; t += npairs, ++local) {
      int mb_, nb_, kb0, kb1;
      unit(t, mb_, nb_, kb0, kb1);
      const int as = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&tfull[as], aph);
      tc_fence_after();
      const int row0 = mb_ * 256 + (int)rank * 128;
      const int row = row0 + q * 32 + lane;
      const int n0 = nb_ * BN2;
      if (EPI == EPI_BF16) {
        // TMEM -> regs -> bf16 -> swizzled smem tile (128 rows x 64 cols) -> TMA bulk store;
        // two staging buffers alternate, the store of one overlaps filling the other.
        const int r_in = q * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < BN2; c += 64, ++chunk_ctr) {
          unsigned char* buf = sC + (chunk_ctr & 1) * CF::EPI_BUF;
          uint32_t r0[32], r1[32];
          const bool use_r = resid != nullptr;
          if (use_r) {
            // fused residual add (h = x + A B^T): the residual chunk is TMA-loaded into this
            // chunk's staging buffer (same swizzled 128 x 64 layout the store uses) while the
            // accumulator is read from TMEM; each thread then adds its row in place
            if (chunk_ctr >= 2) {
              if (et == 0) bulk_wait_read<1>();  // the store issued from this buffer has read it
              named_barrier_sync(1, 128);
            }
            if (et == 0) {
              mbar_arrive_expect_tx(&rbar[chunk_ctr & 1], CF::EPI_BUF);
              tma_load_2d(buf, &map_r, &rbar[chunk_ctr & 1], n0 + c, row0);
            }
          }
          tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + as * BN2 + c, r0);
          tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + as * BN2 + c + 32, r1);
          tmem_ld_wait();
          if (use_r) {
            mbar_wait(&rbar[chunk_ctr & 1], (chunk_ctr >> 1) & 1);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              uint32_t* dst = u < 4 ? &r0[8 * u] : &r1[8 * (u - 4)];
              const uint4 rv = *reinterpret_cast<const uint4*>(buf + r_in * 128 + ((u ^ (r_in & 7)) << 4));
              const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(hv[e]);
                dst[2 * e] = __float_as_uint(__uint_as_float(dst[2 * e]) + f.x);
                dst[2 * e + 1] = __float_as_uint(__uint_as_float(dst[2 * e + 1]) + f.y);
              }
            }
          }
          if (rope_cols > 0 && n0 + c < rope_cols) {  // warp-uniform: the tcgen05.ld below is .sync.aligned
            const int pr = row < M ? rope_pos[row] : 0;  // rows past M are computed but never stored
            if (rope_hd == 64) {
              // fused RoPE (rotate-half): this 64-column chunk is exactly one head of Q or K;
              // r0 holds dims [0,32), r1 dims [32,64) of the row
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const float2 cs = rope_cs_at(rope_cs, pr, k, 32);
                const float a = __uint_as_float(r0[k]), b = __uint_as_float(r1[k]);
                r0[k] = __float_as_uint(a * cs.x - b * cs.y);
                r1[k] = __float_as_uint(b * cs.x + a * cs.y);
              }
            } else {
              // 128-wide heads (heads start at multiples of 128 and BN2 is 128 or 256, so both halves
              // of a head sit in this tile): this chunk is dims [0,64) or [64,128) of a head; the
              // rotate-half partner is the other chunk, read from TMEM alongside
              const bool first = ((n0 + c) & 64) == 0;
              const int pc = first ? c + 64 : c - 64;
              uint32_t p0[32], p1[32];
              tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + as * BN2 + pc, p0);
              tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + as * BN2 + pc + 32, p1);
              tmem_ld_wait();
              const float sg = first ? -1.f : 1.f;  // first half: x cos - x' sin; second: x cos + x' sin
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const float2 c0 = rope_cs_at(rope_cs, pr, k, 64), c1 = rope_cs_at(rope_cs, pr, k + 32, 64);
                r0[k] = __float_as_uint(__uint_as_float(r0[k]) * c0.x + sg * __uint_as_float(p0[k]) * c0.y);
                r1[k] = __float_as_uint(__uint_as_float(r1[k]) * c1.x + sg * __uint_as_float(p1[k]) * c1.y);
              }
            }
          }
          if (swiglu_out != nullptr && row < M && n0 + c < N) {
            // fused SwiGLU: gate/up rows are interleaved in 32-row blocks, so this chunk holds
            // gate (r0) and up (r1) of the same 32 features: s = silu(g) * u
            uint32_t sv[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const float g0 = __uint_as_float(r0[2 * k]), g1 = __uint_as_float(r0[2 * k + 1]);
              const float u0 = __uint_as_float(r1[2 * k]), u1 = __uint_as_float(r1[2 * k + 1]);
              sv[k] = pack_bf16(__fdividef(g0, 1.f + __expf(-g0)) * u0, __fdividef(g1, 1.f + __expf(-g1)) * u1);
            }
            uint4* dst = reinterpret_cast<uint4*>(swiglu_out + (size_t)row * ld_swiglu + (n0 + c) / 2);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint4 val = make_uint4(sv[4 * k], sv[4 * k + 1], sv[4 * k + 2], sv[4 * k + 3]);
              if (l2hint)
                __stcs(dst + k, val);  // streaming store: evict-first in L2
              else
                dst[k] = val;
            }
          }
          if (C == nullptr) continue;  // SwiGLU-only output (forward-only sections): gu is not stored
          if (!use_r && chunk_ctr >= 2) {
            if (et == 0) bulk_wait_read<1>();  // the store issued from this buffer has read it
            named_barrier_sync(1, 128);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t* src = u < 4 ? &r0[8 * u] : &r1[8 * (u - 4)];
            uint4 v;
            v.x = pack_bf16(__uint_as_float(src[0]), __uint_as_float(src[1]));
            v.y = pack_bf16(__uint_as_float(src[2]), __uint_as_float(src[3]));
            v.z = pack_bf16(__uint_as_float(src[4]), __uint_as_float(src[5]));
            v.w = pack_bf16(__uint_as_float(src[6]), __uint_as_float(src[7]));
            *reinterpret_cast<uint4*>(buf + r_in * 128 + ((u ^ (r_in & 7)) << 4)) = v;
          }
          fence_proxy_async_smem();
          named_barrier_sync(1, 128);
          if (et == 0) {
            if (n0 + c < N && row0 < M) {
              if (l2hint)
                tma_store_2d_hint(&map_c, buf, n0 + c, row0, l2_policy_evict_first());
              else
                tma_store_2d(&map_c, buf, n0 + c, row0);
            }
            bulk_commit();  // one group per chunk, even when empty: the wait_read<1> above counts chunks
          }
        }
      } else {
        // fp32 outputs: TMEM -> swizzled smem box (128 rows x 32 fp32, SWIZZLE_128B) -> one TMA op
        // per chunk: a bulk store (EPI_F32) or an L2 reduce-add (EPI_F32_ACC: C += tile;
        // EPI_F32_ATOMIC: split-K slices adding into C).  Full-line transactions instead of a
        // 16-byte segment per row per instruction; the map clips rows/columns past M/N.
        const int r_in = q * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < BN2; c += 32, ++chunk_ctr) {
          unsigned char* buf = sC + (chunk_ctr & 1) * CF::EPI_BUF;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + as * BN2 + c, r);
          tmem_ld_wait();
          if (chunk_ctr >= 2) {
            if (et == 0) bulk_wait_read<1>();  // the op issued from this buffer has read it
            named_barrier_sync(1, 128);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(buf + r_in * 128 + ((j ^ (r_in & 7)) << 4)) =
                make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
          fence_proxy_async_smem();
          named_barrier_sync(1, 128);
          if (et == 0) {
            if (n0 + c < N && row0 < M) {
              if (EPI == EPI_F32)
                tma_store_2d(&map_c, buf, n0 + c, row0);
              else
                tma_reduce_add_2d(&map_c, buf, n0 + c, row0);
            }
            bulk_commit();  // one group per chunk, even when empty: the wait_read<1> above counts chunks
          }
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(tempty_leader0 + (uint32_t)(as * sizeof(uint64_t)));
    }
    if (et == 0) bulk_wait<0>();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, 512);
  }
}

template <int BN2, bool A_MN, bool B_MN, int EPI>
int launch2(const CUtensorMap& ma, const CUtensorMap& mbm, const CUtensorMap& mc, const CUtensorMap& mr, void* C,
            int M, int N, int K,
            int ldc, int splits, cudaStream_t st, const int32_t* rope_pos = nullptr, const float2* rope_cs = nullptr,
            int rope_cols = 0, int rope_hd = 64, __nv_bfloat16* swiglu_out = nullptr, int ld_swiglu = 0,
            const __nv_bfloat16* resid = nullptr, int ldr = 0) {
  constexpr int SMEM = Cfg2<BN2>::SMEM;
  if (ensure_smem<gemm2_kernel<BN2, A_MN, B_MN, EPI>>(SMEM)) return launch_status();
  const int units = ((M + 255) / 256) * ((N + BN2 - 1) / BN2) * splits;
  const int pairs = units < num_sms() / 2 ? units : num_sms() / 2;
  // L2 hints (weights evict-last, outputs evict-first); MAESTRO_GEMM_L2HINT=0 disables
  static const int l2hint = [] {
    const char* e = getenv("MAESTRO_GEMM_L2HINT");
    return e ? atoi(e) : 1;
  }();
  // launched with programmatic stream serialization (MAESTRO_PDL=0 disables)
  launch_pdl(gemm2_kernel<BN2, A_MN, B_MN, EPI>, dim3(2 * pairs), dim3(THREADS), SMEM, st, ma, mbm, mc, mr, C, M, N, K,
             ldc, splits, rope_pos, rope_cs, rope_cols, rope_hd, swiglu_out, ld_swiglu, resid, ldr, l2hint);
  return launch_status();
}

}  // namespace
}  // namespace mb

using namespace mb;

// C[m, n] (+)= sum_k A(m,k) B(n,k).  A(m,k) = A[m*lda + k] (a_mn=0) or A[k*lda + m] (a_mn=1);
// likewise B.  epi: 0 = store bf16, 1 = store fp32, 2 = accumulate into fp32 C.
static int gemm_impl(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t lda,
                     int32_t ldb, int32_t ldc, int32_t a_mn, int32_t b_mn, int32_t epi, void* stream,
                     const int32_t* rope_pos, const float2* rope_cs, int rope_cols, void* swiglu_out = nullptr,
                     int ld_swiglu = 0, const void* resid = nullptr, int ldr = 0, int rope_hd = 64);

MAESTRO_API int maestro_gemm_bf16(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                                  int32_t lda, int32_t ldb, int32_t ldc, int32_t a_mn, int32_t b_mn, int32_t epi,
                                  void* stream) {
  return gemm_impl(A, B, C, M, N, K, lda, ldb, ldc, a_mn, b_mn, epi, stream, nullptr, nullptr, 0);
}

// Forward projection with RoPE fused into the epilogue: C = A B^T (bf16), then every
// head_dim-column head (64 or 128) in columns [0, rope_cols) is rotated (rotate-half) at
// position pos[row]; cos_sin is the position-tiled (cos, sin) table of head_dim/2 frequencies.
// Replaces the separate RoPE pass on the fused QKV output.
MAESTRO_API int maestro_gemm_bf16_rope(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                                       int32_t lda, int32_t ldb, int32_t ldc, const int32_t* pos,
                                       const void* cos_sin, int32_t rope_cols, int32_t head_dim, void* stream) {
  if ((head_dim != 64 && head_dim != 128) || rope_cols % head_dim) return (int)cudaErrorInvalidValue;
  return gemm_impl(A, B, C, M, N, K, lda, ldb, ldc, 0, 0, 0, stream, pos, (const float2*)cos_sin, rope_cols,
                   nullptr, 0, nullptr, 0, head_dim);
}

// Gate/up projection with SwiGLU fused into the epilogue: C = A B^T is the interleaved [g|u]
// activation (gate/up rows of B interleaved in 32-row blocks), S[m, f] = silu(g) * u.
// Output projection with the residual add fused into the epilogue: C = R + A B^T (bf16, fp32
// sum rounded once).  Produces the block's residual stream h directly, so the following norm
// reads h instead of re-reading x and the projection output.
MAESTRO_API int maestro_gemm_bf16_residual(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                                           int32_t lda, int32_t ldb, int32_t ldc, const void* R, int32_t ldr,
                                           void* stream) {
  if (R == nullptr || (ldr % 8)) return (int)cudaErrorInvalidValue;
  return gemm_impl(A, B, C, M, N, K, lda, ldb, ldc, 0, 0, 0, stream, nullptr, nullptr, 0, nullptr, 0, R, ldr);
}

MAESTRO_API int maestro_gemm_bf16_swiglu(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                                         int32_t lda, int32_t ldb, int32_t ldc, void* S, int32_t lds, void* stream) {
  if (N % 64 || S == nullptr) return (int)cudaErrorInvalidValue;
  return gemm_impl(A, B, C, M, N, K, lda, ldb, C ? ldc : N, 0, 0, 0, stream, nullptr, nullptr, 0, S, lds);
}

static int gemm_impl(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t lda,
                     int32_t ldb, int32_t ldc, int32_t a_mn, int32_t b_mn, int32_t epi, void* stream,
                     const int32_t* rope_pos, const float2* rope_cs, int rope_cols, void* swiglu_out,
                     int ld_swiglu, const void* resid, int ldr, int rope_hd) {
  if (M <= 0 || N <= 0 || K <= 0) return (int)cudaErrorInvalidValue;
  if ((lda % 8) || (ldb % 8) || (N % 8) || (ldc % 8)) return (int)cudaErrorInvalidValue;
  const int sms = num_sms();
  cudaStream_t st = (cudaStream_t)stream;
  // CTA-pair path: 256 x BN2 tiles over sms/2 clusters, BN2 in {256, 128} by quantisation;
  // accumulate-into-fp32 GEMMs that cannot fill the pairs split K.
  {
    const int pairs = sms / 2;
    const long long tm = (M + 255) / 256;
    const long long t256 = tm * ((N + 255) / 256), t128 = tm * ((N + 127) / 128);
    const long long c256 = (t256 + pairs - 1) / pairs * 2, c128 = (t128 + pairs - 1) / pairs;
    // per-pair work: ceil(tiles / pairs) * tile cost; a 256x128 tile costs ~0.6 of a 256x256 tile
    // (measured on the step shapes: more operand traffic and epilogue per FLOP), not 0.5
    // (c256 counts 256-wide tiles twice); only short-K, epilogue-bound shapes gain from 128
    int bn2 = (K <= 1024 && 6 * c128 < 5 * c256) ? 128 : 256;
    if (!b_mn) {
      // 256 x 192 tiles (K-major B only: 96 rows per CTA is not a whole SWIZZLE_128B MN atom)
      // fix the quantisation of 768-wide outputs (96 -> 128 tiles on 74 pairs: 2 rounds of 0.75)
      const long long t192 = tm * ((N + 191) / 192);
      const long long c192 = (t192 + pairs - 1) / pairs;  // x 0.8 of a 256-wide tile
      const long long cur = bn2 == 256 ? 10 * c256 / 2 : 6 * c128;  // in tenths of a 256 tile
      // (not with 128-wide RoPE heads: both halves of a head must sit in one tile)
      if (8 * c192 < cur && !(rope_cols > 0 && rope_hd == 128)) bn2 = 192;
    }
    if (const char* e = getenv("MAESTRO_GEMM_BN")) {  // experiments
      const int v = atoi(e);
      bn2 = v == 128 ? 128 : (v == 192 && !b_mn && !(rope_cols > 0 && rope_hd == 128)) ? 192 : 256;
    }
    int splits = 1;
    const int kb = (K + BK - 1) / BK;
    if (epi == EPI_F32_ACC && t256 < pairs && kb >= 8) {
      // split K to fill the pairs; per-pair cost = ceil(tiles*s/pairs) * (k-blocks per slice +
      // epilogue), where a slice's epilogue (a 256x256 fp32 tile reduce-added into C by TMA)
      // costs ~2 k-blocks of MMA and the unsplit one ~1
      bn2 = 256;
      long long best = -1;
      for (int sp = 1; sp <= kb / 2; ++sp) {
        const long long waves = (t256 * sp + pairs - 1) / pairs;
        const long long cost = waves * ((kb + sp - 1) / sp + (sp > 1 ? 2 : 1));
        if (best < 0 || cost < best) {
          best = cost;
          splits = sp;
        }
      }
      const int per = (kb + splits - 1) / splits;
      splits = (kb + per - 1) / per;
    }
    const int epi_k = splits > 1 ? EPI_F32_ATOMIC : epi;
    CUtensorMap ma, mbm, mc, mr;
    const int brows = bn2 / 2;
    memset(&mc, 0, sizeof(mc));
    memset(&mr, 0, sizeof(mr));
    if (resid != nullptr && (epi_k != EPI_BF16 || !make_map_2d(&mr, resid, N, M, ldr, 64, 128)))
      return (int)cudaErrorInvalidValue;
    if (epi_k == EPI_BF16 && C != nullptr && !make_map_2d(&mc, C, N, M, ldc, 64, 128))
      return (int)cudaErrorInvalidValue;
    if (epi_k != EPI_BF16 && !make_map_2d(&mc, C, N, M, ldc, 32, 128, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4))
      return (int)cudaErrorInvalidValue;
    if (C == nullptr && swiglu_out == nullptr) return (int)cudaErrorInvalidValue;
    bool ok = a_mn ? make_map_2d(&ma, A, M, K, lda, 64, 64) : make_map_2d(&ma, A, K, M, lda, 64, 128);
    ok = ok && (b_mn ? make_map_2d(&mbm, B, N, K, ldb, 64, 64) : make_map_2d(&mbm, B, K, N, ldb, 64, brows));
    if (!ok) return (int)cudaErrorInvalidValue;
#define MB_GEMM2_LAUNCH(W, AM, BMN, E)                                                                  \
  launch2<W, AM, BMN, E>(ma, mbm, mc, mr, C, M, N, K, ldc, splits, st, rope_pos, rope_cs, rope_cols, rope_hd, \
                         (__nv_bfloat16*)swiglu_out, ld_swiglu, (const __nv_bfloat16*)resid, ldr)
#define MB_GEMM2_CASE(AM, BMN, E)                                                                    \
  if (a_mn == AM && b_mn == BMN && epi_k == E)                                                       \
    return bn2 == 256 ? MB_GEMM2_LAUNCH(256, AM, BMN, E) : MB_GEMM2_LAUNCH(128, AM, BMN, E);
#define MB_GEMM2_CASE_K(AM, E)                                                                      \
  if (a_mn == AM && b_mn == 0 && epi_k == E)                                                        \
    return bn2 == 256 ? MB_GEMM2_LAUNCH(256, AM, 0, E)                                              \
                      : bn2 == 192 ? MB_GEMM2_LAUNCH(192, AM, 0, E) : MB_GEMM2_LAUNCH(128, AM, 0, E);
    MB_GEMM2_CASE_K(0, 0)
    MB_GEMM2_CASE_K(0, 1)
    MB_GEMM2_CASE_K(0, 2)
    MB_GEMM2_CASE(0, 0, 3)
    MB_GEMM2_CASE(0, 1, 3)
    MB_GEMM2_CASE(0, 1, 0)
    MB_GEMM2_CASE(0, 1, 1)
    MB_GEMM2_CASE(0, 1, 2)
    MB_GEMM2_CASE(1, 1, 0)
    MB_GEMM2_CASE(1, 1, 1)
    MB_GEMM2_CASE(1, 1, 2)
    MB_GEMM2_CASE(1, 1, 3)
#undef MB_GEMM2_CASE
#undef MB_GEMM2_CASE_K
#undef MB_GEMM2_LAUNCH
  }
  return (int)cudaErrorInvalidValue;
}
