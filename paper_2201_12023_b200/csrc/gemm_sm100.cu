// Local-shard GEMM of a ParallelAlgorithm (reference sharding.py:255-299): the
// per-device matmul / batched matmul on `local_dims` (sharding.py:90-92).
//
// sm_100a design: persistent warp-specialised kernel, one CTA per SM.
//   warp 0      TMA producer (one elected lane), 128B-swizzled tiles -> smem ring
//   warp 1      TMEM allocator + tcgen05.mma issuer (one lane), fp32 accum in TMEM
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused op -> global
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile t overlap the
// mainloop of tile t+1.  Operands may be K-major or MN-major (transposed views of
// the IR's transpose reshapes are read in place), with up to two batch dims
// (head split/merge reshapes are strided views, read with rank-4 TMA maps).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <mutex>
#include <cstdlib>
#include "common.cuh"
#include "../../include/mp_exec.h"

namespace mp {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kEpiWarps = 8;   // two warps per TMEM lane quarter, each half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

struct GemmParams {
  int M, N, K;
  int nb0, nb1;
  int tiles_m, tiles_n, num_tiles, k_blocks;
  int a_mn, b_mn;
  int a_mn5, b_mn5;   // MN-major operand staged by one 5-D TMA load per k-block
  int m_fast;         // tile raster: M index fastest (else N fastest)
  void* C;
  int64_t ldc, c_bs0, c_bs1;
  int c_f32;
  float alpha, beta;
  int epi;            // 0 none, 1 gelu, 2 +aux, 3 *gelu'(aux), 4 C=pre & aux:=gelu(pre)
  uint16_t* aux;      // bf16 (M x N) with row stride aux_ld (input for 2/3, output for 4)
  int64_t aux_ld, aux_bs0, aux_bs1;
  int n_wide;         // 2-CTA kernel: tiles [0, n_wide) are 256 x BN; the rest are
                      // half-width splits of the last partial wave (wave-quantisation fix)
  int c_red;          // 2-CTA kernel, fp32 C += alpha * acc: the epilogue hands each 32 x 16
                      // block to a TMA bulk reduce-add (L2 does the read-modify-write)
  int aux_tma;        // 2-CTA kernel, epilogues 2/3: the aux block of the next 32-column chunk
                      // is TMA-loaded into the warp's staging buffer ahead of its use
  int aux_db;         // 2-CTA kernel, aux_tma without c_tma: two aux buffers per warp
  int c_tma;          // 2-CTA kernel, bf16 C (and the epilogue-4 aux output): each 32 x 32
                      // chunk is staged in shared memory (64B swizzle) and written by a TMA
                      // tensor store, so C leaves the SM as whole lines, not 16B row pieces
};

// tile t -> (batch, m block, n block); the faster index is the one with fewer
// blocks' worth of reuse to lose (m_fast when N has more tiles than M), so the
// tiles in flight together share operand blocks in L2
__device__ __forceinline__ void decode1(const GemmParams& p, int t, int tiles_mn, int& b, int& mb,
                                        int& nb) {
  b = t / tiles_mn;
  const int rem = t - b * tiles_mn;
  if (p.m_fast) {
    nb = rem / p.tiles_m;
    mb = rem - nb * p.tiles_m;
  } else {
    mb = rem / p.tiles_n;
    nb = rem - mb * p.tiles_n;
  }
}

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int NACC = 2;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__device__ __forceinline__ void store_chunk(const GemmParams& p, int64_t row_off, int m, int n,
                                            const uint32_t (&r)[32], int b0 = 0, int b1 = 0,
                                            const float* apre = nullptr) {
  // r: 32 consecutive fp32 accumulator columns [n, n+32) of row m
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
  if (p.epi == 1) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 y = gelu_tanh2(v[i], v[i + 1]);
      v[i] = y.x;
      v[i + 1] = y.y;
    }
  } else if (p.epi >= 2) {
    uint16_t* ax = p.aux + (int64_t)b0 * p.aux_bs0 + (int64_t)b1 * p.aux_bs1 +
                   (int64_t)m * p.aux_ld + n;
    if (p.epi == 4) {      // dual output: aux <- gelu(pre), C <- pre
      if (n + 32 <= p.N) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t w[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 y = gelu_tanh2(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
            w[j] = pack_bf2(y.x, y.y);
          }
          reinterpret_cast<uint4*>(ax)[i] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (n + i < p.N) ax[i] = f2bf(gelu_tanh(v[i]));
      }
    } else {
      float a[32];
      if (apre != nullptr) {
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] = apre[i];
      } else if (n + 32 <= p.N) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 u = reinterpret_cast<const uint4*>(ax)[i];
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            a[8 * i + 2 * j] = bf2f(w[j] & 0xffff);
            a[8 * i + 2 * j + 1] = bf2f(w[j] >> 16);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] = (n + i < p.N) ? bf2f(ax[i]) : 0.f;
      }
      if (p.epi == 2) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += a[i];
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 y = gelu_grad_mul2(v[i], v[i + 1], a[i], a[i + 1]);
          v[i] = y.x;
          v[i + 1] = y.y;
        }
      }
    }
  }
  const bool full = (n + 32 <= p.N);
  if (p.c_f32) {
    float* c = reinterpret_cast<float*>(p.C) + row_off + (int64_t)m * p.ldc + n;
    if (full) {
      float4* c4 = reinterpret_cast<float4*>(c);
      if (p.beta != 0.f) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 o = c4[i];
          v[4 * i + 0] += p.beta * o.x;
          v[4 * i + 1] += p.beta * o.y;
          v[4 * i + 2] += p.beta * o.z;
          v[4 * i + 3] += p.beta * o.w;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        c4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)   // static indices keep v[] in registers
        if (n + i < p.N) c[i] = v[i] + (p.beta != 0.f ? p.beta * c[i] : 0.f);
    }
  } else {
    uint16_t* c = reinterpret_cast<uint16_t*>(p.C) + row_off + (int64_t)m * p.ldc + n;
    if (full) {
      uint4* c4 = reinterpret_cast<uint4*>(c);
      if (p.beta != 0.f) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 o = c4[i];
          uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            v[8 * i + 2 * j] += p.beta * bf2f((uint16_t)(w[j] & 0xffff));
            v[8 * i + 2 * j + 1] += p.beta * bf2f((uint16_t)(w[j] >> 16));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        c4[i] = make_uint4(pack_bf2(v[8 * i + 0], v[8 * i + 1]), pack_bf2(v[8 * i + 2], v[8 * i + 3]),
                           pack_bf2(v[8 * i + 4], v[8 * i + 5]), pack_bf2(v[8 * i + 6], v[8 * i + 7]));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (n + i < p.N) {
          float o = (p.beta != 0.f) ? p.beta * bf2f(c[i]) : 0.f;
          c[i] = f2bf(v[i] + o);
        }
      }
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_mn = p.tiles_m * p.tiles_n;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int b, mb, nb;
        decode1(p, t, tiles_mn, b, mb, nb);
        const int b0 = b / p.nb1, b1 = b - (b / p.nb1) * p.nb1;
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
          const int k0 = kb * BK;
          if (p.a_mn5) {
            tma_load_5d(&tmA, &full[stage], a_dst, 0, k0, m0 / 64, b1, b0);
          } else if (p.a_mn) {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_4d(&tmA, &full[stage], a_dst + i * 8192, m0 + 64 * i, k0, b1, b0);
          } else {
            tma_load_4d(&tmA, &full[stage], a_dst, k0, m0, b1, b0);
          }
          if (p.b_mn5) {
            tma_load_5d(&tmB, &full[stage], b_dst, 0, k0, n0 / 64, b1, b0);
          } else if (p.b_mn) {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_4d(&tmB, &full[stage], b_dst + i * 8192, n0 + 64 * i, k0, b1, b0);
          } else {
            tma_load_4d(&tmB, &full[stage], b_dst, k0, n0, b1, b0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(BM, BN, p.a_mn, p.b_mn);
      // K-major: 8-row groups 1024 B apart, K step of 16 elems = +32 B inside the
      // 128 B swizzle atom.  MN-major: 64-elem MN chunks 8 KB apart (LBO), 8-k-row
      // groups 1024 B apart (SBO), K step of 16 = +2048 B.
      const uint32_t a_lbo = p.a_mn ? 8192u : 16u, b_lbo = p.b_mn ? 8192u : 16u;
      const uint32_t a_kstep = p.a_mn ? 2048u : 32u, b_kstep = p.b_mn ? 2048u : 32u;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_base + kk * a_kstep, a_lbo, 1024u);
            const uint64_t bd = umma_desc_sw128(b_base + kk * b_kstep, b_lbo, 1024u);
            tc_mma_f16(d_tmem, ad, bd, idesc, (kb | kk) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        if (Cfg::NACC == 2) {
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        } else {
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // epilogue warps: TMEM lane quarter is fixed by (warp % 4)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int b, mb, nb;
      decode1(p, t, tiles_mn, b, mb, nb);
      const int b0 = b / p.nb1, b1 = b - (b / p.nb1) * p.nb1;
      const int64_t row_off = (int64_t)b0 * p.c_bs0 + (int64_t)b1 * p.c_bs1;
      const int m = mb * BM + row;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int n = nb * BN + c * 32;
        if (m < p.M && n < p.N) store_chunk<BN>(p, row_off, m, n, r, b0, b1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}


// ---------------------------------------------------------------------------
// 2-CTA variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x BN tile.  Each CTA stages its own 128 rows of A and half (BN/2) of the
// B columns; the leader (rank 0) issues tcgen05.mma.cta_group::2 with M = 256,
// which reads both CTAs' shared memory and writes each CTA's 128 accumulator
// rows into its own TMEM.  Per-CTA smem traffic per MMA drops to (4 + BN/32) KB
// per 128*BN/256 cycles, and the 256-row tiles halve the wave count for the
// N = 2048 projections of the GPT plans.
// BN = 512: 256 x 512 pair tiles, two N = 256 MMAs per k-step into all 512 TMEM
// columns (one accumulator, so the epilogue of a tile is not overlapped with the next
// tile's MMAs) -- 25% fewer operand bytes per MAC than 256 x 256, for the wide GEMMs
// whose per-clock rate the L2 -> SM operand stream sets.
template <int BN>
struct Gemm2Cfg {
  static constexpr int A_BYTES = BM * BK * 2;            // 128 rows of A
  static constexpr int B_BYTES = (BN / 2) * BK * 2;      // half of the B columns
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 512) ? 4 : ((BN == 256) ? 6 : 8);
  static constexpr int NACC = (BN == 512) ? 1 : 2;       // TMEM accumulator buffers
  static constexpr int TMEM_COLS = NACC * BN;
  static constexpr int EPI_STAGE = kEpiWarps * 32 * 16 * 4;   // 32 rows x 16 fp32 per warp
  // [stages][epi staging][C store staging][barriers]; both staging areas 1024B aligned
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 2 * EPI_STAGE + 512;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d_2sm(const void* tmap, uint32_t bar_cluster, void* dst,
                                                int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_2sm(const void* tmap, uint32_t bar_cluster, void* dst,
                                                int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tc_mma_f16_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// smem -> global fp32 add of a {16 cols, 32 rows, 1, 1} box (TMA reduction)
__device__ __forceinline__ void tma_reduce_add_4d(const void* tmap, const void* src, int c0, int c1,
                                                  int c2, int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group"
      " [%0, {%2, %3, %4, %5}], [%1];" ::"l"(tmap),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit_g() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_g() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all_g() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void tma_store_4d(const void* tmap, const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group"
      " [%0, {%2, %3, %4, %5}], [%1];" ::"l"(tmap),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// One 32 x 32 chunk of bf16 output through shared memory: row `lane` of the
// chunk goes to cst (+ gelu(pre) to xst for the dual epilogue 4) in the 64B
// swizzle the store maps use (16B piece j of row r at (j ^ ((r >> 1) & 3)),
// conflict-free for the warp's 16B stores), then one TMA store per buffer.
// The previous chunk's stores must have finished reading the buffers first.
__device__ __forceinline__ void tma_store_chunk(const GemmParams& p, const uint32_t (&r)[32],
                                                const float* apre, uint8_t* cst, uint8_t* xst,
                                                const CUtensorMap* tmC, const CUtensorMap* tmX,
                                                int n, int m0, int b0, int b1) {
  const int lane = threadIdx.x & 31;
  float v[32];
  const uint64_t al = pk2(p.alpha, p.alpha);
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    const float2 y = upk2(mul_x2(pk2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), al));
    v[i] = y.x;
    v[i + 1] = y.y;
  }
  if (p.epi == 1) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 y = gelu_tanh2(v[i], v[i + 1]);
      v[i] = y.x;
      v[i + 1] = y.y;
    }
  } else if (p.epi == 2) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 y = upk2(add_x2(pk2(v[i], v[i + 1]), pk2(apre[i], apre[i + 1])));
      v[i] = y.x;
      v[i + 1] = y.y;
    }
  } else if (p.epi == 3) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 y = gelu_grad_mul2(v[i], v[i + 1], apre[i], apre[i + 1]);
      v[i] = y.x;
      v[i + 1] = y.y;
    }
  }
  if (lane == 0) bulk_wait_read_g();
  __syncwarp();
  const int sw = (lane >> 1) & 3;
  uint4* crow = reinterpret_cast<uint4*>(cst + lane * 64);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    crow[j ^ sw] = make_uint4(pack_bf2(v[8 * j], v[8 * j + 1]), pack_bf2(v[8 * j + 2], v[8 * j + 3]),
                              pack_bf2(v[8 * j + 4], v[8 * j + 5]),
                              pack_bf2(v[8 * j + 6], v[8 * j + 7]));
  if (p.epi == 4) {
    uint4* xrow = reinterpret_cast<uint4*>(xst + lane * 64);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 y = gelu_tanh2(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
        w[e] = pack_bf2(y.x, y.y);
      }
      xrow[j ^ sw] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_4d(tmC, cst, n, m0, b1, b0);
    if (p.epi == 4) tma_store_4d(tmX, xst, n, m0, b1, b0);
    bulk_commit_g();
  }
}

struct Tile2 {
  int b0, b1, mb, n0;
  bool narrow;
};
template <int BN>
__device__ __forceinline__ Tile2 decode2(const GemmParams& p, int t) {
  const int tiles_mn = p.tiles_m * p.tiles_n;
  int w = t, extra = 0;
  bool narrow = false;
  if (t >= p.n_wide) {
    const int u = t - p.n_wide;
    w = p.n_wide + (u >> 1);
    extra = (u & 1) * (BN / 2);
    narrow = true;
  }
  int b, mb, nb;
  decode1(p, w, tiles_mn, b, mb, nb);
  return Tile2{b / p.nb1, b - (b / p.nb1) * p.nb1, mb, nb * BN + extra, narrow};
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmBn,
                         const __grid_constant__ CUtensorMap tmC,
                         const __grid_constant__ CUtensorMap tmX, const GemmParams p) {
  using Cfg = Gemm2Cfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* epi_stage = smem + STAGES * Cfg::STAGE_BYTES;   // c_red / aux staging
  uint8_t* cst_stage = epi_stage + Cfg::EPI_STAGE;          // bf16 C store staging
  uint64_t* full = reinterpret_cast<uint64_t*>(cst_stage + Cfg::EPI_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* aux_bar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // [2 * kEpiWarps]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i) mbar_init(&aux_bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < p.num_tiles; t += npairs) {
        const Tile2 tl = decode2<BN>(p, t);
        const int b0 = tl.b0, b1 = tl.b1;
        const int m0 = tl.mb * 2 * BM + rank * BM;
        const int nw = tl.narrow ? BN / 4 : BN / 2;       // B columns staged by this CTA
        const int n0 = tl.n0 + rank * nw;
        const uint32_t bytes = 2u * (Cfg::A_BYTES + nw * BK * 2);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], bytes);
          uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
          const int k0 = kb * BK;
          if (p.a_mn5) {
            tma_load_5d_2sm(&tmA, fb, a_dst, 0, k0, m0 / 64, b1, b0);
          } else if (p.a_mn) {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_4d_2sm(&tmA, fb, a_dst + i * 8192, m0 + 64 * i, k0, b1, b0);
          } else {
            tma_load_4d_2sm(&tmA, fb, a_dst, k0, m0, b1, b0);
          }
          if (BN == 512) {
            // two N = 256 halves; this CTA stages 128 columns of each
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int nh = tl.n0 + h * 256 + rank * 128;
              uint8_t* bh = b_dst + h * (128 * BK * 2);
              if (p.b_mn5) {
                tma_load_5d_2sm(&tmB, fb, bh, 0, k0, nh / 64, b1, b0);
              } else if (p.b_mn) {
                for (int i = 0; i < 2; ++i)
                  tma_load_4d_2sm(&tmB, fb, bh + i * 8192, nh + 64 * i, k0, b1, b0);
              } else {
                tma_load_4d_2sm(&tmB, fb, bh, k0, nh, b1, b0);
              }
            }
          } else if (p.b_mn5) {
            tma_load_5d_2sm(tl.narrow ? &tmBn : &tmB, fb, b_dst, 0, k0, n0 / 64, b1, b0);
          } else if (p.b_mn) {
            for (int i = 0; i < nw / 64; ++i)
              tma_load_4d_2sm(&tmB, fb, b_dst + i * 8192, n0 + 64 * i, k0, b1, b0);
          } else {
            tma_load_4d_2sm(tl.narrow ? &tmBn : &tmB, fb, b_dst, k0, n0, b1, b0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t idesc_w = umma_idesc_bf16(2 * BM, BN == 512 ? 256 : BN, p.a_mn, p.b_mn);
      const uint32_t idesc_n = umma_idesc_bf16(2 * BM, BN / 2, p.a_mn, p.b_mn);
      const uint32_t a_lbo = p.a_mn ? 8192u : 16u, b_lbo = p.b_mn ? 8192u : 16u;
      const uint32_t a_kstep = p.a_mn ? 2048u : 32u, b_kstep = p.b_mn ? 2048u : 32u;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = pair; t < p.num_tiles; t += npairs) {
        const uint32_t idesc = (t >= p.n_wide) ? idesc_n : idesc_w;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_base + kk * a_kstep, a_lbo, 1024u);
            if (BN == 512) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint64_t bd =
                    umma_desc_sw128(b_base + h * (128 * BK * 2) + kk * b_kstep, b_lbo, 1024u);
                tc_mma_f16_2sm(d_tmem + h * 256, ad, bd, idesc, (kb | kk) != 0);
              }
            } else {
              const uint64_t bd = umma_desc_sw128(b_base + kk * b_kstep, b_lbo, 1024u);
              tc_mma_f16_2sm(d_tmem, ad, bd, idesc, (kb | kk) != 0);
            }
          }
          tc_commit_2sm_mc(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_2sm_mc(&tfull[acc]);
        if (Cfg::NACC == 2) {
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        } else {
          acc_phase ^= 1;
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
    uint32_t aux_phase = 0;   // bit b: phase of the warp's aux buffer b
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = pair; t < p.num_tiles; t += npairs) {
      const Tile2 tl = decode2<BN>(p, t);
      const int b0 = tl.b0, b1 = tl.b1;
      const int64_t row_off = (int64_t)b0 * p.c_bs0 + (int64_t)b1 * p.c_bs1;
      const int m = tl.mb * 2 * BM + rank * BM + row;
      const int width = tl.narrow ? BN / 2 : BN;
      const int c_lo = half * (width / 64), c_hi = (half + 1) * (width / 64);
      uint16_t* ast = reinterpret_cast<uint16_t*>(epi_stage + (warp - 2) * 2048);   // 32 x 32 bf16
      uint8_t* cst = cst_stage + (warp - 2) * 2048;                                 // 32 x 32 bf16
      const bool warp_live = (m - lane) < p.M;
      // aux chunks (64B-swizzled, like the C staging): buffer 0 = ast, buffer 1 = cst when
      // C leaves by direct stores (aux_db), so the loads run two chunks ahead
      uint64_t* abar = aux_bar + 2 * (warp - 2);
      if (p.aux_tma && lane == 0) {        // first chunks' aux, under the mainloop's tail
        mbar_arrive_expect_tx(&abar[0], 2048);
        tma_load_4d(&tmX, &abar[0], reinterpret_cast<uint8_t*>(ast), tl.n0 + c_lo * 32, m - lane, b1, b0);
        if (p.aux_db && c_lo + 1 < c_hi) {
          mbar_arrive_expect_tx(&abar[1], 2048);
          tma_load_4d(&tmX, &abar[1], cst, tl.n0 + (c_lo + 1) * 32, m - lane, b1, b0);
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int n = tl.n0 + c * 32;
        if (p.aux_tma) {
          const int ab = p.aux_db ? ((c - c_lo) & 1) : 0;
          mbar_wait(&abar[ab], (aux_phase >> ab) & 1);
          aux_phase ^= 1u << ab;
          float a[32];
          const uint4* src = reinterpret_cast<const uint4*>((ab ? cst : reinterpret_cast<uint8_t*>(ast)) + lane * 64);
          const int sw = (lane >> 1) & 3;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 u = src[i ^ sw];
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              a[8 * i + 2 * j] = bf2f(w4[j] & 0xffff);
              a[8 * i + 2 * j + 1] = bf2f(w4[j] >> 16);
            }
          }
          __syncwarp();                      // buffer read by every lane: refill it
          const int cn = c + 1 + p.aux_db;
          if (cn < c_hi && lane == 0) {
            mbar_arrive_expect_tx(&abar[ab], 2048);
            tma_load_4d(&tmX, &abar[ab], (ab ? cst : reinterpret_cast<uint8_t*>(ast)), tl.n0 + cn * 32, m - lane, b1, b0);
          }
          if (p.c_tma) {
            if (warp_live && n < p.N)
              tma_store_chunk(p, r, a, cst, nullptr, &tmC, &tmX, n, m - lane, b0, b1);
          } else if (m < p.M && n < p.N) {
            store_chunk<BN>(p, row_off, m, n, r, b0, b1, a);
          }
        } else if (p.c_red) {
          // fp32 C += alpha * acc without reading C: rows of this warp -> staging ->
          // TMA reduce-add (out-of-range rows / columns are clipped by the map)
          float* stg = reinterpret_cast<float*>(epi_stage) + (warp - 2) * 32 * 16;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            if (lane == 0) bulk_wait_read_g();     // the previous box has left the buffer
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<float4*>(stg + lane * 16)[i] =
                  make_float4(__uint_as_float(r[sub * 16 + 4 * i]) * p.alpha,
                              __uint_as_float(r[sub * 16 + 4 * i + 1]) * p.alpha,
                              __uint_as_float(r[sub * 16 + 4 * i + 2]) * p.alpha,
                              __uint_as_float(r[sub * 16 + 4 * i + 3]) * p.alpha);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_4d(&tmC, stg, n + sub * 16, m - lane, b1, b0);
              bulk_commit_g();
            }
          }
        } else if (p.c_tma) {
          if (warp_live && n < p.N)
            tma_store_chunk(p, r, nullptr, cst, reinterpret_cast<uint8_t*>(ast), &tmC, &tmX, n,
                            m - lane, b0, b1);
        } else if (m < p.M && n < p.N) {
          store_chunk<BN>(p, row_off, m, n, r, b0, b1);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      if (Cfg::NACC == 2) {
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      } else {
        acc_phase ^= 1;
      }
    }
    if ((p.c_red || p.c_tma) && lane == 0) bulk_wait_all_g();   // staging reads + C writes done
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// rank-4 map: {contig extent, outer extent, nb1, nb0} with element strides.
static int make_map(CUtensorMap* map, const void* base, int64_t d0, int64_t d1, int64_t s1,
                    int64_t nb1, int64_t bs1, int64_t nb0, int64_t bs0, int box0, int box1) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 1;
  }
  const int64_t eb = 2;
  if (nb1 <= 1) bs1 = s1 * d1;
  if (nb0 <= 1) bs0 = bs1 * (nb1 < 1 ? 1 : nb1);
  cuuint64_t dims[4] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)(nb1 < 1 ? 1 : nb1),
                        (cuuint64_t)(nb0 < 1 ? 1 : nb0)};
  cuuint64_t strides[3] = {(cuuint64_t)(s1 * eb), (cuuint64_t)(bs1 * eb), (cuuint64_t)(bs0 * eb)};
  for (int i = 0; i < 3; ++i) {
    if (strides[i] % 16 != 0 || strides[i] == 0) {
      set_error("gemm operand stride not a multiple of 16 bytes (need 8-element aligned rows)");
      return 2;
    }
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) {
    set_error("gemm operand base pointer not 16-byte aligned");
    return 2;
  }
  cuuint32_t box[4] = {(cuuint32_t)box0, (cuuint32_t)box1, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with code " + std::to_string((int)r));
    return 1;
  }
  return 0;
}

// epilogue-side maps (fp32 C reduce-add target, bf16 aux source): {N, M, nb1, nb0},
// box {box0, 32, 1, 1}, no swizzle
static int make_map_box(CUtensorMap* map, void* base, CUtensorMapDataType dt, int64_t eb,
                        int64_t n, int64_t m, int64_t ldc, int64_t nb1, int64_t bs1, int64_t nb0,
                        int64_t bs0, int box0,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 1;
  }
  if (nb1 <= 1) bs1 = ldc * m;
  if (nb0 <= 1) bs0 = bs1 * (nb1 < 1 ? 1 : nb1);
  cuuint64_t dims[4] = {(cuuint64_t)n, (cuuint64_t)m, (cuuint64_t)(nb1 < 1 ? 1 : nb1),
                        (cuuint64_t)(nb0 < 1 ? 1 : nb0)};
  cuuint64_t strides[3] = {(cuuint64_t)(ldc * eb), (cuuint64_t)(bs1 * eb), (cuuint64_t)(bs0 * eb)};
  for (int i = 0; i < 3; ++i) {
    if (strides[i] % 16 != 0 || strides[i] == 0) {
      set_error("epilogue operand stride not a multiple of 16 bytes");
      return 2;
    }
  }
  cuuint32_t box[4] = {(cuuint32_t)box0, 32, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, dt, 4, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (C) failed with code " + std::to_string((int)r));
    return 1;
  }
  return 0;
}

// rank-5 map of an MN-major operand: {64-element MN chunk, K rows, MN / 64 chunks,
// nb1, nb0}; box {64, box_k, chunks, 1, 1} lands chunk-major in smem (8 KB per
// chunk at BK = 64), the layout the MN-major UMMA descriptor expects.
static int make_map_mn5(CUtensorMap* map, const void* base, int64_t mn, int64_t k, int64_t s1,
                        int64_t nb1, int64_t bs1, int64_t nb0, int64_t bs0, int box_k,
                        int chunks) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 1;
  }
  const int64_t eb = 2;
  if (nb1 <= 1) bs1 = s1 * k;
  if (nb0 <= 1) bs0 = bs1 * (nb1 < 1 ? 1 : nb1);
  cuuint64_t dims[5] = {64, (cuuint64_t)k, (cuuint64_t)(mn / 64), (cuuint64_t)(nb1 < 1 ? 1 : nb1),
                        (cuuint64_t)(nb0 < 1 ? 1 : nb0)};
  cuuint64_t strides[4] = {(cuuint64_t)(s1 * eb), 128, (cuuint64_t)(bs1 * eb),
                           (cuuint64_t)(bs0 * eb)};
  for (int i = 0; i < 4; ++i) {
    if (strides[i] % 16 != 0 || strides[i] == 0) {
      set_error("gemm operand stride not a multiple of 16 bytes (need 8-element aligned rows)");
      return 2;
    }
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) {
    set_error("gemm operand base pointer not 16-byte aligned");
    return 2;
  }
  cuuint32_t box[5] = {64, (cuuint32_t)box_k, (cuuint32_t)chunks, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (5-D) failed with code " + std::to_string((int)r));
    return 1;
  }
  return 0;
}

static bool no_mn5() {
  static const bool v = getenv("MPEXEC_GEMM_NO_MN5") != nullptr;
  return v;
}

static int raster_m_fast(int tiles_m, int tiles_n) {
  static const char* env = getenv("MPEXEC_GEMM_RASTER");
  if (env && env[0] == 'n') return 0;
  if (env && env[0] == 'm') return 1;
  return tiles_n > tiles_m ? 1 : 0;
}

template <int BN>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, GemmParams p,
                       cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return 1;
    }
    configured = true;
  }
  p.tiles_n = (p.N + BN - 1) / BN;
  p.m_fast = raster_m_fast(p.tiles_m, p.tiles_n);
  p.num_tiles = p.tiles_m * p.tiles_n * p.nb0 * p.nb1;
  int grid = p.num_tiles < num_sms() ? p.num_tiles : num_sms();
  gemm_bf16_kernel<BN><<<grid, kThreads, Cfg::SMEM, stream>>>(ma, mb, p);
  return 0;
}


template <int BN>
static int launch_gemm_2sm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mbn,
                           const CUtensorMap& mc, const CUtensorMap& mx, GemmParams p,
                           cudaStream_t stream) {
  using Cfg = Gemm2Cfg<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_2sm_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return 1;
    }
    configured = true;
  }
  p.tiles_m = (p.M + 2 * BM - 1) / (2 * BM);
  p.tiles_n = (p.N + BN - 1) / BN;
  p.m_fast = raster_m_fast(p.tiles_m, p.tiles_n);
  const int wide = p.tiles_m * p.tiles_n * p.nb0 * p.nb1;
  int pairs = num_sms() / 2;
  // Wave quantisation: when the last wave is less than half full, split its
  // tiles into two half-width tiles so it finishes in half the time.
  static const bool no_split = getenv("MPEXEC_GEMM_NO_TAIL_SPLIT") != nullptr;
  const int r = wide % pairs;
  p.n_wide = wide;
  if (!no_split && BN == 256 && wide > pairs && r > 0 && 2 * r <= pairs) p.n_wide = wide - r;
  // (BN = 512 has no half-width tail tiles: it is only chosen when its waves are full)
  p.num_tiles = p.n_wide + 2 * (wide - p.n_wide);
  if (p.num_tiles < pairs) pairs = p.num_tiles;
  gemm_bf16_2sm_kernel<BN><<<2 * pairs, kThreads, Cfg::SMEM, stream>>>(ma, mb, mbn, mc, mx, p);
  return 0;
}


// Force-load this file's kernels (lazy module loading would load a kernel at its
// first launch, which blocks the host while an NCCL kernel spins on the device:
// a deadlock the executor's watchdog could not see).  See mp_preload_kernels.
template <typename F>
static inline int preload_one(F* f) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f)) == cudaSuccess ? 0 : 1;
}
int preload_gemm() {
  return preload_one(gemm_bf16_kernel<64>) | preload_one(gemm_bf16_kernel<128>) |
         preload_one(gemm_bf16_kernel<256>) | preload_one(gemm_bf16_2sm_kernel<128>) |
         preload_one(gemm_bf16_2sm_kernel<256>) | preload_one(gemm_bf16_2sm_kernel<512>);
}
}  // namespace mp

using namespace mp;

extern "C" int mp_gemm_bf16_ex(const void* A, const int64_t* ad, const void* B,
                               const int64_t* bd, void* C, const int64_t* cd, int c_dtype,
                               int64_t nbatch0, int64_t nbatch1, float alpha, float beta,
                               int epilogue, void* aux, const int64_t* aux_desc, void* stream);

extern "C" int mp_gemm_bf16(const void* A, const int64_t* ad, const void* B, const int64_t* bd,
                            void* C, const int64_t* cd, int c_dtype, int64_t nbatch0,
                            int64_t nbatch1, float alpha, float beta, int epilogue,
                            void* stream) {
  return mp_gemm_bf16_ex(A, ad, B, bd, C, cd, c_dtype, nbatch0, nbatch1, alpha, beta, epilogue,
                         nullptr, nullptr, stream);
}

extern "C" int mp_gemm_bf16_ex(const void* A, const int64_t* ad, const void* B,
                               const int64_t* bd, void* C, const int64_t* cd, int c_dtype,
                               int64_t nbatch0, int64_t nbatch1, float alpha, float beta,
                               int epilogue, void* aux, const int64_t* aux_desc, void* stream) {
  clear_error();
  MP_CHECK_ARG(A && B && C && ad && bd && cd, "null argument");
  const int64_t M = ad[0], K = ad[1], N = bd[1];
  MP_CHECK_ARG(bd[0] == K, "A cols != B rows");
  MP_CHECK_ARG(cd[0] == M && cd[1] == N, "C shape mismatch");
  MP_CHECK_ARG(M > 0 && N > 0 && K > 0, "empty gemm");
  MP_CHECK_ARG(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), "gemm dims too large");
  MP_CHECK_ARG(cd[3] == 1, "C must have unit column stride");
  MP_CHECK_ARG(c_dtype == 0 || c_dtype == 1, "c_dtype must be 0 (bf16) or 1 (f32)");
  MP_CHECK_ARG(epilogue >= 0 && epilogue <= 4, "bad epilogue");
  MP_CHECK_ARG(epilogue == 0 || beta == 0.f, "fused epilogues require beta == 0");
  MP_CHECK_ARG(epilogue < 2 || (aux && aux_desc && reinterpret_cast<uintptr_t>(aux) % 16 == 0 &&
                                aux_desc[0] % 8 == 0),
               "epilogues 2-4 need a 16-byte aligned bf16 aux matrix with 8-element rows");
  MP_CHECK_ARG(nbatch0 >= 1 && nbatch1 >= 1, "bad batch extents");
  MP_CHECK_ARG(reinterpret_cast<uintptr_t>(C) % 16 == 0 && cd[2] % (c_dtype ? 4 : 8) == 0,
               "C must be 16-byte aligned with 16-byte aligned rows");
  // the epilogue's 16-byte C / aux accesses start at every batch's base too
  MP_CHECK_ARG((nbatch0 == 1 || cd[4] % (c_dtype ? 4 : 8) == 0) &&
                   (nbatch1 == 1 || cd[5] % (c_dtype ? 4 : 8) == 0),
               "C batch strides must be 16-byte multiples");
  MP_CHECK_ARG(epilogue < 2 || ((nbatch0 == 1 || aux_desc[1] % 8 == 0) &&
                                (nbatch1 == 1 || aux_desc[2] % 8 == 0)),
               "aux batch strides must be 16-byte multiples");

  GemmParams p{};
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.nb0 = (int)nbatch0;
  p.nb1 = (int)nbatch1;
  p.tiles_m = (int)((M + BM - 1) / BM);
  p.k_blocks = (int)((K + BK - 1) / BK);
  p.C = C;
  p.ldc = cd[2];
  p.c_bs0 = cd[4];
  p.c_bs1 = cd[5];
  p.c_f32 = c_dtype;
  p.alpha = alpha;
  p.beta = beta;
  p.epi = epilogue;
  p.aux = reinterpret_cast<uint16_t*>(aux);
  if (epilogue >= 2) {
    p.aux_ld = aux_desc[0];
    p.aux_bs0 = aux_desc[1];
    p.aux_bs1 = aux_desc[2];
  }

  // A (M x K): K-major if col stride 1, else MN-major (row stride 1).
  CUtensorMap ma, mb;
  int rc;
  if (ad[3] == 1) {
    p.a_mn = 0;
    rc = make_map(&ma, A, K, M, ad[2], nbatch1, ad[5], nbatch0, ad[4], BK, BM);
  } else if (ad[2] == 1) {
    p.a_mn = 1;
    p.a_mn5 = (M % 64 == 0 && !no_mn5()) ? 1 : 0;
    rc = p.a_mn5 ? make_map_mn5(&ma, A, M, K, ad[3], nbatch1, ad[5], nbatch0, ad[4], BK, BM / 64)
                 : make_map(&ma, A, M, K, ad[3], nbatch1, ad[5], nbatch0, ad[4], 64, BK);
  } else {
    set_error("mp_gemm_bf16: A needs a unit stride");
    return 2;
  }
  if (rc) return rc;

  // Tile shape: the 2-CTA kernel (256-row pair tiles) whenever M >= 256, with BN
  // chosen to minimise wave-quantisation waste; else the 1-CTA kernel.
  static const bool force_1sm = getenv("MPEXEC_GEMM_1SM") != nullptr;
  const int64_t nb = nbatch0 * nbatch1;
  static const int mode = getenv("MPEXEC_GEMM_2SM_BN") ? atoi(getenv("MPEXEC_GEMM_2SM_BN")) : 256;
  bool two_sm = !force_1sm && M >= 256 && N >= 256;
  int BN;
  (void)nb;
  if (two_sm) {
    BN = mode == 128 ? 128 : 256;
    // 256 x 512 pair tiles on the wide GEMMs when their waves come out (nearly) full
    static const bool bn512 = getenv("MPEXEC_GEMM_BN512") != nullptr &&
                              atoi(getenv("MPEXEC_GEMM_BN512")) != 0;
    if (bn512 && mode != 128 && N % 512 == 0) {
      const int64_t t512 = ((M + 255) / 256) * (N / 512) * nbatch0 * nbatch1;
      const int64_t pairs_n = num_sms() / 2;
      const int64_t waves = (t512 + pairs_n - 1) / pairs_n;
      if (waves >= 4 && t512 * 100 >= waves * pairs_n * 95) BN = 512;
    }
  } else {
    BN = (N > 128) ? 256 : (N > 64 ? 128 : 64);
  }
  const int b_box_n = two_sm ? (BN == 512 ? 128 : BN / 2) : BN;
  CUtensorMap mbn;
  if (bd[3] == 1) {
    p.b_mn = 1;
    p.b_mn5 = (N % 64 == 0 && b_box_n % 64 == 0 && !no_mn5()) ? 1 : 0;
    if (p.b_mn5) {
      rc = make_map_mn5(&mb, B, N, K, bd[2], nbatch1, bd[5], nbatch0, bd[4], BK, b_box_n / 64);
      if (!rc && two_sm && b_box_n >= 128)
        rc = make_map_mn5(&mbn, B, N, K, bd[2], nbatch1, bd[5], nbatch0, bd[4], BK, b_box_n / 128);
      else
        mbn = mb;
    } else {
      rc = make_map(&mb, B, N, K, bd[2], nbatch1, bd[5], nbatch0, bd[4], 64, BK);
      mbn = mb;
    }
  } else if (bd[2] == 1) {
    p.b_mn = 0;
    rc = make_map(&mb, B, K, N, bd[3], nbatch1, bd[5], nbatch0, bd[4], BK, b_box_n);
    if (!rc && two_sm)
      rc = make_map(&mbn, B, K, N, bd[3], nbatch1, bd[5], nbatch0, bd[4], BK, b_box_n / 2);
    else
      mbn = mb;
  } else {
    set_error("mp_gemm_bf16: B needs a unit stride");
    return 2;
  }
  if (rc) return rc;

  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // fp32 C += alpha * A B (the dW accumulations): TMA reduce-add epilogue
  static const bool no_red = getenv("MPEXEC_GEMM_NO_REDUCE_EPI") != nullptr;
  CUtensorMap mc = mb;
  p.c_red = 0;
  if (two_sm && c_dtype == 1 && beta == 1.f && epilogue == 0 && !no_red) {
    rc = make_map_box(&mc, C, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, N, M, cd[2], nbatch1, cd[5],
                      nbatch0, cd[4], 16);
    if (rc) return rc;
    p.c_red = 1;
  }
  // epilogues reading aux (residual add, GeLU'): TMA-staged aux chunks
  static const bool no_aux_tma = getenv("MPEXEC_GEMM_NO_AUX_TMA") != nullptr;
  CUtensorMap mx = mb;
  p.aux_tma = 0;
  if (two_sm && (epilogue == 2 || epilogue == 3) && !no_aux_tma) {
    rc = make_map_box(&mx, aux, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, N, M, aux_desc[0], nbatch1,
                      aux_desc[2], nbatch0, aux_desc[1], 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
    p.aux_tma = 1;
  }
  // bf16 C (+ the dual epilogue's aux output) by TMA stores from swizzled staging;
  // operands whose strides a tensor map cannot describe keep the direct stores
  static const bool no_c_tma = getenv("MPEXEC_GEMM_NO_C_TMA") != nullptr;
  static const bool aux_direct = getenv("MPEXEC_GEMM_AUX_DIRECT") != nullptr;
  p.c_tma = 0;
  // (aux-reading epilogues only unbatched: on the batched MoE expert GEMMs at K = 1024
  // the staged GeLU' path measured 20% slower than direct stores, 616 vs 769 TF/s)
  if (two_sm && c_dtype == 0 && beta == 0.f && !no_c_tma &&
      (epilogue == 0 || epilogue == 1 || epilogue == 4 ||
       (p.aux_tma && nbatch0 * nbatch1 == 1 && !aux_direct))) {
    CUtensorMap mc2, mx2 = mx;
    int rc2 = make_map_box(&mc2, C, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, N, M, cd[2], nbatch1,
                           cd[5], nbatch0, cd[4], 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (!rc2 && epilogue == 4)
      rc2 = make_map_box(&mx2, aux, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, N, M, aux_desc[0],
                         nbatch1, aux_desc[2], nbatch0, aux_desc[1], 32,
                         CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc2 == 0) {
      mc = mc2;
      mx = mx2;
      p.c_tma = 1;
    } else {
      clear_error();
    }
  }
  static const bool no_aux_db = getenv("MPEXEC_GEMM_NO_AUX_DB") != nullptr;
  p.aux_db = (p.aux_tma && !p.c_tma && !no_aux_db) ? 1 : 0;
  if (two_sm)
    rc = (BN == 512) ? launch_gemm_2sm<512>(ma, mb, mbn, mc, mx, p, s)
         : (BN == 256) ? launch_gemm_2sm<256>(ma, mb, mbn, mc, mx, p, s)
                       : launch_gemm_2sm<128>(ma, mb, mbn, mc, mx, p, s);
  else if (BN == 256)
    rc = launch_gemm<256>(ma, mb, p, s);
  else if (BN == 128)
    rc = launch_gemm<128>(ma, mb, p, s);
  else
    rc = launch_gemm<64>(ma, mb, p, s);
  if (rc) return rc;
  MP_CHECK_LAUNCH();
  return 0;
}
