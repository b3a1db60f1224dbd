// Fused attention for stages whose softmax dimension is local (SURVEY §2.1:
// "when specs allow (softmax dim local), fuse scores -> softmax -> ctx into one
// FMHA kernel").  It replaces the IR cluster
//   scores = bmm(q_h, k_h^T) -> probs = softmax(scores / sqrt(d)) -> ctx = bmm(probs, v_h)
// (reference graph.py:297-302) and its structural backward (graph.py:341-361)
// without materialising scores / probs.
//
// Layout: Q, K, V, O, dO, dQ, dK, dV are (T, ld) row-major with head `hh` in
// columns [hh*64, hh*64+64) and batch b in rows [b*s, b*s+s) — exactly the
// (tokens, hidden) tensors of the projection matmuls, so head split / merge
// stay views.  d = 64 (GPT-1.3B), s % 128 == 0.
//
// Forward (persistent: work tiles of 128 queries of one (b, head)):
//   warp 0     TMA: Q once, K/V tiles through a 2-stage ring
//   warp 1     tcgen05.mma: S = Q K^T (TMEM, 128 cols), O += P V (TMEM, 64 cols)
//   warps 2-5  softmax, one thread per query row: online max / sum in the log2
//              domain with lazy O rescaling, P -> smem (128B-swizzled K-major),
//              epilogue O / l -> bf16, LSE -> fp32
// Backward (one CTA per 128-key tile, loop over query tiles, FA2 order):
//   S^T = K Q^T, dP^T = V dO^T (TMEM); P^T = exp(S^T - LSE), dS^T = P^T (dP^T - D)
//   (smem); dV += P^T dO, dK += dS^T Q (TMEM accumulators), dQ_i = dS K (TMEM) ->
//   fp32 atomics.  The same swizzled smem tiles serve as K-major and MN-major
//   operands, so no transposes are materialised.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "common.cuh"
#include "../../include/mp_exec.h"

namespace mp {

constexpr int FA_D = 64;
constexpr int FA_BM = 128;   // query rows per tile
constexpr int FA_BN = 128;   // keys per tile
constexpr int FA_TILE = 128 * 64 * 2;  // 16 KB: 128 rows x 64 bf16, SW128

// tcgen05.ld 32 lanes x 32b x 16 columns
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(const void* tmap, uint64_t* bar, void* dst, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// smem -> global element-wise fp32 add of a 2-D box (TMA reduction, L2 does the adds)
__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, const void* src, int c0,
                                                  int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group"
      " [%0, {%2, %3}], [%1];" ::"l"(tmap), "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Packed fp32 pairs (Blackwell FFMA2 / FADD2) and the 3-input FMNMX3: the
// forward softmax is issue-bound in its 4 softmax warps (not MUFU-bound: moving
// a share of the exponentials to an FMA-pipe polynomial made it slower), so
// the per-element instruction count is what sets its speed.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// Store 8 bf16 (one 16-byte unit) of row r, unit u of a 128B-swizzled chunk
// (explicit st.shared: a generic store would go through the LSU's generic path).
__device__ __forceinline__ void st_sw128(uint8_t* chunk, int r, int u, uint4 v) {
  const uint32_t a = smem_u32(chunk) + r * 128 + ((u ^ (r & 7)) << 4);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// diagnostics: %globaltimer stamp `k` of tile g (query tile in the backward, key tile
// in the forward).  Compiled in only with
// -DMP_FA_TRACE (MPEXEC_NVCC_EXTRA) and written when MPEXEC_FA_BWD_TRACE names a file
__device__ __forceinline__ void fa_stamp(long long* trace, int g, int k) {
#ifdef MP_FA_TRACE
  if (trace && g < 1024) {
    long long ts;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ts));
    trace[((int64_t)blockIdx.x * 1024 + g) * 8 + k] = ts;
  }
#endif
}

struct FaFwdParams {
  int B, H, s, ld;
  int kv0, nkv;      // key range: tiles [kv0/128, kv0/128 + nkv) of every sequence
  float scale_log2;  // log2(e) / sqrt(d)
  uint16_t* O;
  float* lse;        // [B*H, s]
  long long* trace;  // diagnostics (MPEXEC_FA_FWD_TRACE, -DMP_FA_TRACE)
};

// smem: Q 16K | K[2] 32K | V 16K | P 32K | barriers  (97 KB: two CTAs per SM).
// With P in TMEM (PT, the default) the P tiles are not allocated: 65 KB.
constexpr int FA_FWD_SMEM = FA_TILE * 6 + 1024 + 256;
constexpr int FA_FWD_SMEM_PT = FA_TILE * 5 + 1024 + 256;   // PT: V double-buffered

// tcgen05.mma with A read from tensor memory (TS form): P V with P in TMEM
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// tcgen05.ld 32 lanes x 32b x 32 columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  tmem_ld_32x32b_x32(taddr, r);
}

// PT: P (bf16) goes to its own 64 TMEM columns with tcgen05.st and P V reads it from
// there (TS-form MMA) -- no shared-memory P tiles, no st.shared / proxy fence on
// the softmax path, and the P V MMA only streams V from shared memory.
template <bool PT>
__global__ void __launch_bounds__(192, 2)
    fa_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const FaFwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + FA_TILE;          // 2 stages
  uint8_t* sV = smem + 3 * FA_TILE;      // 1 stage (PT: 2, in the smem freed by P)
  uint8_t* sP = smem + 4 * FA_TILE;      // 2 chunks of 64 keys (not PT)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (PT ? 5 : 6) * FA_TILE);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;    // [2]
  uint64_t* k_empty = bars + 3;   // [2]
  uint64_t* v_full = bars + 5;    // [PT: 2] stage 1 at bars + 16
  uint64_t* v_empty = bars + 6;   // [PT: 2] stage 1 at bars + 17
  constexpr int VST = PT ? 2 : 1;
  auto vfull = [&](int st) { return st ? bars + 16 : v_full; };
  auto vempty = [&](int st) { return st ? bars + 17 : v_empty; };
  uint64_t* s_full = bars + 7;
  uint64_t* s_free = bars + 8;
  uint64_t* p_full = bars + 9;     // P keys 0-63 in smem (4 softmax warps)
  uint64_t* o_done = bars + 10;
  uint64_t* p_full1 = bars + 14;   // P keys 64-127 in smem
  uint64_t* p0_free = bars + 15;   // PV has read P keys 0-63 (first four K steps done)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x;                  // query tile
  const int bh = blockIdx.y;
  const int b = bh / p.H, hh = bh - (bh / p.H) * p.H;
  const int n_kv = p.nkv;
  const int row0 = b * p.s;
  const int krow0 = row0 + p.kv0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(vfull(i), 1);
      mbar_init(vempty(i), 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(p_full, 4);
    mbar_init(p_full1, 4);
    mbar_init(p0_free, 1);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128, tP = tmem + 192;   // tP: PT only

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, FA_TILE);
      tma_load_2d(&tmQ, q_full, sQ, hh * FA_D, row0 + qt * FA_BM);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[st], FA_TILE);
        tma_load_2d(&tmK, &k_full[st], sK + st * FA_TILE, hh * FA_D, krow0 + j * FA_BN);
        const int vs = VST == 2 ? (j & 1) : 0;
        const uint32_t vpar = VST == 2 ? (((j >> 1) & 1) ^ 1) : ((j & 1) ^ 1);
        mbar_wait(vempty(vs), vpar);
        mbar_arrive_expect_tx(vfull(vs), FA_TILE);
        tma_load_2d(&tmV, vfull(vs), sV + vs * FA_TILE, hh * FA_D, krow0 + j * FA_BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = umma_idesc_bf16(128, 128, 0, 0);   // Q K-major, K K-major
      const uint32_t id_o = umma_idesc_bf16(128, 64, 0, 1);    // P K-major, V MN-major
      mbar_wait(q_full, 0);
      const uint32_t q_base = smem_u32(sQ), p_base = smem_u32(sP), v_base = smem_u32(sV);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        if (j > 0) mbar_wait(s_free, (j - 1) & 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sK + st * FA_TILE);
#pragma unroll
        for (int kk = 0; kk < FA_D / 16; ++kk)
          tc_mma_f16(tS, umma_desc_sw128(q_base + kk * 32, 16, 1024),
                     umma_desc_sw128(k_base + kk * 32, 16, 1024), id_s, kk > 0);
        tc_commit(s_full);
        tc_commit(&k_empty[st]);
      };
      issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_s(j + 1);
        const int vs = VST == 2 ? (j & 1) : 0;
        mbar_wait(vfull(vs), VST == 2 ? ((j >> 1) & 1) : (j & 1));
        const uint32_t vb = v_base + vs * FA_TILE;
        // O += P V in two halves of 64 keys: the first half starts as soon as the
        // softmax warps have written P's first 64 keys, and its completion
        // (p0_free) lets them write the next tile's first half while the
        // second half still runs
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(h ? p_full1 : p_full, j & 1);
          tc_fence_after();
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = h * 4 + k4;
            const uint64_t bd = umma_desc_sw128(vb + kk * 2048, 8192, 1024);
            if (PT) {
              tc_mma_f16_ts(tO, tP + kk * 8, bd, id_o, (j | kk) != 0);   // 16 keys = 8 columns
            } else {
              const uint64_t ad = umma_desc_sw128(p_base + h * FA_TILE + k4 * 32, 16, 1024);
              tc_mma_f16(tO, ad, bd, id_o, (j | kk) != 0);
            }
          }
          if (h == 0) tc_commit(p0_free);
        }
        tc_commit(vempty(vs));
        tc_commit(o_done);
      }
    }
  } else {
    const int q = warp & 3;
    const int r = q * 32 + lane;                       // query row within the tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    float m_used = -INFINITY;                          // log2-domain running max
    float l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      // The whole S row (128 fp32) moves to registers at once, so S is released
      // before the max: the next S = Q K^T runs under this tile's exp / P pass.
      uint32_t sv[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + lane_off + c * 32, sv[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int e = 0; e < 32; e += 2)
          mx = fmax3(mx, __uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1]));
      mx *= p.scale_log2;
      // lazy rescale: only when the max grows by more than 2^8
      const bool need = (mx > m_used + 8.f);
      float alpha = 1.f;
      if (need) {
        alpha = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx);
        m_used = mx;
      }
      // P must not overwrite smem before PV_{j-1} has consumed it: the first half
      // once PV_{j-1}'s first four K steps are done, the second once all are
      // (a rescale of O needs the whole PV_{j-1} first)
      const bool any_need = __any_sync(0xffffffffu, need);
      if (j > 0) {
        mbar_wait(any_need ? o_done : p0_free, (j - 1) & 1);
        tc_fence_after();
        if (any_need) {
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t o32[32];
            tmem_ld32(tO + lane_off + c * 32, o32);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o32[e] = __float_as_uint(__uint_as_float(o32[e]) * alpha);
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
                    tO + lane_off + c * 32),
                "r"(o32[0]), "r"(o32[1]), "r"(o32[2]), "r"(o32[3]), "r"(o32[4]), "r"(o32[5]),
                "r"(o32[6]), "r"(o32[7]), "r"(o32[8]), "r"(o32[9]), "r"(o32[10]), "r"(o32[11]),
                "r"(o32[12]), "r"(o32[13]), "r"(o32[14]), "r"(o32[15]), "r"(o32[16]),
                "r"(o32[17]), "r"(o32[18]), "r"(o32[19]), "r"(o32[20]), "r"(o32[21]),
                "r"(o32[22]), "r"(o32[23]), "r"(o32[24]), "r"(o32[25]), "r"(o32[26]),
                "r"(o32[27]), "r"(o32[28]), "r"(o32[29]), "r"(o32[30]), "r"(o32[31]));
          }
          tmem_st_wait();
        }
      }
      l *= alpha;
      const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2), nm2 = f2pack(-m_used, -m_used);
      uint64_t sum2 = f2pack(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c == 2) {
          // first 64 keys of P are written: PV's first half may start
          if (PT)
            tmem_st_wait();
          else
            fence_async_smem();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full);
          if (j > 0 && !any_need) {
            mbar_wait(o_done, (j - 1) & 1);
            tc_fence_after();
          }
        }
        const uint32_t(&t32)[32] = sv[c];
        uint8_t* chunk = sP + (c >> 1) * FA_TILE;
        uint32_t pk[16];   // PT: the chunk's 32 keys as 16 packed bf16 pairs
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float pv[8];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            float x0, x1;
            f2unpack(ffma2(f2pack(__uint_as_float(t32[t * 8 + e]),
                                  __uint_as_float(t32[t * 8 + e + 1])), sc2, nm2), x0, x1);
            pv[e] = ex2(x0);
            pv[e + 1] = ex2(x1);
            sum2 = fadd2(sum2, f2pack(pv[e], pv[e + 1]));
          }
          if (PT) {
#pragma unroll
            for (int e = 0; e < 4; ++e) pk[t * 4 + e] = pack_bf2(pv[2 * e], pv[2 * e + 1]);
          } else {
            st_sw128(chunk, r, (c & 1) * 4 + t,
                     make_uint4(pack_bf2(pv[0], pv[1]), pack_bf2(pv[2], pv[3]),
                                pack_bf2(pv[4], pv[5]), pack_bf2(pv[6], pv[7])));
          }
        }
        if (PT) tmem_st16(tP + lane_off + c * 16, pk);
      }
      float s0, s1;
      f2unpack(sum2, s0, s1);
      l += s0 + s1;
      if (PT)
        tmem_st_wait();
      else
        fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full1);
    }
    // epilogue
    mbar_wait(o_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const int grow = row0 + qt * FA_BM + r;
    uint16_t* orow = p.O + (int64_t)grow * p.ld + hh * FA_D;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t o16[16];
      tmem_ld16(tO + lane_off + c * 16, o16);
      tmem_ld_wait();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
      dst[0] = make_uint4(pack_bf2(__uint_as_float(o16[0]) * inv, __uint_as_float(o16[1]) * inv),
                          pack_bf2(__uint_as_float(o16[2]) * inv, __uint_as_float(o16[3]) * inv),
                          pack_bf2(__uint_as_float(o16[4]) * inv, __uint_as_float(o16[5]) * inv),
                          pack_bf2(__uint_as_float(o16[6]) * inv, __uint_as_float(o16[7]) * inv));
      dst[1] = make_uint4(pack_bf2(__uint_as_float(o16[8]) * inv, __uint_as_float(o16[9]) * inv),
                          pack_bf2(__uint_as_float(o16[10]) * inv, __uint_as_float(o16[11]) * inv),
                          pack_bf2(__uint_as_float(o16[12]) * inv, __uint_as_float(o16[13]) * inv),
                          pack_bf2(__uint_as_float(o16[14]) * inv, __uint_as_float(o16[15]) * inv));
    }
    // natural-log LSE of the scaled scores: ln(l) + m_used * ln 2
    p.lse[(int64_t)bh * p.s + qt * FA_BM + r] = logf(l) + m_used * 0.6931471805599453f;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// Persistent forward (P in TMEM): two CTAs per SM walk work tiles w = (bh, query
// tile) with stride gridDim.x.  Barrier phases run on the CTA-global key-tile
// counter J, so the pipeline does not drain between work tiles: Q is
// double-buffered (the next tile's Q lands while this one still streams K/V),
// the next tile's first S = Q K^T is issued as soon as the last S of this tile
// has been read, and the O epilogue (TMEM -> bf16 global) overlaps that S MMA;
// the next tile's first P V (which overwrites O) waits for o_free.
// smem: Q[2] 32K | K[2] 32K | V[2] 32K | barriers (97 KB: two CTAs per SM).
constexpr int FA_FWD_SMEM_PERSIST = FA_TILE * 6 + 1024 + 256;

// 2^x for a pair on the FMA / ALU pipes instead of MUFU (which runs at 16 / clk / SM and
// bounds the forward at d = 64): x = n + f with n = rint(x) via the 1.5 * 2^23 trick,
// 2^f on [-0.5, 0.5] by a degree-3 fit (max relative error 7.8e-5, far below bf16's
// 3.9e-3), and n added straight into the exponent field.  x >= -126 keeps the exponent
// field non-negative (2^-126 is 0 for the softmax either way).
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& y0, float& y1) {
  const uint64_t x = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t t = fadd2(x, f2pack(12582912.f, 12582912.f));
  const uint64_t fr = ffma2(fadd2(t, f2pack(-12582912.f, -12582912.f)), f2pack(-1.f, -1.f), x);
  uint64_t pp = ffma2(f2pack(0.055268411f, 0.055268411f), fr, f2pack(0.24262036f, 0.24262036f));
  pp = ffma2(pp, fr, f2pack(0.69324332f, 0.69324332f));
  pp = ffma2(pp, fr, f2pack(0.99992698f, 0.99992698f));
  float p0, p1, t0, t1;
  f2unpack(pp, p0, p1);
  f2unpack(t, t0, t1);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// EMU: how many of every eight exponent pairs go to exp2_poly2 instead of MUFU
template <int EMU>
__global__ void __launch_bounds__(192, 2)
    fa_fwd_persist_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV, const FaFwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sQ = smem;                    // 2 stages
  uint8_t* sK = smem + 2 * FA_TILE;      // 2 stages
  uint8_t* sV = smem + 4 * FA_TILE;      // 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * FA_TILE);
  uint64_t* q_full = bars;         // [2]
  uint64_t* q_empty = bars + 2;    // [2]
  uint64_t* k_full = bars + 4;     // [2]
  uint64_t* k_empty = bars + 6;    // [2]
  uint64_t* v_full = bars + 8;     // [2]
  uint64_t* v_empty = bars + 10;   // [2]
  uint64_t* s_full = bars + 12;
  uint64_t* s_free = bars + 13;
  uint64_t* p_full = bars + 14;    // P keys 0-63 in TMEM
  uint64_t* p_full1 = bars + 15;   // P keys 64-127
  uint64_t* p0_free = bars + 16;   // P V has read P keys 0-63
  uint64_t* o_done = bars + 17;
  uint64_t* o_free = bars + 18;    // epilogue has read O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = p.s / FA_BM;
  const int n_work = n_qt * p.B * p.H;
  const int n_kv = p.nkv;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(p_full, 4);
    mbar_init(p_full1, 4);
    mbar_init(p0_free, 1);
    mbar_init(o_done, 1);
    mbar_init(o_free, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128, tP = tmem + 192;

  // work tile -> (first row of the sequence, head, query tile); consecutive w share
  // a (b, head) so co-resident CTAs re-read the same K/V from L2
  auto decode = [&](int w, int& row0, int& hh, int& qt, int& bh) {
    bh = w / n_qt;
    qt = w - bh * n_qt;
    const int b = bh / p.H;
    hh = bh - b * p.H;
    row0 = b * p.s;
  };

  if (warp == 0) {
    if (lane == 0) {
      int J = 0, tt = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++tt) {
        int row0, hh, qt, bh;
        decode(w, row0, hh, qt, bh);
        const int qs = tt & 1;
        mbar_wait(&q_empty[qs], ((tt >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qs], FA_TILE);
        tma_load_2d(&tmQ, &q_full[qs], sQ + qs * FA_TILE, hh * FA_D, row0 + qt * FA_BM);
        const int krow0 = row0 + p.kv0;
        for (int j = 0; j < n_kv; ++j, ++J) {
          const int st = J & 1;
          const uint32_t par = ((J >> 1) & 1) ^ 1;
          mbar_wait(&k_empty[st], par);
          mbar_arrive_expect_tx(&k_full[st], FA_TILE);
          tma_load_2d(&tmK, &k_full[st], sK + st * FA_TILE, hh * FA_D, krow0 + j * FA_BN);
          mbar_wait(&v_empty[st], par);
          mbar_arrive_expect_tx(&v_full[st], FA_TILE);
          tma_load_2d(&tmV, &v_full[st], sV + st * FA_TILE, hh * FA_D, krow0 + j * FA_BN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = umma_idesc_bf16(128, 128, 0, 0);   // Q K-major, K K-major
      const uint32_t id_o = umma_idesc_bf16(128, 64, 0, 1);    // P (TMEM), V MN-major
      const uint32_t v_base = smem_u32(sV);
      const int n_tiles = blockIdx.x < n_work ? (n_work - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      // S for global key tile Jn, which is key tile jn of local work tile tn
      auto issue_s = [&](int Jn, int tn, int jn) {
        const int qs = tn & 1;
        if (jn == 0) mbar_wait(&q_full[qs], (tn >> 1) & 1);
        const int st = Jn & 1;
        mbar_wait(&k_full[st], (Jn >> 1) & 1);
        if (Jn > 0) mbar_wait(s_free, (Jn - 1) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ + qs * FA_TILE);
        const uint32_t k_base = smem_u32(sK + st * FA_TILE);
#pragma unroll
        for (int kk = 0; kk < FA_D / 16; ++kk)
          tc_mma_f16(tS, umma_desc_sw128(q_base + kk * 32, 16, 1024),
                     umma_desc_sw128(k_base + kk * 32, 16, 1024), id_s, kk > 0);
        fa_stamp(p.trace, Jn, 7);
        tc_commit(s_full);
        tc_commit(&k_empty[st]);
        if (jn == n_kv - 1) tc_commit(&q_empty[qs]);
      };
      if (n_tiles > 0) issue_s(0, 0, 0);
      int J = 0;
      for (int tt = 0; tt < n_tiles; ++tt) {
        for (int j = 0; j < n_kv; ++j, ++J) {
          if (j + 1 < n_kv)
            issue_s(J + 1, tt, j + 1);
          else if (tt + 1 < n_tiles)
            issue_s(J + 1, tt + 1, 0);
          // the first P V of a tile overwrites O: the previous epilogue must have read it
          if (j == 0 && tt > 0) mbar_wait(o_free, (tt - 1) & 1);
          const int st = J & 1;
          mbar_wait(&v_full[st], (J >> 1) & 1);
          fa_stamp(p.trace, J, 4);
          const uint32_t vb = v_base + st * FA_TILE;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            mbar_wait(h ? p_full1 : p_full, J & 1);
            fa_stamp(p.trace, J, 5 + h);
            tc_fence_after();
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const int kk = h * 4 + k4;
              tc_mma_f16_ts(tO, tP + kk * 8, umma_desc_sw128(vb + kk * 2048, 8192, 1024), id_o,
                            (j | kk) != 0);
            }
            if (h == 0) tc_commit(p0_free);
          }
          tc_commit(&v_empty[st]);
          tc_commit(o_done);
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int r = q * 32 + lane;                       // query row within the tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int J = 0;
    for (int w = blockIdx.x, tt = 0; w < n_work; w += gridDim.x, ++tt) {
      int row0, hh, qt, bh;
      decode(w, row0, hh, qt, bh);
      float m_used = -INFINITY;                        // log2-domain running max
      float l = 0.f;
      for (int j = 0; j < n_kv; ++j, ++J) {
        mbar_wait(s_full, J & 1);
        if (warp == 2 && lane == 0) fa_stamp(p.trace, J, 0);
        tc_fence_after();
        uint32_t sv[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + lane_off + c * 32, sv[c]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            mx = fmax3(mx, __uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1]));
        mx *= p.scale_log2;
        const bool need = (mx > m_used + 8.f);
        float alpha = 1.f;
        if (need) {
          alpha = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx);
          m_used = mx;
        }
        // P (TMEM) must not be overwritten before the previous P V has read it; at
        // j == 0 the previous tile's epilogue already waited for its last P V
        const bool any_need = __any_sync(0xffffffffu, need);
        if (j > 0) {
          mbar_wait(any_need ? o_done : p0_free, (J - 1) & 1);
          tc_fence_after();
          if (any_need) {
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t o16[16];
              tmem_ld16(tO + lane_off + c * 16, o16);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e)
                o16[e] = __float_as_uint(__uint_as_float(o16[e]) * alpha);
              tmem_st16(tO + lane_off + c * 16, o16);
            }
            tmem_st_wait();
          }
        }
        l *= alpha;
        const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2), nm2 = f2pack(-m_used, -m_used);
        uint64_t sum2 = f2pack(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c == 2) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
            if (j > 0 && !any_need) {
              mbar_wait(o_done, (J - 1) & 1);
              tc_fence_after();
            }
          }
          const uint32_t(&t32)[32] = sv[c];
          uint32_t pk[16];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            float pv[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              float x0, x1;
              f2unpack(ffma2(f2pack(__uint_as_float(t32[t * 8 + e]),
                                    __uint_as_float(t32[t * 8 + e + 1])), sc2, nm2), x0, x1);
              if (((t * 4 + e / 2) & 7) < EMU) {
                exp2_poly2(x0, x1, pv[e], pv[e + 1]);
              } else {
                pv[e] = ex2(x0);
                pv[e + 1] = ex2(x1);
              }
              sum2 = fadd2(sum2, f2pack(pv[e], pv[e + 1]));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) pk[t * 4 + e] = pack_bf2(pv[2 * e], pv[2 * e + 1]);
          }
          tmem_st16(tP + lane_off + c * 16, pk);
        }
        float s0, s1;
        f2unpack(sum2, s0, s1);
        l += s0 + s1;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full1);
        if (warp == 2 && lane == 0) fa_stamp(p.trace, J, 1);
      }
      // epilogue: O / l -> bf16, then release O for the next tile's first P V
      mbar_wait(o_done, (J - 1) & 1);
      if (warp == 2 && lane == 0) fa_stamp(p.trace, J - 1, 2);
      tc_fence_after();
      const float inv = 1.f / l;
      uint16_t* orow = p.O + (int64_t)(row0 + qt * FA_BM + r) * p.ld + hh * FA_D;
      uint32_t o16[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(tO + lane_off + c * 16, o16[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          pk[e] = pack_bf2(__uint_as_float(o16[c][2 * e]) * inv,
                           __uint_as_float(o16[c][2 * e + 1]) * inv);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      p.lse[(int64_t)bh * p.s + qt * FA_BM + r] = logf(l) + m_used * 0.6931471805599453f;
      if (warp == 2 && lane == 0) fa_stamp(p.trace, J - 1, 3);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// ------------------------------------------------------------------ backward
struct FaBwdParams {
  int B, H, s, ld;
  int kv0;            // first key of the range covered
  int n_kt;           // key tiles in the range (work tiles = n_kt * B * H)
  float scale;        // 1/sqrt(d)
  const float* lse;   // [B*H, s]
  const float* dvec;  // D = rowsum(dO * O), [B*H, s]
  float* dQacc;       // fp32 (T, ld), zero-initialised
  uint16_t* dK;
  uint16_t* dV;
  long long* trace;   // diagnostics (MPEXEC_FA_BWD_TRACE): globaltimer per query tile
};

// smem: K 16K | V 16K | Q[2] 32K | dO[2] 32K | P^T[2] 64K | dS^T[2] 64K | barriers (224 KB)
// P^T / dS^T are double-buffered so the P/dS math of query tile i overlaps the
// dV / dK / dQ MMAs of tile i-1; LSE / D are read straight from global (L1-broadcast).
// (no alignment slack: the dynamic smem window of a cluster-less CTA is 1 KB
// aligned on sm_100; the kernel checks it and reports instead of corrupting)
constexpr int FA_BWD_SMEM = FA_TILE * 14 + 2048 + 256;
constexpr int FA_BWD_THREADS = 448;   // TMA, MMA, 8 P/dS warps, 4 dQ warps

// Persistent: one CTA per SM walks work tiles w = (bh, key tile) with stride
// gridDim.x.  Every barrier phase runs on the CTA-global query-tile counter g
// (tile t, query tile i: g = t * n_q + i), so the pipeline does not drain
// between work tiles: the next tile's Q/dO loads start as soon as stages free
// up, its K/V as soon as the last MMA of the previous tile has read K/V
// (kv_empty), and the dK/dV epilogue of tile t overlaps the K/V load of t+1
// (the first dV/dK MMA of t+1 waits for acc_free).
// PT: P^T (bf16) goes to TMEM with tcgen05.st and the dV MMA reads it from there (TS
// form), so P^T costs neither shared-memory stores nor shared-memory operand reads
// (the backward is bound by shared-memory bandwidth); the dQ accumulator is
// single-buffered to make room for it.

template <bool PT>
__global__ void __launch_bounds__(FA_BWD_THREADS, 1)
    fa_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                  const __grid_constant__ CUtensorMap tmdQ, const FaBwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023) {   // never observed; poison dQ so parity tests catch it
    if (threadIdx.x == 0) p.dQacc[0] = __int_as_float(0x7fc00000);
    return;
  }
  uint8_t* smem = smem_raw;
  uint8_t* sK = smem;
  uint8_t* sV = smem + FA_TILE;
  uint8_t* sQ = smem + 2 * FA_TILE;    // [2]
  uint8_t* sdO = smem + 4 * FA_TILE;   // [2]
  uint8_t* sPt = smem + 6 * FA_TILE;   // [2] x 2 chunks (queries 0-63 | 64-127)
  uint8_t* sdSt = smem + 10 * FA_TILE; // [2] x 2 chunks
  float* sLse = reinterpret_cast<float*>(smem + 14 * FA_TILE);   // [2][128], log2 domain
  float* sD = sLse + 256;                                        // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 14 * FA_TILE + 2048);
  uint64_t* kv_full = bars;          // K, V of the work tile
  uint64_t* q_full = bars + 1;       // [2] Q_g, dO_g (+ lse / D staged)
  uint64_t* q_empty = bars + 3;      // [2]
  uint64_t* st_full = bars + 5;      // S^T and dP^T of g in TMEM
  uint64_t* ps_full = bars + 6;      // P^T / dS^T of g in smem (8 warps)
  uint64_t* pbuf_free = bars + 7;    // [2] P^T / dS^T buffer free (MMAs and dQ reduction done)
  uint64_t* dq_full = bars + 16;     // [2] dQ of g in TMEM buffer g & 1
  uint64_t* dq_free = bars + 18;     // [2] 4 dQ warps have read the buffer
  uint64_t* acc_done = bars + 11;    // dV / dK of the work tile complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  uint64_t* s_free = bars + 13;      // 8 P/dS warps hold S^T / dP^T of g in registers
  uint64_t* kv_empty = bars + 14;    // last MMA of the work tile has read K / V
  uint64_t* acc_free = bars + 15;    // dK / dV TMEM drained by the epilogue (8 warps)
  uint64_t* pt_free = bars + 20;     // PT: the dV MMAs of g have read P^T(g) from TMEM

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_q = p.s / FA_BM;
  const int n_work = p.n_kt * p.B * p.H;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmdO);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1 + 32);   // tx arrive + 32 lanes staging lse / D
      mbar_init(&q_empty[i], 1);
      mbar_init(&pbuf_free[i], 1);
    }
    mbar_init(st_full, 1);
    mbar_init(ps_full, 8);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dq_full[i], 1);
      mbar_init(&dq_free[i], 4);
    }
    mbar_init(acc_done, 1);
    mbar_init(s_free, 8);
    mbar_init(kv_empty, 1);
    mbar_init(acc_free, 8);
    mbar_init(pt_free, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tSt = tmem, tdPt = tmem + 128, tdV = tmem + 256, tdK = tmem + 320,
                 tdQ = tmem + 384;   // [2] x 64 columns (PT: one buffer)
  const uint32_t tPt = tmem + 448;   // PT: P^T as 64 columns of packed bf16 pairs

  if (warp == 0) {
    // TMA producer (lane 0) + lse / D staging (all lanes; the next query tile's
    // values are prefetched into registers so their latency stays off the chain)
    float nl[4], nd[4];
    auto fetch = [&](int w, int i) {
      const int bh = w / p.n_kt;
      const int64_t base = (int64_t)bh * p.s + i * FA_BM;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        nl[k] = p.lse[base + k * 32 + lane];
        nd[k] = p.dvec[base + k * 32 + lane];
      }
    };
    int g = 0, t = 0;
    if ((int)blockIdx.x < n_work) fetch(blockIdx.x, 0);
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
      const int bh = w / p.n_kt, kt = w - (w / p.n_kt) * p.n_kt;
      const int b = bh / p.H, hh = bh - (bh / p.H) * p.H;
      const int row0 = b * p.s;
      for (int i = 0; i < n_q; ++i, ++g) {
        const int st = g & 1;
        mbar_wait(&q_empty[st], ((g >> 1) & 1) ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&q_full[st], 2 * FA_TILE);
          tma_load_2d(&tmQ, &q_full[st], sQ + st * FA_TILE, hh * FA_D, row0 + i * FA_BM);
          tma_load_2d(&tmdO, &q_full[st], sdO + st * FA_TILE, hh * FA_D, row0 + i * FA_BM);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // staged negated and pre-scaled for the packed P / dS math:
          // -LSE * log2(e) and -D * scale
          sts32(smem_u32(sLse + st * 128 + k * 32 + lane), nl[k] * -1.4426950408889634f);
          sts32(smem_u32(sD + st * 128 + k * 32 + lane), nd[k] * -p.scale);
        }
        mbar_arrive(&q_full[st]);   // release: publishes the lse / D stores
        if (i == 0) {                // K / V of this tile once the previous tile is done with them
          if (t > 0) mbar_wait(kv_empty, (t - 1) & 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, 2 * FA_TILE);
            tma_load_2d(&tmK, kv_full, sK, hh * FA_D, row0 + p.kv0 + kt * FA_BN);
            tma_load_2d(&tmV, kv_full, sV, hh * FA_D, row0 + p.kv0 + kt * FA_BN);
          }
        }
        const int wn = w + (int)gridDim.x;
        if (i + 1 < n_q) fetch(w, i + 1);
        else if (wn < n_work) fetch(wn, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_st = umma_idesc_bf16(128, 128, 0, 0);  // K/V (K-major) x Q/dO (K-major)
      const uint32_t id_acc = umma_idesc_bf16(128, 64, 0, 1);  // P^T/dS^T (K-major) x dO/Q (MN)
      const uint32_t id_dq = umma_idesc_bf16(128, 64, 1, 1);   // dS (MN-major) x K (MN-major)
      const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
      // dV/dK/dQ of query tile j (global gj) of work tile t
      auto issue_acc = [&](int j, int gj, int t) {
        const int bj = gj & 1;
        if (j == 0 && t > 0) {      // the epilogue of work tile t-1 has drained dK / dV
          mbar_wait(acc_free, (t - 1) & 1);
          tc_fence_after();
        }
        fa_stamp(p.trace, gj, 5);
        const uint32_t pt = smem_u32(sPt + bj * 2 * FA_TILE), ds = smem_u32(sdSt + bj * 2 * FA_TILE);
        const uint32_t qb = smem_u32(sQ + bj * FA_TILE), dob = smem_u32(sdO + bj * FA_TILE);
        if (PT) {
          // dV += P^T dO with P^T from TMEM (16 queries = 8 columns per K step)
#pragma unroll
          for (int kk = 0; kk < FA_BM / 16; ++kk)
            tc_mma_f16_ts(tdV, tPt + kk * 8, umma_desc_sw128(dob + kk * 2048, 8192, 1024), id_acc,
                          (j | kk) != 0);
          tc_commit(pt_free);
#pragma unroll
          for (int kk = 0; kk < FA_BM / 16; ++kk) {
            const uint32_t aoff = (kk >> 2) * FA_TILE + (kk & 3) * 32;
            tc_mma_f16(tdK, umma_desc_sw128(ds + aoff, 16, 1024),
                       umma_desc_sw128(qb + kk * 2048, 8192, 1024), id_acc, (j | kk) != 0);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < FA_BM / 16; ++kk) {
            const uint32_t aoff = (kk >> 2) * FA_TILE + (kk & 3) * 32;
            tc_mma_f16(tdV, umma_desc_sw128(pt + aoff, 16, 1024),
                       umma_desc_sw128(dob + kk * 2048, 8192, 1024), id_acc, (j | kk) != 0);
            tc_mma_f16(tdK, umma_desc_sw128(ds + aoff, 16, 1024),
                       umma_desc_sw128(qb + kk * 2048, 8192, 1024), id_acc, (j | kk) != 0);
          }
        }
        tc_commit(&q_empty[bj]);     // Q / dO of gj read: the next load may start
        // the dQ TMEM buffer this MMA writes was last read by the dQ warps for gj-2
        // (two buffers) or gj-1 (PT: one buffer)
        if (PT) {
          if (gj >= 1) mbar_wait(&dq_free[(gj - 1) & 1], ((gj - 1) >> 1) & 1);
        } else if (gj >= 2) {
          mbar_wait(&dq_free[bj], ((gj >> 1) & 1) ^ 1);
        }
        fa_stamp(p.trace, gj, 6);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < FA_BN / 16; ++kk)
          tc_mma_f16(tdQ + (PT ? 0 : bj * 64), umma_desc_sw128(ds + kk * 2048, FA_TILE, 1024),
                     umma_desc_sw128(k_base + kk * 2048, 8192, 1024), id_dq, kk > 0);
        tc_commit(&dq_full[bj]);   // also: dK / dQ MMAs done with dS^T (the dQ warps reuse it)
      };
      int g = 0, t = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
        mbar_wait(kv_full, t & 1);
        for (int i = 0; i < n_q; ++i, ++g) {
          const int st = g & 1;
          mbar_wait(&q_full[st], (g >> 1) & 1);
          if (g > 0) mbar_wait(s_free, (g - 1) & 1);    // S^T/dP^T(g-1) in the P warps' registers
          fa_stamp(p.trace, g, 4);
          tc_fence_after();
          const uint32_t q_base = smem_u32(sQ + st * FA_TILE);
          const uint32_t do_base = smem_u32(sdO + st * FA_TILE);
#pragma unroll
          for (int kk = 0; kk < FA_D / 16; ++kk) {
            tc_mma_f16(tSt, umma_desc_sw128(k_base + kk * 32, 16, 1024),
                       umma_desc_sw128(q_base + kk * 32, 16, 1024), id_st, kk > 0);
            tc_mma_f16(tdPt, umma_desc_sw128(v_base + kk * 32, 16, 1024),
                       umma_desc_sw128(do_base + kk * 32, 16, 1024), id_st, kk > 0);
          }
          tc_commit(st_full);
          if (i > 0) {
            mbar_wait(ps_full, (g - 1) & 1);           // P^T/dS^T(g-1) written
            tc_fence_after();
            issue_acc(i - 1, g - 1, t);
          }
        }
        mbar_wait(ps_full, (g - 1) & 1);
        tc_fence_after();
        issue_acc(n_q - 1, g - 1, t);
        tc_commit(acc_done);
        tc_commit(kv_empty);
      }
    }
  } else if (warp < 10) {
    // 8 P/dS warps: lane quarter q = warp % 4 selects the TMEM lanes (key rows),
    // `half` selects which 64 of the 128 query columns this warp processes.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q * 32 + lane;                        // key row (S^T / dP^T lane)
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float sl2 = p.scale * 1.4426950408889634f;
    const uint64_t sl2_2 = f2pack(sl2, sl2), sc_2 = f2pack(p.scale, p.scale);
    int g = 0, t = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++t) {
      for (int i = 0; i < n_q; ++i, ++g) {
        const int bi = g & 1;
        mbar_wait(&q_full[bi], (g >> 1) & 1);   // lse / D of g staged
        if (warp == 2 && lane == 0) fa_stamp(p.trace, g, 0);
        mbar_wait(st_full, g & 1);
        if (warp == 2 && lane == 0) fa_stamp(p.trace, g, 1);
        tc_fence_after();
        // this P^T / dS^T buffer was last read by the MMAs of g-2
        // (PT: dQ is staged elsewhere, so the dK / dQ MMAs of g-2 are the last readers)
        if (g >= 2) mbar_wait(PT ? &dq_full[bi] : &pbuf_free[bi], ((g >> 1) & 1) ^ 1);
        if (warp == 2 && lane == 0) fa_stamp(p.trace, g, 2);
        uint8_t* pt = sPt + bi * 2 * FA_TILE;
        uint8_t* dst = sdSt + bi * 2 * FA_TILE;

        const uint32_t lse_a = smem_u32(sLse + bi * 128), d_a = smem_u32(sD + bi * 128);
        // 4 chunks of 16 queries, software-pipelined: the TMEM load of chunk
        // cc+1 is in flight while chunk cc is computed; once the last chunk is
        // in registers S^T / dP^T are released (s_free) so the next tile's
        // S^T / dP^T MMAs overlap this tile's tail
        uint32_t sa[16], da[16], sb[16], db[16];
        tmem_ld16(tSt + lane_off + (half * 4) * 16, sa);
        tmem_ld16(tdPt + lane_off + (half * 4) * 16, da);
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c = half * 4 + cc;
          uint32_t(&s16)[16] = (cc & 1) ? sb : sa;
          uint32_t(&d16)[16] = (cc & 1) ? db : da;
          if (cc + 1 < 4) {
            tmem_ld16(tSt + lane_off + (c + 1) * 16, (cc & 1) ? sa : sb);
            tmem_ld16(tdPt + lane_off + (c + 1) * 16, (cc & 1) ? da : db);
          } else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_free);
          }
          float lse2[16], dvv[16];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 a = lds128(lse_a + (c * 16 + k * 4) * 4);
            const float4 bq = lds128(d_a + (c * 16 + k * 4) * 4);
            lse2[4 * k] = a.x; lse2[4 * k + 1] = a.y; lse2[4 * k + 2] = a.z; lse2[4 * k + 3] = a.w;
            dvv[4 * k] = bq.x; dvv[4 * k + 1] = bq.y; dvv[4 * k + 2] = bq.z; dvv[4 * k + 3] = bq.w;
          }
          // P = 2^(S * scale * log2e - LSE * log2e), dS = P * (dP * scale - D * scale)
          // in packed fp32 pairs (scale = 2^-3 at d = 64: bit-identical to the
          // unpacked P * (dP - D) * scale)
          float pv[16], ds[16];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            float x0, x1;
            f2unpack(ffma2(f2pack(__uint_as_float(s16[e]), __uint_as_float(s16[e + 1])), sl2_2,
                           f2pack(lse2[e], lse2[e + 1])), x0, x1);
            pv[e] = ex2(x0);
            pv[e + 1] = ex2(x1);
            f2unpack(fmul2(f2pack(pv[e], pv[e + 1]),
                           ffma2(f2pack(__uint_as_float(d16[e]), __uint_as_float(d16[e + 1])), sc_2,
                                 f2pack(dvv[e], dvv[e + 1]))), ds[e], ds[e + 1]);
          }
          const int ch = c >> 2, u0 = (c & 3) * 2;
          if (PT) {
            // P^T(g) overwrites P^T(g-1) in TMEM once the dV MMAs of g-1 have read it
            if (cc == 0 && g >= 1) {
              mbar_wait(pt_free, (g - 1) & 1);
              tc_fence_after();
            }
            const uint32_t pk[8] = {pack_bf2(pv[0], pv[1]),   pack_bf2(pv[2], pv[3]),
                                    pack_bf2(pv[4], pv[5]),   pack_bf2(pv[6], pv[7]),
                                    pack_bf2(pv[8], pv[9]),   pack_bf2(pv[10], pv[11]),
                                    pack_bf2(pv[12], pv[13]), pack_bf2(pv[14], pv[15])};
            tmem_st8(tPt + lane_off + c * 8, pk);
          } else {
            st_sw128(pt + ch * FA_TILE, r, u0,
                     make_uint4(pack_bf2(pv[0], pv[1]), pack_bf2(pv[2], pv[3]),
                                pack_bf2(pv[4], pv[5]), pack_bf2(pv[6], pv[7])));
            st_sw128(pt + ch * FA_TILE, r, u0 + 1,
                     make_uint4(pack_bf2(pv[8], pv[9]), pack_bf2(pv[10], pv[11]),
                                pack_bf2(pv[12], pv[13]), pack_bf2(pv[14], pv[15])));
          }
          st_sw128(dst + ch * FA_TILE, r, u0,
                   make_uint4(pack_bf2(ds[0], ds[1]), pack_bf2(ds[2], ds[3]), pack_bf2(ds[4], ds[5]),
                              pack_bf2(ds[6], ds[7])));
          st_sw128(dst + ch * FA_TILE, r, u0 + 1,
                   make_uint4(pack_bf2(ds[8], ds[9]), pack_bf2(ds[10], ds[11]),
                              pack_bf2(ds[12], ds[13]), pack_bf2(ds[14], ds[15])));
          if (cc + 1 < 4) tmem_ld_wait();
        }
        if (PT) tmem_st_wait();
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ps_full);
        if (warp == 2 && lane == 0) fa_stamp(p.trace, g, 3);
      }
      // dK (half 0) / dV (half 1) epilogue: key row r
      const int bh = w / p.n_kt, kt = w - (w / p.n_kt) * p.n_kt;
      const int b = bh / p.H, hh = bh - (bh / p.H) * p.H;
      mbar_wait(acc_done, t & 1);
      tc_fence_after();
      const int64_t grow = (int64_t)b * p.s + p.kv0 + kt * FA_BN + r;
      const uint32_t tacc = half ? tdV : tdK;
      uint16_t* out = (half ? p.dV : p.dK) + grow * p.ld + hh * FA_D;
      uint32_t t16[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(tacc + lane_off + c * 16, t16[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_free);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4* dstg = reinterpret_cast<uint4*>(out + c * 16);
        dstg[0] = make_uint4(pack_bf2(__uint_as_float(t16[c][0]), __uint_as_float(t16[c][1])),
                             pack_bf2(__uint_as_float(t16[c][2]), __uint_as_float(t16[c][3])),
                             pack_bf2(__uint_as_float(t16[c][4]), __uint_as_float(t16[c][5])),
                             pack_bf2(__uint_as_float(t16[c][6]), __uint_as_float(t16[c][7])));
        dstg[1] = make_uint4(pack_bf2(__uint_as_float(t16[c][8]), __uint_as_float(t16[c][9])),
                             pack_bf2(__uint_as_float(t16[c][10]), __uint_as_float(t16[c][11])),
                             pack_bf2(__uint_as_float(t16[c][12]), __uint_as_float(t16[c][13])),
                             pack_bf2(__uint_as_float(t16[c][14]), __uint_as_float(t16[c][15])));
      }
    }
  } else {
    // 4 dQ warps: query row r of query tile g.  dQ(g) leaves TMEM into the
    // dS^T buffer of g (free once the dQ MMA has read it) as fp32, 128B-swizzled
    // in two 32-column halves, and is added into dQacc by two TMA bulk
    // reductions; the buffer is handed back to the P warps once TMA has read it.
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool leader = warp == 10 && lane == 0;
    int g = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
      const int bh = w / p.n_kt;
      const int b = bh / p.H, hh = bh - (bh / p.H) * p.H;
      const int row0 = b * p.s;
      for (int i = 0; i < n_q; ++i, ++g) {
        const int bj = g & 1;
        mbar_wait(&dq_full[bj], (g >> 1) & 1);
        if (leader) fa_stamp(p.trace, g, 7);
        tc_fence_after();
        uint32_t t16[4][16];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld16(tdQ + (PT ? 0 : bj * 64) + lane_off + c * 16, t16[c]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dq_free[bj]);
#ifndef MP_FA_NO_DQ_RED
        // PT: dQ is staged in the (otherwise unused) smem P^T buffers, two-deep, so the
        // P warps never wait on the dQ reduction; the leader's wait for the TMA read of
        // the buffer's previous use (wait_group.read 1 at the end of the last
        // iteration) is published to the other dQ warps by this barrier
        if (PT) asm volatile("bar.sync 1, 128;" ::: "memory");
        uint8_t* stage = (PT ? sPt : sdSt) + bj * 2 * FA_TILE;
#pragma unroll
        for (int c = 0; c < 4; ++c) {        // columns 16c .. 16c+15: half c/2, units 4(c&1)..+3
          uint8_t* chunk = stage + (c >> 1) * FA_TILE;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int u = (c & 1) * 4 + e;
            const uint32_t a = smem_u32(chunk) + r * 128 + ((u ^ (r & 7)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                         "r"(t16[c][4 * e]), "r"(t16[c][4 * e + 1]), "r"(t16[c][4 * e + 2]),
                         "r"(t16[c][4 * e + 3])
                         : "memory");
          }
        }
        fence_async_smem();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (leader) {
          tma_reduce_add_2d(&tmdQ, stage, hh * FA_D, row0 + i * FA_BM);
          tma_reduce_add_2d(&tmdQ, stage + FA_TILE, hh * FA_D + 32, row0 + i * FA_BM);
          bulk_commit();
          if (PT) {
            bulk_wait_read1();            // the other staging buffer has been read
          } else {
            bulk_wait_read0();
            mbar_arrive(&pbuf_free[bj]);
          }
        }
#else
        if (leader) mbar_arrive(&pbuf_free[bj]);
#endif
      }
    }
    if (leader) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// D[bh, t] = sum_d dO * O   (warp per row of 64); the same pass zeroes the row's
// dQ accumulator (the backward adds into it with TMA bulk reductions)
__global__ void fa_bwd_pre_kernel(const uint16_t* __restrict__ O, const uint16_t* __restrict__ dO,
                                  float* __restrict__ dvec, float* __restrict__ dq_acc, int B,
                                  int H, int s, int ld) {
  // D[r] = sum_d dO[r,d] * O[r,d] and dQ accumulator zeroing: 8 lanes per row, one
  // 16-byte vector of O and dO per lane (a warp covers 4 rows), 32-bit row math
  const int lane = threadIdx.x & 31, g = lane >> 3, sub = lane & 7;
  const int rows = B * H * s;
  const int warps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int w4 = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); w4 * 4 < rows; w4 += warps) {
    const int r = w4 * 4 + g;
    float acc = 0.f;
    if (r < rows) {
      const int bh = r / s, t = r - bh * s;
      const int b = bh / H, hh = bh - b * H;
      const int64_t off = ((int64_t)b * s + t) * ld + hh * FA_D + sub * 8;
      const uint4 o = __ldg(reinterpret_cast<const uint4*>(O + off));
      const uint4 gg = __ldg(reinterpret_cast<const uint4*>(dO + off));
      float4* dq = reinterpret_cast<float4*>(dq_acc + off);
      dq[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      dq[1] = make_float4(0.f, 0.f, 0.f, 0.f);
      const uint32_t ow[4] = {o.x, o.y, o.z, o.w}, gw[4] = {gg.x, gg.y, gg.z, gg.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        acc += bf2f(ow[j] & 0xffff) * bf2f(gw[j] & 0xffff) + bf2f(ow[j] >> 16) * bf2f(gw[j] >> 16);
    }
#pragma unroll
    for (int k = 4; k; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
    if (sub == 0 && r < rows) dvec[r] = acc;
  }
}

// Key-split attention (keys sharded over a mesh axis): each device holds O and
// LSE over its own keys; with M = max over devices of LSE, w = exp(LSE - M),
// O = sum(w * O_loc) / sum(w) and LSE = M + log(sum w).  Warp per (bh, t) row.
__global__ void attn_combine_scale_kernel(uint16_t* __restrict__ O, const float* __restrict__ lse,
                                          const float* __restrict__ m, float* __restrict__ w,
                                          int B, int H, int s, int ld) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)B * H * s;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb) {
    const int64_t bh = r / s, t = r - (r / s) * s;
    const int64_t b = bh / H, hh = bh - (bh / H) * H;
    const float wt = __expf(lse[r] - m[r]);
    uint32_t* o = reinterpret_cast<uint32_t*>(O + (b * s + t) * ld + hh * FA_D) + lane;
    const uint32_t v = *o;
    *o = pack_bf2(bf2f(v & 0xffff) * wt, bf2f(v >> 16) * wt);
    if (lane == 0) w[r] = wt;
  }
}

__global__ void attn_combine_finish_kernel(uint16_t* __restrict__ O, const float* __restrict__ wsum,
                                           const float* __restrict__ m, float* __restrict__ lse,
                                           int B, int H, int s, int ld) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)B * H * s;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb) {
    const int64_t bh = r / s, t = r - (r / s) * s;
    const int64_t b = bh / H, hh = bh - (bh / H) * H;
    const float ws = wsum[r];
    const float inv = 1.f / ws;
    uint32_t* o = reinterpret_cast<uint32_t*>(O + (b * s + t) * ld + hh * FA_D) + lane;
    const uint32_t v = *o;
    *o = pack_bf2(bf2f(v & 0xffff) * inv, bf2f(v >> 16) * inv);
    if (lane == 0) lse[r] = m[r] + __logf(ws);
  }
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 fa_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// (rows x ld) bf16 matrix, box 64 cols x 128 rows, 128B swizzle
static int fa_map(CUtensorMap* m, const void* base, int64_t rows, int64_t ld) {
  auto enc = fa_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 1;
  }
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return 1;
  }
  return 0;
}

// (rows x ld) fp32 matrix (dQ accumulator), box 32 cols x 128 rows, 128B swizzle
static int fa_map_f32(CUtensorMap* m, const void* base, int64_t rows, int64_t ld) {
  auto enc = fa_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return 1;
  }
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (f32) failed: " + std::to_string((int)r));
    return 1;
  }
  return 0;
}

static bool fa_args_ok(const void* p, int64_t ld) {
  return p && (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 8 == 0);
}


// Force-load this file's kernels (lazy module loading would load a kernel at its
// first launch, which blocks the host while an NCCL kernel spins on the device:
// a deadlock the executor's watchdog could not see).  See mp_preload_kernels.
template <typename F>
static inline int preload_one(F* f) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f)) == cudaSuccess ? 0 : 1;
}
int preload_attention() {
  return preload_one(fa_fwd_kernel<true>) | preload_one(fa_fwd_kernel<false>) |
         preload_one(fa_fwd_persist_kernel<0>) | preload_one(fa_fwd_persist_kernel<1>) |
         preload_one(fa_fwd_persist_kernel<2>) | preload_one(fa_fwd_persist_kernel<3>) |
         preload_one(fa_fwd_persist_kernel<4>) | preload_one(fa_fwd_persist_kernel<5>) |
         preload_one(fa_bwd_kernel<true>) | preload_one(fa_bwd_kernel<false>) | preload_one(fa_bwd_pre_kernel) |
         preload_one(attn_combine_scale_kernel) | preload_one(attn_combine_finish_kernel);
}
}  // namespace mp

using namespace mp;

static unsigned row_warps_grid(int64_t rows) {
  int64_t blocks = (rows * 32 + 255) / 256;
  if (blocks > num_sms() * 16) blocks = num_sms() * 16;
  return (unsigned)(blocks > 0 ? blocks : 1);
}

extern "C" int mp_attn_fwd_kv(const void* q, const void* k, const void* v, void* o, float* lse,
                              int64_t B, int64_t H, int64_t s, int64_t d, int64_t ld, float scale,
                              int64_t kv0, int64_t kv_len, void* stream) {
  clear_error();
  MP_CHECK_ARG(d == FA_D, "head dim must be 64");
  MP_CHECK_ARG(s % 128 == 0 && s > 0, "sequence length must be a multiple of 128");
  MP_CHECK_ARG(kv0 % 128 == 0 && kv_len % 128 == 0 && kv_len > 0 && kv0 >= 0 && kv0 + kv_len <= s,
               "key range must be 128-aligned and inside the sequence");
  MP_CHECK_ARG(ld >= H * d, "row stride smaller than heads*d");
  MP_CHECK_ARG(fa_args_ok(q, ld) && fa_args_ok(k, ld) && fa_args_ok(v, ld) && fa_args_ok(o, ld) &&
                   lse,
               "pointers must be 16-byte aligned with 8-element aligned rows");
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = fa_map(&mq, q, B * s, ld)) || (rc = fa_map(&mk, k, B * s, ld)) ||
      (rc = fa_map(&mv, v, B * s, ld)))
    return rc;
  // MPEXEC_FA_FWD=tile: one CTA per query tile (P in TMEM); =smem: the same with P
  // through shared memory (SS-form P V).  Default: the persistent kernel.
  // P in TMEM measured 127.9 -> 121.6 us at B=8, H=32, s=1024 (bench_gemm.py --attn)
  static const int mode = [] {
    const char* e = getenv("MPEXEC_FA_FWD");
    if (e && !strcmp(e, "smem")) return 2;
    if (e && !strcmp(e, "tile")) return 1;
    return 0;
  }();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(fa_fwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM);
    cudaFuncSetAttribute(fa_fwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM_PT);
    cudaFuncSetAttribute(fa_fwd_persist_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM_PERSIST);
    cudaFuncSetAttribute(fa_fwd_persist_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM_PERSIST);
    cudaFuncSetAttribute(fa_fwd_persist_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM_PERSIST);
    cudaFuncSetAttribute(fa_fwd_persist_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM_PERSIST);
    cudaFuncSetAttribute(fa_fwd_persist_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM_PERSIST);
    cudaFuncSetAttribute(fa_fwd_persist_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_FWD_SMEM_PERSIST);
    configured = true;
  }
  FaFwdParams p{(int)B, (int)H, (int)s, (int)ld, (int)kv0, (int)(kv_len / FA_BN),
                scale * 1.4426950408889634f, reinterpret_cast<uint16_t*>(o), lse};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // MPEXEC_FA_FWD_TRACE=<file>: diagnostics only (stamps need -DMP_FA_TRACE); every launch
  // syncs and overwrites <file> with int64 stamps [grid][1024][8]
  static const char* trace_path = getenv("MPEXEC_FA_FWD_TRACE");
  static long long* trace_buf = nullptr;
  const size_t trace_n = (size_t)2 * num_sms() * 1024 * 8;
  if (trace_path && mode == 0) {
    if (!trace_buf) cudaMalloc(&trace_buf, trace_n * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0xff, trace_n * sizeof(long long), st);
    p.trace = trace_buf;
  }
  if (mode == 0) {
    const int64_t work = (s / FA_BM) * B * H;
    const int64_t slots = 2 * (int64_t)num_sms();
    // MPEXEC_FA_FWD_EMU=k: k of every eight exponent pairs on the FMA pipe (0-5).
    // At B=8, H=32, s=1024: 0 -> 106.5 us, 1 -> 101.7, 2 -> 98.8, 3 -> 97.0 (default),
    // 4 -> 104.2, 5 -> 109.2 (profiles/r2/fa_fwd_exp2_emulation.txt)
    static const int emu = [] {
      const char* e = getenv("MPEXEC_FA_FWD_EMU");
      const int v = e ? atoi(e) : 3;
      return v < 0 ? 0 : (v > 5 ? 5 : v);
    }();
    const unsigned nb = (unsigned)(work < slots ? work : slots);
    if (emu == 5)
      fa_fwd_persist_kernel<5><<<nb, 192, FA_FWD_SMEM_PERSIST, st>>>(mq, mk, mv, p);
    else if (emu == 4)
      fa_fwd_persist_kernel<4><<<nb, 192, FA_FWD_SMEM_PERSIST, st>>>(mq, mk, mv, p);
    else if (emu == 3)
      fa_fwd_persist_kernel<3><<<nb, 192, FA_FWD_SMEM_PERSIST, st>>>(mq, mk, mv, p);
    else if (emu == 2)
      fa_fwd_persist_kernel<2><<<nb, 192, FA_FWD_SMEM_PERSIST, st>>>(mq, mk, mv, p);
    else if (emu == 1)
      fa_fwd_persist_kernel<1><<<nb, 192, FA_FWD_SMEM_PERSIST, st>>>(mq, mk, mv, p);
    else
      fa_fwd_persist_kernel<0><<<nb, 192, FA_FWD_SMEM_PERSIST, st>>>(mq, mk, mv, p);
  } else {
    dim3 grid((unsigned)(s / FA_BM), (unsigned)(B * H));
    if (mode == 2)
      fa_fwd_kernel<false><<<grid, 192, FA_FWD_SMEM, st>>>(mq, mk, mv, p);
    else
      fa_fwd_kernel<true><<<grid, 192, FA_FWD_SMEM_PT, st>>>(mq, mk, mv, p);
  }
  if (p.trace) {
    long long* h = (long long*)malloc(trace_n * sizeof(long long));
    cudaMemcpyAsync(h, trace_buf, trace_n * sizeof(long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE* fp = fopen(trace_path, "wb")) {
      fwrite(h, sizeof(long long), trace_n, fp);
      fclose(fp);
    }
    free(h);
  }
  MP_CHECK_LAUNCH();
  return 0;
}

extern "C" int mp_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                           int64_t B, int64_t H, int64_t s, int64_t d, int64_t ld, float scale,
                           void* stream) {
  return mp_attn_fwd_kv(q, k, v, o, lse, B, H, s, d, ld, scale, 0, s, stream);
}

extern "C" int mp_attn_bwd_kv(const void* q, const void* k, const void* v, const void* o,
                              const void* dout, const float* lse, float* dvec, float* dq_acc,
                              void* dk, void* dv, int64_t B, int64_t H, int64_t s, int64_t d,
                              int64_t ld, float scale, int64_t kv0, int64_t kv_len, void* stream) {
  clear_error();
  MP_CHECK_ARG(d == FA_D, "head dim must be 64");
  MP_CHECK_ARG(s % 128 == 0 && s > 0, "sequence length must be a multiple of 128");
  MP_CHECK_ARG(kv0 % 128 == 0 && kv_len % 128 == 0 && kv_len > 0 && kv0 >= 0 && kv0 + kv_len <= s,
               "key range must be 128-aligned and inside the sequence");
  MP_CHECK_ARG(fa_args_ok(q, ld) && fa_args_ok(k, ld) && fa_args_ok(v, ld) && fa_args_ok(o, ld) &&
                   fa_args_ok(dout, ld) && fa_args_ok(dk, ld) && fa_args_ok(dv, ld) && lse &&
                   dvec && dq_acc,
               "bad pointers");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  MP_CHECK_ARG(B * H * s < (1LL << 31) && ld % 8 == 0, "attention rows exceed int32 / ld not 8-aligned");
  fa_bwd_pre_kernel<<<row_warps_grid((B * H * s + 3) / 4), 256, 0, st>>>(
      reinterpret_cast<const uint16_t*>(o), reinterpret_cast<const uint16_t*>(dout), dvec, dq_acc,
      (int)B, (int)H, (int)s, (int)ld);
  MP_CHECK_LAUNCH();
  CUtensorMap mq, mk, mv, mdo, mdq;
  int rc;
  if ((rc = fa_map(&mq, q, B * s, ld)) || (rc = fa_map(&mk, k, B * s, ld)) ||
      (rc = fa_map(&mv, v, B * s, ld)) || (rc = fa_map(&mdo, dout, B * s, ld)) ||
      (rc = fa_map_f32(&mdq, dq_acc, B * s, ld)))
    return rc;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(fa_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_BWD_SMEM);
    cudaFuncSetAttribute(fa_bwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FA_BWD_SMEM);
    configured = true;
  }
  FaBwdParams p{(int)B, (int)H, (int)s, (int)ld, (int)kv0, (int)(kv_len / FA_BN), scale, lse,
                dvec, dq_acc, reinterpret_cast<uint16_t*>(dk), reinterpret_cast<uint16_t*>(dv),
                nullptr};
  const int64_t work = (kv_len / FA_BN) * B * H;
  dim3 grid((unsigned)(work < num_sms() ? work : num_sms()));
  // MPEXEC_FA_BWD_TRACE=<file>: diagnostics only -- every launch syncs and overwrites
  // <file> with int64 globaltimer stamps [grid][1024][8] (fa_stamp slots, -1 unused)
  static const char* trace_path = getenv("MPEXEC_FA_BWD_TRACE");
  static long long* trace_buf = nullptr;
  if (trace_path) {
    if (!trace_buf) cudaMalloc(&trace_buf, (size_t)num_sms() * 1024 * 8 * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0xff, (size_t)num_sms() * 1024 * 8 * sizeof(long long), st);
    p.trace = trace_buf;
  }
  // MPEXEC_FA_BWD_PT=1: P^T in TMEM (TS-form dV MMA, single dQ buffer).  Parity-green
  // but measured no faster (273.0 -> 275.1 us): off by default
  static const bool smem_p = getenv("MPEXEC_FA_BWD_PT") == nullptr;
  if (smem_p)
    fa_bwd_kernel<false><<<grid, FA_BWD_THREADS, FA_BWD_SMEM, st>>>(mq, mk, mv, mdo, mdq, p);
  else
    fa_bwd_kernel<true><<<grid, FA_BWD_THREADS, FA_BWD_SMEM, st>>>(mq, mk, mv, mdo, mdq, p);
  MP_CHECK_LAUNCH();
  if (trace_path) {
    const size_t n = (size_t)grid.x * 1024 * 8;
    long long* h = (long long*)malloc(n * sizeof(long long));
    cudaMemcpyAsync(h, trace_buf, n * sizeof(long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE* fp = fopen(trace_path, "wb")) {
      fwrite(h, sizeof(long long), n, fp);
      fclose(fp);
    }
    free(h);
  }
  return 0;
}

extern "C" int mp_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                           const void* dout, const float* lse, float* dvec, float* dq_acc,
                           void* dk, void* dv, int64_t B, int64_t H, int64_t s, int64_t d,
                           int64_t ld, float scale, void* stream) {
  return mp_attn_bwd_kv(q, k, v, o, dout, lse, dvec, dq_acc, dk, dv, B, H, s, d, ld, scale, 0, s,
                        stream);
}

extern "C" int mp_attn_combine_scale(void* o, const float* lse, const float* m, float* w, int64_t B,
                                     int64_t H, int64_t s, int64_t d, int64_t ld, void* stream) {
  clear_error();
  MP_CHECK_ARG(d == FA_D && fa_args_ok(o, ld) && lse && m && w, "bad arguments");
  attn_combine_scale_kernel<<<row_warps_grid(B * H * s), 256, 0,
                              reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint16_t*>(o), lse, m, w, (int)B, (int)H, (int)s, (int)ld);
  MP_CHECK_LAUNCH();
  return 0;
}

extern "C" int mp_attn_combine_finish(void* o, const float* wsum, const float* m, float* lse,
                                      int64_t B, int64_t H, int64_t s, int64_t d, int64_t ld,
                                      void* stream) {
  clear_error();
  MP_CHECK_ARG(d == FA_D && fa_args_ok(o, ld) && wsum && m && lse, "bad arguments");
  attn_combine_finish_kernel<<<row_warps_grid(B * H * s), 256, 0,
                               reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint16_t*>(o), wsum, m, lse, (int)B, (int)H, (int)s, (int)ld);
  MP_CHECK_LAUNCH();
  return 0;
}
