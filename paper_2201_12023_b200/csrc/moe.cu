// GShard top-2 routing for the MoE builder's layout adapters (builders.py,
// binding.py): the gates -> dispatch-mask / combine-weight reshapes and their
// backward.  Integer work plus byte scatter; HBM-bound (the masks are written
// once per microbatch and mostly zero).
//
// Routing of one group of S tokens (tokens t = g*S + s, s ascending), E experts,
// capacity C (GShard Alg. 1, arXiv 2006.16668):
//   e1 = argmax_e gates[t, e], e2 = argmax_{e != e1} gates[t, e]   (lowest index on ties)
//   pos1 = #{s' < s : e1(s') = e1(s)}                 kept if pos1 < C
//   pos2 = min(C, #{s : e1(s) = e2(t)}) + #{s' < s : e2(s') = e2(s)}   kept if pos2 < C
// route[t] = {e1, pos1 or -1, e2, pos2 or -1}.
#include "common.cuh"
#include "../../include/mp_exec.h"

#define MP_STREAM(s) reinterpret_cast<cudaStream_t>(s)

namespace mp {
namespace {

constexpr int kRouteThreads = 1024;
constexpr int kMaxExperts = 64;

__device__ __forceinline__ void top2(const uint16_t* row, int E, int& e1, int& e2) {
  float b1 = -INFINITY, b2 = -INFINITY;
  e1 = 0;
  e2 = E > 1 ? 1 : 0;
  int i1 = -1, i2 = -1;
  for (int e = 0; e < E; ++e) {
    float v = bf2f(row[e]);
    if (i1 < 0 || v > b1) {
      b2 = b1; i2 = i1;
      b1 = v; i1 = e;
    } else if (i2 < 0 || v > b2) {
      b2 = v; i2 = e;
    }
  }
  e1 = i1;
  e2 = i2 < 0 ? i1 : i2;
}

// Exclusive rank of every active thread's key among the block's earlier threads
// with the same key, plus `base[key]`; base[] is advanced by the block's counts.
// cnt: [32][kMaxExperts] shared scratch.
__device__ __forceinline__ int block_rank(int key, bool active, int E, int* cnt, int* base) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  int k = active ? key : -1;
  unsigned peers = __match_any_sync(0xffffffffu, k);
  int rank = __popc(peers & ((1u << lane) - 1u));
  if (active && rank == 0) cnt[warp * E + key] = __popc(peers);
  __syncthreads();
  if (threadIdx.x < E) {
    int e = threadIdx.x, run = base[e];
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      int c = cnt[w * E + e];
      cnt[w * E + e] = run;
      run += c;
    }
    base[e] = run;
  }
  __syncthreads();
  int pos = active ? cnt[warp * E + key] + rank : -1;
  __syncthreads();
  return pos;
}

__global__ void __launch_bounds__(kRouteThreads)
moe_route_kernel(const uint16_t* __restrict__ gates, int64_t ld, int S, int E, int C,
                 int* __restrict__ route) {
  __shared__ int cnt[32 * kMaxExperts];
  __shared__ int base[kMaxExperts];
  const int64_t g0 = (int64_t)blockIdx.x * S;
  if (threadIdx.x < E) base[threadIdx.x] = 0;
  __syncthreads();
  // pass 1: top-1 positions
  for (int c0 = 0; c0 < S; c0 += blockDim.x) {
    int s = c0 + threadIdx.x;
    bool act = s < S;
    int e1 = 0, e2 = 0;
    if (act) top2(gates + (g0 + s) * ld, E, e1, e2);
    int p1 = block_rank(e1, act, E, cnt, base);
    if (act) {
      int* r = route + (g0 + s) * 4;
      r[0] = e1;
      r[1] = p1 < C ? p1 : -1;
      r[2] = e2;
    }
  }
  __syncthreads();
  if (threadIdx.x < E) base[threadIdx.x] = min(base[threadIdx.x], C);
  __syncthreads();
  // pass 2: top-2 positions behind the kept top-1 tokens
  for (int c0 = 0; c0 < S; c0 += blockDim.x) {
    int s = c0 + threadIdx.x;
    bool act = s < S;
    int e2 = act ? route[(g0 + s) * 4 + 2] : 0;
    int p2 = block_rank(e2, act, E, cnt, base);
    if (act) route[(g0 + s) * 4 + 3] = p2 < C ? p2 : -1;
  }
}

// mode 0: dispatch mask (G, E*C, S) of ones; mode 1: combine weights (G, S, E*C) = gates.
// `out` is zeroed by the caller.
__global__ void moe_mask_kernel(const int* __restrict__ route, const uint16_t* __restrict__ gates,
                                int64_t ld, uint16_t* __restrict__ out, int64_t T, int S, int E,
                                int C, int mode) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int64_t g = t / S, s = t % S, EC = (int64_t)E * C;
  const int* r = route + t * 4;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int e = r[2 * k], p = r[2 * k + 1];
    if (p < 0) continue;
    if (mode == 0)
      out[(g * EC + (int64_t)e * C + p) * S + s] = 0x3f80;  // 1.0
    else
      out[(g * S + s) * EC + (int64_t)e * C + p] = gates[t * ld + e];
  }
}

// Backward of the two adapters, (T, E) bf16.  Combine (mode 1): out[t, e] = d at
// the routed slot of (t, e), else 0 -- the combine weights are the gates there.
// Dispatch (mode 0): zero -- routing and the 0/1 mask are piecewise constant in
// the gates, so the exact gradient vanishes.
__global__ void moe_mask_grad_kernel(const int* __restrict__ route, const uint16_t* __restrict__ d,
                                     uint16_t* __restrict__ out, int64_t T, int S, int E, int C,
                                     int mode) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T * E) return;
  const int64_t t = i / E;
  const int e = (int)(i % E);
  const int64_t g = t / S, s = t % S, EC = (int64_t)E * C;
  const int* r = route + t * 4;
  uint16_t v = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int p = r[2 * k + 1];
    if (mode == 1 && r[2 * k] == e && p >= 0) v = d[(g * S + s) * EC + (int64_t)e * C + p];
  }
  out[i] = v;
}


// Force-load this file's kernels (lazy module loading would load a kernel at its
// first launch, which blocks the host while an NCCL kernel spins on the device:
// a deadlock the executor's watchdog could not see).  See mp_preload_kernels.
template <typename F>
static inline int preload_one(F* f) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f)) == cudaSuccess ? 0 : 1;
}
int preload_moe_impl() {
  return preload_one(moe_route_kernel) | preload_one(moe_mask_kernel) |
         preload_one(moe_mask_grad_kernel);
}
}  // namespace
int preload_moe() { return preload_moe_impl(); }
}  // namespace mp


using namespace mp;

extern "C" {

int mp_moe_route(const void* gates, int64_t ld, int64_t groups, int S, int E, int C, int* route,
                 void* stream) {
  clear_error();
  MP_CHECK_ARG(gates && route && groups >= 0 && S > 0 && E >= 2 && E <= kMaxExperts && C > 0 &&
                   ld >= E,
               "bad args");
  if (groups == 0) return 0;
  moe_route_kernel<<<(unsigned)groups, kRouteThreads, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)gates, ld, S, E, C, route);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_moe_mask(const int* route, const void* gates, int64_t ld, void* out, int64_t tokens, int S,
                int E, int C, int mode, void* stream) {
  clear_error();
  MP_CHECK_ARG(route && gates && out && tokens >= 0 && S > 0 && tokens % S == 0 && E > 0 &&
                   C > 0 && (mode == 0 || mode == 1),
               "bad args");
  if (tokens == 0) return 0;
  cudaStream_t s = MP_STREAM(stream);
  if (cudaMemsetAsync(out, 0, (size_t)tokens * E * C * 2, s) != cudaSuccess) {
    set_error("mp_moe_mask: memset failed");
    return 1;
  }
  moe_mask_kernel<<<(unsigned)((tokens + 255) / 256), 256, 0, s>>>(
      route, (const uint16_t*)gates, ld, (uint16_t*)out, tokens, S, E, C, mode);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_moe_mask_grad(const int* route, const void* d, void* out, int64_t tokens, int S, int E,
                     int C, int mode, void* stream) {
  clear_error();
  MP_CHECK_ARG(route && d && out && tokens >= 0 && S > 0 && tokens % S == 0 && E > 0 && C > 0 &&
                   (mode == 0 || mode == 1),
               "bad args");
  int64_t n = tokens * E;
  if (n == 0) return 0;
  moe_mask_grad_kernel<<<(unsigned)((n + 255) / 256), 256, 0, MP_STREAM(stream)>>>(
      route, (const uint16_t*)d, (uint16_t*)out, tokens, S, E, C, mode);
  MP_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
