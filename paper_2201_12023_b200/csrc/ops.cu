// Memory-bound kernels of the plan executor: trivial-member ops (elementwise /
// softmax, reference intra.py:93-160 merge + propagate), box pack/unpack for
// cross-mesh transfers (reshard.py:97-157), the fused optimizer step and casts.
// All are HBM-bound: 16-byte vector accesses, grid sized in multiples of the SM
// count, one warp per row for row ops.
#include <cuda_runtime.h>
#include <atomic>
#include <mutex>
#include <algorithm>
#include "common.cuh"
#include "../../include/mp_exec.h"

namespace mp {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
void clear_error() { g_err.clear(); }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int num_sms() {
  static int dev_sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!dev_sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    dev_sms[dev] = v > 0 ? v : 148;
  }
  return dev_sms[dev];
}

static inline int grid_for(int64_t work_items, int threads) {
  int64_t blocks = (work_items + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

// ------------------------------------------------------------ elementwise (bf16)
// Vector path handles 8 elements per 16-byte access; tail is scalar.
template <typename F>
__global__ void unary_bf16_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
                                  int64_t n, F f) {
  const int64_t nv = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 a = reinterpret_cast<const uint4*>(x)[i];
    uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w[j] = pack_bf2(f(bf2f(w[j] & 0xffff)), f(bf2f(w[j] >> 16)));
    reinterpret_cast<uint4*>(y)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  for (int64_t i = nv * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = f2bf(f(bf2f(x[i])));
}

template <typename F>
__global__ void binary_bf16_kernel(const uint16_t* __restrict__ a, const uint16_t* __restrict__ b,
                                   uint16_t* __restrict__ y, int64_t n, F f) {
  const int64_t nv = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 u = reinterpret_cast<const uint4*>(a)[i];
    uint4 v = reinterpret_cast<const uint4*>(b)[i];
    uint32_t wa[4] = {u.x, u.y, u.z, u.w}, wb[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      wa[j] = pack_bf2(f(bf2f(wa[j] & 0xffff), bf2f(wb[j] & 0xffff)),
                       f(bf2f(wa[j] >> 16), bf2f(wb[j] >> 16)));
    reinterpret_cast<uint4*>(y)[i] = make_uint4(wa[0], wa[1], wa[2], wa[3]);
  }
  for (int64_t i = nv * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = f2bf(f(bf2f(a[i]), bf2f(b[i])));
}

struct GeluF {
  __device__ float operator()(float x) const { return gelu_tanh(x); }
};
struct GeluBwdF {
  __device__ float operator()(float x, float g) const { return gelu_tanh_grad(x) * g; }
};
struct AddF {
  __device__ float operator()(float a, float b) const { return a + b; }
};
struct ScaleF {
  float s;
  __device__ float operator()(float x) const { return s * x; }
};

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__global__ void sumsq_kernel(const uint16_t* __restrict__ x, float* out, int64_t n) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv = n / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 a = reinterpret_cast<const uint4*>(x)[i];
    uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float lo = bf2f(w[j] & 0xffff), hi = bf2f(w[j] >> 16);
      acc += lo * lo + hi * hi;
    }
  }
  for (int64_t i = nv * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float v = bf2f(x[i]);
    acc += v * v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(out, v);
  }
}

// ------------------------------------------------------------ softmax rows
// One warp per row; row length arbitrary; two passes over the row (the second
// hits L1/L2).  Inputs bf16, math fp32.
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// local (max, sumexp) of scale*x over the row; online merge per lane
__device__ __forceinline__ void row_stats(const uint16_t* __restrict__ xr, int64_t cols,
                                          float scale, int lane, float& m_out, float& s_out) {
  float m = -INFINITY, s = 0.f;
  const bool vec = ((cols & 7) == 0) && ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
  if (vec) {
    for (int64_t c = (int64_t)lane * 8; c < cols; c += 256) {
      uint4 a = *reinterpret_cast<const uint4*>(xr + c);
      uint32_t w[4] = {a.x, a.y, a.z, a.w};
      float v[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[2 * j] = scale * bf2f(w[j] & 0xffff);
        v[2 * j + 1] = scale * bf2f(w[j] >> 16);
      }
      float lm = v[0];
#pragma unroll
      for (int j = 1; j < 8; ++j) lm = fmaxf(lm, v[j]);
      float nm = fmaxf(m, lm);
      float acc = s * __expf(m - nm);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += __expf(v[j] - nm);
      m = nm;
      s = acc;
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) {
      float v = scale * bf2f(xr[c]);
      float nm = fmaxf(m, v);
      s = s * __expf(m - nm) + __expf(v - nm);
      m = nm;
    }
  }
  float gm = warp_max(m);
  float ls = (m == -INFINITY) ? 0.f : s * __expf(m - gm);
  m_out = gm;
  s_out = warp_sum(ls);
}

__device__ __forceinline__ void row_write(const uint16_t* __restrict__ xr, uint16_t* __restrict__ yr,
                                          int64_t cols, float scale, float m, float inv, int lane) {
  const bool vec = ((cols & 7) == 0) && ((reinterpret_cast<uintptr_t>(xr) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(yr) & 15) == 0);
  if (vec) {
    for (int64_t c = (int64_t)lane * 8; c < cols; c += 256) {
      uint4 a = *reinterpret_cast<const uint4*>(xr + c);
      uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        w[j] = pack_bf2(__expf(scale * bf2f(w[j] & 0xffff) - m) * inv,
                        __expf(scale * bf2f(w[j] >> 16) - m) * inv);
      *reinterpret_cast<uint4*>(yr + c) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) yr[c] = f2bf(__expf(scale * bf2f(xr[c]) - m) * inv);
  }
}

__global__ void softmax_fwd_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
                                   int64_t rows, int64_t cols, int64_t ld, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb) {
    const uint16_t* xr = x + r * ld;
    float m, s;
    row_stats(xr, cols, scale, lane, m, s);
    row_write(xr, y + r * ld, cols, scale, m, 1.f / s, lane);
  }
}

__global__ void softmax_stats_kernel(const uint16_t* __restrict__ x, float* __restrict__ stats,
                                     int64_t rows, int64_t cols, int64_t ld, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb) {
    float m, s;
    row_stats(x + r * ld, cols, scale, lane, m, s);
    if (lane == 0) {   // planar [3, rows]: max (all-reduced in place), sum, max copy
      stats[r] = m;
      stats[rows + r] = s;
      stats[2 * rows + r] = m;
    }
  }
}

// after the MAX all-reduce of stats[0]: rescale the local sums to the group max
__global__ void softmax_rescale_kernel(float* __restrict__ stats, int64_t rows) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += stride) {
    const float mg = stats[r], ml = stats[2 * rows + r];
    stats[rows + r] = (ml == -INFINITY) ? 0.f : stats[rows + r] * __expf(ml - mg);
  }
}

__global__ void softmax_apply_kernel(const uint16_t* __restrict__ x, const float* __restrict__ stats,
                                     uint16_t* __restrict__ y, int64_t rows, int64_t cols,
                                     int64_t ld, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb)
    row_write(x + r * ld, y + r * ld, cols, scale, stats[r], 1.f / stats[rows + r], lane);
}

__device__ __forceinline__ float row_dot(const uint16_t* __restrict__ yr,
                                         const uint16_t* __restrict__ gr, int64_t cols, int lane) {
  float acc = 0.f;
  const bool vec = ((cols & 7) == 0) && ((reinterpret_cast<uintptr_t>(yr) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(gr) & 15) == 0);
  if (vec) {
    for (int64_t c = (int64_t)lane * 8; c < cols; c += 256) {
      uint4 a = *reinterpret_cast<const uint4*>(yr + c);
      uint4 b = *reinterpret_cast<const uint4*>(gr + c);
      uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        acc += bf2f(wa[j] & 0xffff) * bf2f(wb[j] & 0xffff) + bf2f(wa[j] >> 16) * bf2f(wb[j] >> 16);
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) acc += bf2f(yr[c]) * bf2f(gr[c]);
  }
  return warp_sum(acc);
}

__global__ void softmax_rowdot_kernel(const uint16_t* __restrict__ y, const uint16_t* __restrict__ g,
                                      float* __restrict__ out, int64_t rows, int64_t cols,
                                      int64_t ld) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb) {
    float d = row_dot(y + r * ld, g + r * ld, cols, lane);
    if (lane == 0) out[r] = d;
  }
}

__global__ void softmax_bwd_kernel(const uint16_t* __restrict__ y, const uint16_t* __restrict__ g,
                                   uint16_t* __restrict__ dx, const float* __restrict__ rowdot,
                                   int64_t rows, int64_t cols, int64_t ld, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb) {
    const uint16_t* yr = y + r * ld;
    const uint16_t* gr = g + r * ld;
    uint16_t* dr = dx + r * ld;
    float d = rowdot ? rowdot[r] : row_dot(yr, gr, cols, lane);
    const bool vec = ((cols & 7) == 0) && ((reinterpret_cast<uintptr_t>(yr) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(gr) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(dr) & 15) == 0);
    if (vec) {
      for (int64_t c = (int64_t)lane * 8; c < cols; c += 256) {
        uint4 a = *reinterpret_cast<const uint4*>(yr + c);
        uint4 b = *reinterpret_cast<const uint4*>(gr + c);
        uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float y0 = bf2f(wa[j] & 0xffff), y1 = bf2f(wa[j] >> 16);
          float g0 = bf2f(wb[j] & 0xffff), g1 = bf2f(wb[j] >> 16);
          wa[j] = pack_bf2(scale * y0 * (g0 - d), scale * y1 * (g1 - d));
        }
        *reinterpret_cast<uint4*>(dr + c) = make_uint4(wa[0], wa[1], wa[2], wa[3]);
      }
    } else {
      for (int64_t c = lane; c < cols; c += 32) {
        float yy = bf2f(yr[c]);
        dr[c] = f2bf(scale * yy * (bf2f(gr[c]) - d));
      }
    }
  }
}

// ------------------------------------------------------------ box pack / unpack
struct BoxArgs {
  int64_t ext[4];
  int64_t str[4];  // strides of the strided side, elements
  int64_t off;     // element offset of lo on the strided side
  int rank;
};

template <typename T, bool PACK>
__global__ void box_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, BoxArgs a,
                                int64_t total) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    int64_t rem = i, off = a.off;
#pragma unroll
    for (int d = 3; d >= 0; --d) {
      if (d < a.rank) {
        int64_t c = rem % a.ext[d];
        rem /= a.ext[d];
        off += c * a.str[d];
      }
    }
    if (PACK)
      dst[i] = src[off];
    else
      dst[off] = src[i];
  }
}

// Row form of box_copy_kernel: one warp per row of the innermost (unit-stride)
// dimension, the row's strided offset decoded once per row instead of once per
// element (64-bit div / mod per element capped the element form at ~0.8 TB/s).
template <typename T, bool PACK>
__global__ void box_rows_kernel(const T* __restrict__ src, T* __restrict__ dst, BoxArgs a,
                                int64_t rows, int64_t inner) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += wstride) {
    int64_t rem = row, off = a.off;
#pragma unroll
    for (int d = 2; d >= 0; --d) {
      if (d < a.rank - 1) {
        const int64_t c = rem % a.ext[d];
        rem /= a.ext[d];
        off += c * a.str[d];
      }
    }
    const T* s = PACK ? src + off : src + row * inner;
    T* t = PACK ? dst + row * inner : dst + off;
    for (int64_t c = lane; c < inner; c += 32) t[c] = s[c];
  }
}

static int box_copy(const void* src, void* dst, const int64_t* strides, const int64_t* lo,
                    const int64_t* ext, int rank, int elem_bytes, bool pack, cudaStream_t s) {
  if (rank < 1 || rank > 4) {
    set_error("box rank must be 1..4");
    return 2;
  }
  BoxArgs a{};
  a.rank = rank;
  a.off = 0;
  int64_t total = 1;
  for (int d = 0; d < rank; ++d) {
    a.ext[d] = ext[d];
    a.str[d] = strides[d];
    a.off += lo[d] * strides[d];
    total *= ext[d];
  }
  if (total == 0) return 0;
  // Vectorise the innermost dim when it is unit-stride and 16-byte divisible.
  int vec = 1;
  if (strides[rank - 1] == 1) {
    const int64_t inner_b = ext[rank - 1] * elem_bytes;
    bool ok = (inner_b % 16 == 0) && ((a.off * elem_bytes) % 16 == 0) && aligned16(src) &&
              aligned16(dst);
    for (int d = 0; d < rank - 1 && ok; ++d) ok = ((strides[d] * elem_bytes) % 16 == 0);
    if (ok) vec = 16 / elem_bytes;
  }
  const int threads = 256;
  if (vec > 1) {
    BoxArgs v = a;
    v.ext[rank - 1] = a.ext[rank - 1] / vec;
    for (int d = 0; d < rank - 1; ++d) v.str[d] = a.str[d] / vec;
    v.str[rank - 1] = 1;
    v.off = a.off / vec;
    int64_t tv = total / vec;
    const int64_t inner = v.ext[rank - 1], rows = tv / inner;
    if (rank > 1 && rows >= 64 && inner >= 8) {
      const int64_t warps = threads / 32;
      const int64_t blocks = std::min<int64_t>((rows + warps - 1) / warps, 148 * 16);
      if (pack)
        box_rows_kernel<uint4, true><<<(unsigned)blocks, threads, 0, s>>>(
            (const uint4*)src, (uint4*)dst, v, rows, inner);
      else
        box_rows_kernel<uint4, false><<<(unsigned)blocks, threads, 0, s>>>(
            (const uint4*)src, (uint4*)dst, v, rows, inner);
    } else if (pack) {
      box_copy_kernel<uint4, true><<<grid_for(tv, threads), threads, 0, s>>>(
          (const uint4*)src, (uint4*)dst, v, tv);
    } else {
      box_copy_kernel<uint4, false><<<grid_for(tv, threads), threads, 0, s>>>(
          (const uint4*)src, (uint4*)dst, v, tv);
    }
  } else if (elem_bytes == 2) {
    if (pack)
      box_copy_kernel<uint16_t, true><<<grid_for(total, threads), threads, 0, s>>>(
          (const uint16_t*)src, (uint16_t*)dst, a, total);
    else
      box_copy_kernel<uint16_t, false><<<grid_for(total, threads), threads, 0, s>>>(
          (const uint16_t*)src, (uint16_t*)dst, a, total);
  } else if (elem_bytes == 4) {
    if (pack)
      box_copy_kernel<uint32_t, true><<<grid_for(total, threads), threads, 0, s>>>(
          (const uint32_t*)src, (uint32_t*)dst, a, total);
    else
      box_copy_kernel<uint32_t, false><<<grid_for(total, threads), threads, 0, s>>>(
          (const uint32_t*)src, (uint32_t*)dst, a, total);
  } else {
    set_error("elem_bytes must be 2 or 4");
    return 2;
  }
  return 0;
}

// ------------------------------------------------------------ optimizer / casts
__global__ void adam_kernel(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                            const float* __restrict__ g, uint16_t* __restrict__ p, int64_t n,
                            float lr, float b1, float b2, float eps, float wd, float gscale,
                            float bc1, float bc2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float gi = g[i] * gscale;
    float mi = b1 * m[i] + (1.f - b1) * gi;
    float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    float w = master[i];
    float upd = (mi / bc1) / (sqrtf(vi / bc2) + eps) + wd * w;
    w -= lr * upd;
    master[i] = w;
    p[i] = f2bf(w);
  }
}

// 4 parameters per thread (16-byte fp32 / 8-byte bf16 accesses); same math as adam_kernel
__global__ void adam4_kernel(float4* __restrict__ master, float4* __restrict__ m,
                             float4* __restrict__ v, const float4* __restrict__ g,
                             uint2* __restrict__ p, int64_t n4, float lr, float b1, float b2,
                             float eps, float wd, float gscale, float bc1, float bc2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 g4 = __ldcs(g + i);
    float4 m4 = m[i], v4 = v[i], w4 = master[i];
    float* gp = (float*)&g4;
    float* mp_ = (float*)&m4;
    float* vp = (float*)&v4;
    float* wp = (float*)&w4;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gi = gp[e] * gscale;
      mp_[e] = b1 * mp_[e] + (1.f - b1) * gi;
      vp[e] = b2 * vp[e] + (1.f - b2) * gi * gi;
      const float upd = (mp_[e] / bc1) / (sqrtf(vp[e] / bc2) + eps) + wd * wp[e];
      wp[e] -= lr * upd;
    }
    m[i] = m4;
    v[i] = v4;
    master[i] = w4;
    p[i] = make_uint2(pack_bf2(w4.x, w4.y), pack_bf2(w4.z, w4.w));
  }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ x, uint16_t* __restrict__ y, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) y[i] = f2bf(x[i]);
}
__global__ void cast4_f32_bf16_kernel(const float4* __restrict__ x, uint2* __restrict__ y,
                                      int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 a = __ldcs(x + i);
    y[i] = make_uint2(pack_bf2(a.x, a.y), pack_bf2(a.z, a.w));
  }
}
__global__ void cast_bf16_f32_kernel(const uint16_t* __restrict__ x, float* __restrict__ y, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) y[i] = bf2f(x[i]);
}
__global__ void accum_bf16_f32_kernel(const uint16_t* __restrict__ x, float* __restrict__ y, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) y[i] += bf2f(x[i]);
}

// y = beta * y + sum_p parts[p] (split-K partials, summed in fixed order p = 0..)
__global__ void sum_parts_f32_kernel(const float4* __restrict__ parts, int64_t nparts, int64_t n4,
                                     float4* __restrict__ y, float beta) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (beta != 0.f) {
      float4 v = y[i];
      acc = make_float4(beta * v.x, beta * v.y, beta * v.z, beta * v.w);
    }
    for (int64_t p = 0; p < nparts; ++p) {
      float4 v = __ldcs(parts + p * n4 + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    y[i] = acc;
  }
}


// Force-load this file's kernels (lazy module loading would load a kernel at its
// first launch, which blocks the host while an NCCL kernel spins on the device:
// a deadlock the executor's watchdog could not see).  See mp_preload_kernels.
template <typename F>
static inline int preload_one(F* f) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f)) == cudaSuccess ? 0 : 1;
}
int preload_ops() {
  return preload_one(unary_bf16_kernel<ScaleF>) | preload_one(unary_bf16_kernel<GeluF>) |
         preload_one(binary_bf16_kernel<AddF>) | preload_one(binary_bf16_kernel<GeluBwdF>) |
         preload_one(sumsq_kernel) | preload_one(softmax_fwd_kernel) |
         preload_one(softmax_stats_kernel) | preload_one(softmax_rescale_kernel) |
         preload_one(softmax_apply_kernel) | preload_one(softmax_rowdot_kernel) |
         preload_one(softmax_bwd_kernel) | preload_one(box_copy_kernel<uint32_t, false>) |
         preload_one(box_copy_kernel<uint32_t, true>) | preload_one(box_copy_kernel<uint16_t, false>) |
         preload_one(box_copy_kernel<uint16_t, true>) | preload_one(box_copy_kernel<uint4, false>) |
         preload_one(box_copy_kernel<uint4, true>) | preload_one(box_rows_kernel<uint4, true>) |
         preload_one(box_rows_kernel<uint4, false>) | preload_one(adam_kernel) |
         preload_one(adam4_kernel) | preload_one(cast_f32_bf16_kernel) |
         preload_one(cast4_f32_bf16_kernel) | preload_one(cast_bf16_f32_kernel) |
         preload_one(accum_bf16_f32_kernel) | preload_one(sum_parts_f32_kernel);
}
int preload_gemm();
int preload_attention();
int preload_conv();
int preload_moe();
}  // namespace mp

using namespace mp;

#define MP_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

int mp_abi_version(void) { return 1; }
const char* mp_last_error(void) { return g_err.c_str(); }
uint64_t mp_launch_count(void) { return g_launches.load(); }
int mp_preload_kernels(void) {
  clear_error();
  const int bad = preload_ops() | preload_gemm() | preload_attention() | preload_conv() |
                  preload_moe();
  if (bad) {
    set_error(std::string("kernel preload failed: ") + cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  return 0;
}

int mp_gelu_fwd(const void* x, void* y, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && y && n >= 0, "bad args");
  MP_CHECK_ARG(aligned16(x) && aligned16(y), "pointers must be 16-byte aligned");
  if (n == 0) return 0;
  unary_bf16_kernel<<<grid_for((n + 7) / 8, 256), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)x, (uint16_t*)y, n, GeluF{});
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_gelu_bwd(const void* x, const void* dy, void* dx, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && dy && dx && n >= 0, "bad args");
  MP_CHECK_ARG(aligned16(x) && aligned16(dy) && aligned16(dx), "pointers must be 16-byte aligned");
  if (n == 0) return 0;
  binary_bf16_kernel<<<grid_for((n + 7) / 8, 256), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)x, (const uint16_t*)dy, (uint16_t*)dx, n, GeluBwdF{});
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_add(const void* a, const void* b, void* y, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(a && b && y && n >= 0, "bad args");
  MP_CHECK_ARG(aligned16(a) && aligned16(b) && aligned16(y), "pointers must be 16-byte aligned");
  if (n == 0) return 0;
  binary_bf16_kernel<<<grid_for((n + 7) / 8, 256), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)a, (const uint16_t*)b, (uint16_t*)y, n, AddF{});
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_scale(const void* x, void* y, float scale, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && y && n >= 0, "bad args");
  MP_CHECK_ARG(aligned16(x) && aligned16(y), "pointers must be 16-byte aligned");
  if (n == 0) return 0;
  unary_bf16_kernel<<<grid_for((n + 7) / 8, 256), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)x, (uint16_t*)y, n, ScaleF{scale});
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_sumsq(const void* x, float* out, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && out && n >= 0, "bad args");
  MP_CHECK_ARG(aligned16(x), "pointer must be 16-byte aligned");
  if (n == 0) return 0;
  sumsq_kernel<<<grid_for((n + 7) / 8, 256), 256, 0, MP_STREAM(stream)>>>((const uint16_t*)x, out, n);
  MP_CHECK_LAUNCH();
  return 0;
}

static int row_grid(int64_t rows) { return grid_for(rows * 32, 256); }

int mp_softmax_fwd(const void* x, void* y, int64_t rows, int64_t cols, int64_t ld, float scale,
                   void* stream) {
  clear_error();
  MP_CHECK_ARG(x && y && rows >= 0 && cols > 0 && ld >= cols, "bad args");
  if (rows == 0) return 0;
  softmax_fwd_kernel<<<row_grid(rows), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)x, (uint16_t*)y, rows, cols, ld, scale);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_softmax_stats(const void* x, float* stats, int64_t rows, int64_t cols, int64_t ld,
                     float scale, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && stats && rows >= 0 && cols > 0 && ld >= cols, "bad args");
  if (rows == 0) return 0;
  softmax_stats_kernel<<<row_grid(rows), 256, 0, MP_STREAM(stream)>>>((const uint16_t*)x, stats,
                                                                      rows, cols, ld, scale);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_softmax_rescale(float* stats, int64_t rows, void* stream) {
  clear_error();
  MP_CHECK_ARG(stats && rows >= 0, "bad args");
  if (rows == 0) return 0;
  softmax_rescale_kernel<<<grid_for(rows, 256), 256, 0, MP_STREAM(stream)>>>(stats, rows);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_softmax_apply(const void* x, const float* stats, void* y, int64_t rows, int64_t cols,
                     int64_t ld, float scale, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && stats && y && rows >= 0 && cols > 0 && ld >= cols, "bad args");
  if (rows == 0) return 0;
  softmax_apply_kernel<<<row_grid(rows), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)x, stats, (uint16_t*)y, rows, cols, ld, scale);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_softmax_bwd(const void* y, const void* dy, void* dx, const float* rowdot, int64_t rows,
                   int64_t cols, int64_t ld, float scale, void* stream) {
  clear_error();
  MP_CHECK_ARG(y && dy && dx && rows >= 0 && cols > 0 && ld >= cols, "bad args");
  if (rows == 0) return 0;
  softmax_bwd_kernel<<<row_grid(rows), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)y, (const uint16_t*)dy, (uint16_t*)dx, rowdot, rows, cols, ld, scale);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_softmax_rowdot(const void* y, const void* dy, float* rowdot, int64_t rows, int64_t cols,
                      int64_t ld, void* stream) {
  clear_error();
  MP_CHECK_ARG(y && dy && rowdot && rows >= 0 && cols > 0 && ld >= cols, "bad args");
  if (rows == 0) return 0;
  softmax_rowdot_kernel<<<row_grid(rows), 256, 0, MP_STREAM(stream)>>>(
      (const uint16_t*)y, (const uint16_t*)dy, rowdot, rows, cols, ld);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_pack_box(const void* src, const int64_t* src_strides, const int64_t* lo, const int64_t* ext,
                int rank, int elem_bytes, void* dst, void* stream) {
  clear_error();
  MP_CHECK_ARG(src && dst && src_strides && lo && ext, "null argument");
  int rc = box_copy(src, dst, src_strides, lo, ext, rank, elem_bytes, true, MP_STREAM(stream));
  if (rc) return rc;
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_unpack_box(const void* src, void* dst, const int64_t* dst_strides, const int64_t* lo,
                  const int64_t* ext, int rank, int elem_bytes, void* stream) {
  clear_error();
  MP_CHECK_ARG(src && dst && dst_strides && lo && ext, "null argument");
  int rc = box_copy(src, dst, dst_strides, lo, ext, rank, elem_bytes, false, MP_STREAM(stream));
  if (rc) return rc;
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_adam_step(float* master, float* m, float* v, const float* grad, void* param_bf16, int64_t n,
                 float lr, float beta1, float beta2, float eps, float weight_decay,
                 float grad_scale, int64_t step, void* stream) {
  clear_error();
  MP_CHECK_ARG(master && m && v && grad && param_bf16 && n >= 0 && step >= 1, "bad args");
  if (n == 0) return 0;
  float bc1 = 1.f - powf(beta1, (float)step);
  float bc2 = 1.f - powf(beta2, (float)step);
  auto al = [](const void* q, int a) { return reinterpret_cast<uintptr_t>(q) % a == 0; };
  const int64_t n4 = (al(master, 16) && al(m, 16) && al(v, 16) && al(grad, 16) &&
                      al(param_bf16, 8)) ? n / 4 : 0;
  if (n4)
    adam4_kernel<<<grid_for(n4, 256), 256, 0, MP_STREAM(stream)>>>(
        (float4*)master, (float4*)m, (float4*)v, (const float4*)grad, (uint2*)param_bf16, n4, lr,
        beta1, beta2, eps, weight_decay, grad_scale, bc1, bc2);
  if (n - 4 * n4)
    adam_kernel<<<grid_for(n - 4 * n4, 256), 256, 0, MP_STREAM(stream)>>>(
        master + 4 * n4, m + 4 * n4, v + 4 * n4, grad + 4 * n4, (uint16_t*)param_bf16 + 4 * n4,
        n - 4 * n4, lr, beta1, beta2, eps, weight_decay, grad_scale, bc1, bc2);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && y && n >= 0, "bad args");
  if (n == 0) return 0;
  const int64_t n4 = (reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(y) % 8 == 0) ? n / 4 : 0;
  if (n4)
    cast4_f32_bf16_kernel<<<grid_for(n4, 256), 256, 0, MP_STREAM(stream)>>>(
        (const float4*)x, (uint2*)y, n4);
  if (n - 4 * n4)
    cast_f32_bf16_kernel<<<grid_for(n - 4 * n4, 256), 256, 0, MP_STREAM(stream)>>>(
        x + 4 * n4, (uint16_t*)y + 4 * n4, n - 4 * n4);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_cast_bf16_f32(const void* x, float* y, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && y && n >= 0, "bad args");
  if (n == 0) return 0;
  cast_bf16_f32_kernel<<<grid_for(n, 256), 256, 0, MP_STREAM(stream)>>>((const uint16_t*)x, y, n);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_sum_parts_f32(const float* parts, int64_t nparts, int64_t n, float* y, float beta,
                     void* stream) {
  clear_error();
  MP_CHECK_ARG(parts && y && nparts >= 1 && n >= 0 && n % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(parts) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(y) % 16 == 0,
               "bad args (16-byte aligned, n % 4 == 0)");
  if (n == 0) return 0;
  sum_parts_f32_kernel<<<grid_for(n / 4, 256), 256, 0, MP_STREAM(stream)>>>(
      (const float4*)parts, nparts, n / 4, (float4*)y, beta);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_accum_bf16_f32(const void* x, float* y, int64_t n, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && y && n >= 0, "bad args");
  if (n == 0) return 0;
  accum_bf16_f32_kernel<<<grid_for(n, 256), 256, 0, MP_STREAM(stream)>>>((const uint16_t*)x, y, n);
  MP_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
