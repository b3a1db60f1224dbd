// Layout adapters of the Wide-ResNet builder (builders.build_wide_resnet,
// binding.py): the IR has no convolution, so a k x k / stride-s
// convolution is an im2col reshape + matmul, stride-2 shortcuts and the stem
// pool are subsampling reshapes, and the head pools with a reduction.
// Activations are NHWC row-major: row = (n*H + y)*W + x, column = channel.
// im2col column order is (ky, kx, c); padding p = k/2 reads zeros.
// All of these move bytes (HBM-bound); the backward forms are gathers, so every
// output element is written once in a fixed summation order (deterministic).
#include <type_traits>
#include <cstring>
#include "common.cuh"
#include "../../include/mp_exec.h"

#define MP_STREAM(s) reinterpret_cast<cudaStream_t>(s)

namespace mp {
namespace {

inline int grid_of(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads, cap = (int64_t)num_sms() * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

struct ConvGeom {
  int64_t N, H, W, C, Ho, Wo;
  int k, s, p;
};

// out[(n, oy, ox), (ky, kx, c)] = in[(n, oy*s+ky-p, ox*s+kx-p), c]; V = elements per
// access (8: one 16-byte vector when C % 8 == 0).  32-bit index math (element
// counts < 2^31 are checked on the host): the 64-bit div/mod chain made these
// byte-moving kernels instruction-bound.
template <int V>
__global__ void im2col_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                              ConvGeom g) {
  const int cv = (int)(g.C / V), kk = g.k * g.k;
  const int Ho = (int)g.Ho, Wo = (int)g.Wo, H = (int)g.H, W = (int)g.W;
  const int total = (int)(g.N * g.Ho * g.Wo) * kk * cv;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int c = i % cv;
    int r = i / cv;
    const int tap = r % kk;
    r /= kk;
    const int ox = r % Wo, t = r / Wo, oy = t % Ho, n = t / Ho;
    const int ky = tap / g.k, kx = tap - ky * g.k;
    const int y = oy * g.s + ky - g.p, x = ox * g.s + kx - g.p;
    const bool in_img = y >= 0 && y < H && x >= 0 && x < W;
    if (V == 8) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (in_img) v = reinterpret_cast<const uint4*>(in)[((int64_t)(n * H + y) * W + x) * cv + c];
      reinterpret_cast<uint4*>(out)[i] = v;
    } else {
      out[i] = in_img ? in[((int64_t)(n * H + y) * W + x) * g.C + c] : (uint16_t)0;
    }
  }
}

// dx[(n, y, x), c] = sum over taps (ky, kx) with y + p - ky = oy*s, x + p - kx = ox*s
// in range of dcol[(n, oy, ox), (ky, kx, c)]  (fp32 accumulation, fixed tap order;
// 8 channels per thread when C % 8 == 0)
template <int V>
__global__ void col2im_kernel(const uint16_t* __restrict__ dcol, uint16_t* __restrict__ dx,
                              ConvGeom g) {
  const int cv = (int)(g.C / V), kkc = g.k * g.k * (int)g.C;
  const int Ho = (int)g.Ho, Wo = (int)g.Wo, H = (int)g.H, W = (int)g.W;
  const int total = (int)(g.N * g.H * g.W) * cv;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int c = (i % cv) * V;
    const int r = i / cv;
    const int x = r % W, t = r / W, y = t % H, n = t / H;
    float acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f;
    for (int ky = 0; ky < g.k; ++ky) {
      const int yy = y + g.p - ky;
      if (yy < 0 || yy % g.s) continue;
      const int oy = yy / g.s;
      if (oy >= Ho) continue;
      for (int kx = 0; kx < g.k; ++kx) {
        const int xx = x + g.p - kx;
        if (xx < 0 || xx % g.s) continue;
        const int ox = xx / g.s;
        if (ox >= Wo) continue;
        const int64_t off = ((int64_t)(n * Ho + oy) * Wo + ox) * kkc + (ky * g.k + kx) * (int)g.C + c;
        if (V == 8) {
          const uint4 v = *reinterpret_cast<const uint4*>(dcol + off);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[2 * e] += bf2f(w[e] & 0xffff);
            acc[2 * e + 1] += bf2f(w[e] >> 16);
          }
        } else {
          acc[0] += bf2f(dcol[off]);
        }
      }
    }
    if (V == 8) {
      reinterpret_cast<uint4*>(dx)[i] = make_uint4(pack_bf2(acc[0], acc[1]), pack_bf2(acc[2], acc[3]),
                                                   pack_bf2(acc[4], acc[5]), pack_bf2(acc[6], acc[7]));
    } else {
      dx[i] = f2bf(acc[0]);
    }
  }
}

// out[(n, oy, ox), c] = in[(n, oy*s, ox*s), c]; grad: dx = dy at those pixels, else 0
// (V channels per thread: 8 = one 16-byte vector when C % 8 == 0)
template <int V>
__global__ void subsample_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                 ConvGeom g, int backward) {
  using T = typename std::conditional<V == 8, uint4, uint16_t>::type;
  const T* src = reinterpret_cast<const T*>(in);
  T* dst = reinterpret_cast<T*>(out);
  const int cv = (int)(g.C / V);
  const int Ho = (int)g.Ho, Wo = (int)g.Wo, H = (int)g.H, W = (int)g.W;
  const int total = (backward ? (int)(g.N * g.H * g.W) : (int)(g.N * g.Ho * g.Wo)) * cv;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int c = i % cv, r = i / cv;
    if (!backward) {
      const int ox = r % Wo, t = r / Wo, oy = t % Ho, n = t / Ho;
      dst[i] = src[((int64_t)(n * H + oy * g.s) * W + ox * g.s) * cv + c];
    } else {
      const int x = r % W, t = r / W, y = t % H, n = t / H;
      T v;
      memset(&v, 0, sizeof(T));
      if (y % g.s == 0 && x % g.s == 0 && y / g.s < Ho && x / g.s < Wo)
        v = src[((int64_t)(n * Ho + y / g.s) * Wo + x / g.s) * cv + c];
      dst[i] = v;
    }
  }
}

// (A, B, C): reduce_mid out[a, c] = sum_b x[a, b, c]; broadcast_mid out[a, b, c] = x[a, c]
__global__ void reduce_mid_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ out,
                                  int64_t A, int64_t B, int64_t C) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A * C; i += stride) {
    int64_t a = i / C, c = i % C;
    float acc = 0.f;
    for (int64_t b = 0; b < B; ++b) acc += bf2f(x[(a * B + b) * C + c]);
    out[i] = f2bf(acc);
  }
}

__global__ void broadcast_mid_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ out,
                                     int64_t A, int64_t B, int64_t C) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A * B * C; i += stride)
    out[i] = x[(i / (B * C)) * C + i % C];
}

ConvGeom geom(int64_t N, int64_t H, int64_t W, int64_t C, int k, int s) {
  ConvGeom g;
  g.N = N; g.H = H; g.W = W; g.C = C; g.k = k; g.s = s; g.p = k / 2;
  g.Ho = (H + 2 * g.p - k) / s + 1;
  g.Wo = (W + 2 * g.p - k) / s + 1;
  return g;
}


// Force-load this file's kernels (lazy module loading would load a kernel at its
// first launch, which blocks the host while an NCCL kernel spins on the device:
// a deadlock the executor's watchdog could not see).  See mp_preload_kernels.
template <typename F>
static inline int preload_one(F* f) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f)) == cudaSuccess ? 0 : 1;
}
int preload_conv_impl() {
  return preload_one(im2col_kernel<1>) | preload_one(im2col_kernel<8>) |
         preload_one(col2im_kernel<1>) | preload_one(col2im_kernel<8>) |
         preload_one(subsample_kernel<1>) | preload_one(subsample_kernel<8>) |
         preload_one(reduce_mid_kernel) | preload_one(broadcast_mid_kernel);
}
}  // namespace
int preload_conv() { return preload_conv_impl(); }
}  // namespace mp


using namespace mp;

extern "C" {

int mp_im2col(const void* x, void* out, int64_t N, int64_t H, int64_t W, int64_t C, int k, int s,
              int backward, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && out && N > 0 && H > 0 && W > 0 && C > 0 && k >= 1 && (k & 1) && s >= 1,
               "bad args");
  ConvGeom g = geom(N, H, W, C, k, s);
  cudaStream_t st = MP_STREAM(stream);
  MP_CHECK_ARG(N * H * W * C < (1LL << 31) && N * g.Ho * g.Wo * k * k * C < (1LL << 31),
               "tensor too large for 32-bit indexing");
  const bool vec = C % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(out) % 16 == 0;
  if (!backward) {
    int64_t n = N * g.Ho * g.Wo * k * k * (vec ? C / 8 : C);
    if (vec)
      im2col_kernel<8><<<grid_of(n, 256), 256, 0, st>>>((const uint16_t*)x, (uint16_t*)out, g);
    else
      im2col_kernel<1><<<grid_of(n, 256), 256, 0, st>>>((const uint16_t*)x, (uint16_t*)out, g);
  } else {
    int64_t n = N * H * W * (vec ? C / 8 : C);
    if (vec)
      col2im_kernel<8><<<grid_of(n, 256), 256, 0, st>>>((const uint16_t*)x, (uint16_t*)out, g);
    else
      col2im_kernel<1><<<grid_of(n, 256), 256, 0, st>>>((const uint16_t*)x, (uint16_t*)out, g);
  }
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_subsample(const void* x, void* out, int64_t N, int64_t H, int64_t W, int64_t C, int s,
                 int backward, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && out && N > 0 && H > 0 && W > 0 && C > 0 && s >= 1, "bad args");
  ConvGeom g = geom(N, H, W, C, 1, s);
  MP_CHECK_ARG(N * H * W * C < (1LL << 31), "tensor too large for 32-bit indexing");
  const bool vec = C % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(out) % 16 == 0;
  int64_t n = (backward ? N * H * W : N * g.Ho * g.Wo) * (vec ? C / 8 : C);
  if (vec)
    subsample_kernel<8><<<grid_of(n, 256), 256, 0, MP_STREAM(stream)>>>(
        (const uint16_t*)x, (uint16_t*)out, g, backward);
  else
    subsample_kernel<1><<<grid_of(n, 256), 256, 0, MP_STREAM(stream)>>>(
        (const uint16_t*)x, (uint16_t*)out, g, backward);
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_reduce_mid(const void* x, void* out, int64_t A, int64_t B, int64_t C, int broadcast,
                  void* stream) {
  clear_error();
  MP_CHECK_ARG(x && out && A > 0 && B > 0 && C > 0, "bad args");
  cudaStream_t st = MP_STREAM(stream);
  if (!broadcast)
    reduce_mid_kernel<<<grid_of(A * C, 256), 256, 0, st>>>((const uint16_t*)x, (uint16_t*)out, A,
                                                           B, C);
  else
    broadcast_mid_kernel<<<grid_of(A * B * C, 256), 256, 0, st>>>((const uint16_t*)x,
                                                                  (uint16_t*)out, A, B, C);
  MP_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
