// Layout adapters of the Wide-ResNet builder (builders.build_wide_resnet,
// binding.py): the IR has no convolution, so a k x k / stride-s
// convolution is an im2col reshape + matmul, stride-2 shortcuts and the stem
// pool are subsampling reshapes, and the head pools with a reduction.
// Activations are NHWC row-major: row = (n*H + y)*W + x, column = channel.
// im2col column order is (ky, kx, c); padding p = k/2 reads zeros.
// All of these move bytes (HBM-bound); the backward forms are gathers, so every
// output element is written once in a fixed summation order (deterministic).
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

// out[(n, oy, ox), (ky, kx, c)] = in[(n, oy*s+ky-p, ox*s+kx-p), c]; V = elements per access
template <int V>
__global__ void im2col_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                              ConvGeom g) {
  const int64_t cv = g.C / V, kk = (int64_t)g.k * g.k;
  const int64_t total = g.N * g.Ho * g.Wo * kk * cv;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    int64_t c = i % cv, r = i / cv;
    int64_t tap = r % kk;
    r /= kk;
    int64_t ox = r % g.Wo, t = r / g.Wo, oy = t % g.Ho, n = t / g.Ho;
    int64_t y = oy * g.s + tap / g.k - g.p, x = ox * g.s + tap % g.k - g.p;
    if (V == 8) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (y >= 0 && y < g.H && x >= 0 && x < g.W)
        v = reinterpret_cast<const uint4*>(in)[((n * g.H + y) * g.W + x) * cv + c];
      reinterpret_cast<uint4*>(out)[i] = v;
    } else {
      uint16_t v = 0;
      if (y >= 0 && y < g.H && x >= 0 && x < g.W) v = in[((n * g.H + y) * g.W + x) * g.C + c];
      out[i] = v;
    }
  }
}

// dx[(n, y, x), c] = sum over taps (ky, kx) with (y + p - ky) = oy*s, (x + p - kx) = ox*s
// in range of dcol[(n, oy, ox), (ky, kx, c)]  (fp32 accumulation, fixed tap order)
__global__ void col2im_kernel(const uint16_t* __restrict__ dcol, uint16_t* __restrict__ dx,
                              ConvGeom g) {
  const int64_t total = g.N * g.H * g.W * g.C, kkc = (int64_t)g.k * g.k * g.C;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    int64_t c = i % g.C, r = i / g.C;
    int64_t x = r % g.W, t = r / g.W, y = t % g.H, n = t / g.H;
    float acc = 0.f;
    for (int ky = 0; ky < g.k; ++ky) {
      int64_t yy = y + g.p - ky;
      if (yy < 0 || yy % g.s) continue;
      int64_t oy = yy / g.s;
      if (oy >= g.Ho) continue;
      for (int kx = 0; kx < g.k; ++kx) {
        int64_t xx = x + g.p - kx;
        if (xx < 0 || xx % g.s) continue;
        int64_t ox = xx / g.s;
        if (ox >= g.Wo) continue;
        acc += bf2f(dcol[((n * g.Ho + oy) * g.Wo + ox) * kkc + (ky * g.k + kx) * g.C + c]);
      }
    }
    dx[i] = f2bf(acc);
  }
}

// out[(n, oy, ox), c] = in[(n, oy*s, ox*s), c]; grad: dx = dy at those pixels, else 0
__global__ void subsample_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                 ConvGeom g, int backward) {
  const int64_t total = backward ? g.N * g.H * g.W * g.C : g.N * g.Ho * g.Wo * g.C;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    int64_t c = i % g.C, r = i / g.C;
    if (!backward) {
      int64_t ox = r % g.Wo, t = r / g.Wo, oy = t % g.Ho, n = t / g.Ho;
      out[i] = in[((n * g.H + oy * g.s) * g.W + ox * g.s) * g.C + c];
    } else {
      int64_t x = r % g.W, t = r / g.W, y = t % g.H, n = t / g.H;
      uint16_t v = 0;
      if (y % g.s == 0 && x % g.s == 0 && y / g.s < g.Ho && x / g.s < g.Wo)
        v = in[((n * g.Ho + y / g.s) * g.Wo + x / g.s) * g.C + c];
      out[i] = v;
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

}  // namespace
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
  if (!backward) {
    bool vec = C % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
               reinterpret_cast<uintptr_t>(out) % 16 == 0;
    int64_t n = N * g.Ho * g.Wo * k * k * (vec ? C / 8 : C);
    if (vec)
      im2col_kernel<8><<<grid_of(n, 256), 256, 0, st>>>((const uint16_t*)x, (uint16_t*)out, g);
    else
      im2col_kernel<1><<<grid_of(n, 256), 256, 0, st>>>((const uint16_t*)x, (uint16_t*)out, g);
  } else {
    col2im_kernel<<<grid_of(N * H * W * C, 256), 256, 0, st>>>((const uint16_t*)x,
                                                               (uint16_t*)out, g);
  }
  MP_CHECK_LAUNCH();
  return 0;
}

int mp_subsample(const void* x, void* out, int64_t N, int64_t H, int64_t W, int64_t C, int s,
                 int backward, void* stream) {
  clear_error();
  MP_CHECK_ARG(x && out && N > 0 && H > 0 && W > 0 && C > 0 && s >= 1, "bad args");
  ConvGeom g = geom(N, H, W, C, 1, s);
  int64_t n = backward ? N * H * W * C : N * g.Ho * g.Wo * C;
  subsample_kernel<<<grid_of(n, 256), 256, 0, MP_STREAM(stream)>>>((const uint16_t*)x,
                                                                   (uint16_t*)out, g, backward);
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
