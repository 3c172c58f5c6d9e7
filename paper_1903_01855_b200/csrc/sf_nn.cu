// sf_nn.cu — kernels behind the ResNet-50 plugin ops (BASELINE configs C4/C5).
//
// The reference has no convolution, pooling or cross-entropy;
// these ops are registered through its own plugin ABI (nn.py).  Layout is
// NHWC, filters are (KH, KW, Cin, Cout), float32 or float64.
//
//   conv2d            = im2col (this file) + the GEMM of sf_matmul.cu
//   conv2d_grad_input = GEMM (dy @ W^T) + col2im gather (this file)
//   conv2d_grad_filter= GEMM (cols^T @ dy, split-K for long M)
//   max_pool / max_pool_grad, softmax_xent / softmax_xent_grad (this file)
//
// Every reduction here has a fixed order (gathers instead of atomics), so an
// op gives identical bits eagerly and inside a staged program.
#include "sf_internal.h"
#include "sf_ops.cuh"

namespace sfrt {

struct ConvGeom {
  long long n, h, w, c, kh, kw, s, p, ho, wo;
};

static unsigned grid_for_n(Device* d, long long n) {
  long long b = (n + 255) / 256;
  const long long cap = (long long)d->sm_count * 32;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// ---------------------------------------------------------------------------
// Segment kernels (used whenever C is a multiple of the 16-byte vector width
// and the tensors have < 2^31 elements).  In NHWC, one window tap (kh, kw)
// of one output pixel is C contiguous channels in x and C contiguous columns
// in cols, so one warp copies a whole tap with 16-byte vectors and does the
// index arithmetic once per tap (the per-element kernels below spent their
// time in 64-bit divisions: im2col 105 µs at 1.2% of DRAM bandwidth).
// ---------------------------------------------------------------------------
template <class T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

__device__ __forceinline__ void split4(const float4 v, float4& h, float4& l) {
  h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u); l.x = v.x - h.x;
  h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u); l.y = v.y - h.y;
  h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u); l.z = v.z - h.z;
  h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u); l.w = v.w - h.w;
}

// im2col, NHWC, 16-byte vectors: work items are (segment,
// 16-byte vector) pairs flattened over the whole output, and each thread
// keeps UNROLL items' loads in flight before it stores any of them (a
// one-warp-per-segment form left half the warp idle at C = 64 — the
// 3x3 convolutions of layer1 — and waited one HBM round trip per segment:
// ~1.1 TB/s in the ResNet-50 step, profiles/r02e_resnet50_step.md).
template <class T, bool SPLIT, int UNROLL>
__global__ void __launch_bounds__(256) im2col_vec_kernel(const T* __restrict__ x,
                                                         T* __restrict__ out,
                                                         float* __restrict__ lo, ConvGeom g,
                                                         int kp) {
  using V = typename Vec16<T>::type;
  constexpr int VW = Vec16<T>::n;
  const int C = (int)g.c, KW = (int)g.kw, KK = (int)(g.kh * g.kw), K = KK * C;
  const int CV = C / VW, PV = (kp - K) / VW;  // vectors per tap, per K padding
  const int SV = CV > PV ? CV : PV;           // item slots per (row, tap)
  const int taps = KK + (kp > K ? 1 : 0);
  const int WO = (int)g.wo, HO = (int)g.ho, W = (int)g.w, H = (int)g.h;
  const int S = (int)g.s, P = (int)g.p;
  // 32-bit index math throughout (the host checks rows * kp < 2^31): 64-bit
  // divisions made this copy ALU-bound
  const unsigned total = (unsigned)(g.n * g.ho * g.wo) * (unsigned)(taps * SV);
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned base = blockIdx.x * blockDim.x + threadIdx.x; base < total;
       base += stride * UNROLL) {
    V v[UNROLL];
    long long dst[UNROLL];  // element offset of the item in out (-1: none)
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const unsigned i = base + (unsigned)u * stride;
      dst[u] = -1;
      if (i >= total) continue;
      const unsigned sgm = i / (unsigned)SV;
      const int q = (int)(i - sgm * (unsigned)SV);
      const int m = (int)(sgm / (unsigned)taps), t = (int)(sgm - (unsigned)m * (unsigned)taps);
      if (t == KK) {  // K padding: zeros in the first PV vectors of the tap slot
        if (q < PV) {
          memset(&v[u], 0, sizeof(V));
          dst[u] = (long long)m * kp + K + (long long)q * VW;
        }
        continue;
      }
      if (q >= CV) continue;
      const int kh = t / KW, kw = t - kh * KW;
      const int t2 = (int)((unsigned)m / (unsigned)WO), ow = m - t2 * WO;
      const int n = (int)((unsigned)t2 / (unsigned)HO), oh = t2 - n * HO;
      const int ih = oh * S - P + kh, iw = ow * S - P + kw;
      if (ih >= 0 && ih < H && iw >= 0 && iw < W)
        v[u] = reinterpret_cast<const V*>(x + (unsigned)((n * H + ih) * W + iw) * (unsigned)C)[q];
      else
        memset(&v[u], 0, sizeof(V));
      dst[u] = (long long)m * kp + (long long)t * C + (long long)q * VW;
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (dst[u] < 0) continue;
      if constexpr (SPLIT) {
        float4 h, l;
        split4(v[u], h, l);
        *reinterpret_cast<float4*>(out + dst[u]) = h;
        *reinterpret_cast<float4*>(lo + dst[u]) = l;
      } else {
        *reinterpret_cast<V*>(out + dst[u]) = v[u];
      }
    }
  }
}

// dx[n, h, w, c..c+VW) = sum over taps (kh, kw ascending, the order of
// col2im_kernel) of dcols rows; one thread per (pixel, channel vector)
template <class T>
__global__ void col2im_vec_kernel(const T* __restrict__ dcols, T* __restrict__ dx, ConvGeom g) {
  using V = typename Vec16<T>::type;
  constexpr int VW = Vec16<T>::n;
  const int C = (int)g.c, CV = C / VW, KW = (int)g.kw, K = (int)(g.kh * g.kw) * C;
  const int W = (int)g.w, H = (int)g.h, WO = (int)g.wo, HO = (int)g.ho;
  const int S = (int)g.s, P = (int)g.p;
  const int total = (int)(g.n * g.h * g.w) * CV;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int cv = i % CV, pix = i / CV;
    const int w = pix % W, t2 = pix / W;
    const int h = t2 % H, n = t2 / H;
    T acc[VW];
    bool any = false;
    for (int kh = 0; kh < (int)g.kh; ++kh) {
      const int y = h + P - kh;
      if (y < 0 || y % S) continue;
      const int oh = y / S;
      if (oh >= HO) continue;
      for (int kw = 0; kw < KW; ++kw) {
        const int xx = w + P - kw;
        if (xx < 0 || xx % S) continue;
        const int ow = xx / S;
        if (ow >= WO) continue;
        const V v = reinterpret_cast<const V*>(
            dcols + (long long)((n * HO + oh) * WO + ow) * K + (kh * KW + kw) * C)[cv];
        const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int j = 0; j < VW; ++j) acc[j] = any ? sf::add(acc[j], e[j]) : e[j];
        any = true;
      }
    }
    V out;
    T* o = reinterpret_cast<T*>(&out);
#pragma unroll
    for (int j = 0; j < VW; ++j) o[j] = any ? acc[j] : T(0);
    reinterpret_cast<V*>(dx + (long long)pix * C)[cv] = out;
  }
}

// col2im for KH x KW <= 3 x 3 filters: the taps unrolled at compile time, so
// every contributing tap's load is issued before the (in-order) adds — the
// same sum as col2im_vec_kernel (taps kh, kw ascending), without its
// one-dependent-load-per-tap scan (~2.5 TB/s in the ResNet-50 step)
template <class T, int KH, int KW>
__global__ void __launch_bounds__(256) col2im_small_kernel(const T* __restrict__ dcols,
                                                           T* __restrict__ dx, ConvGeom g) {
  using V = typename Vec16<T>::type;
  constexpr int VW = Vec16<T>::n;
  const int C = (int)g.c, CV = C / VW, K = KH * KW * C;
  const int W = (int)g.w, H = (int)g.h, WO = (int)g.wo, HO = (int)g.ho;
  const int S = (int)g.s, P = (int)g.p;
  const int total = (int)(g.n * g.h * g.w) * CV;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int cv = i % CV, pix = i / CV;
    const int w = pix % W, t2 = pix / W;
    const int h = t2 % H, n = t2 / H;
    V buf[KH * KW];
    bool ok[KH * KW];
#pragma unroll
    for (int kh = 0; kh < KH; ++kh) {
#pragma unroll
      for (int kw = 0; kw < KW; ++kw) {
        const int y = h + P - kh, xx = w + P - kw;
        const int oh = y / S, ow = xx / S;
        const bool v = y >= 0 && xx >= 0 && y - oh * S == 0 && xx - ow * S == 0 && oh < HO &&
                       ow < WO;
        ok[kh * KW + kw] = v;
        if (v)
          buf[kh * KW + kw] = reinterpret_cast<const V*>(
              dcols + (long long)((n * HO + oh) * WO + ow) * K + (kh * KW + kw) * C)[cv];
      }
    }
    T acc[VW];
    bool any = false;
#pragma unroll
    for (int t = 0; t < KH * KW; ++t) {
      if (!ok[t]) continue;
      const T* e = reinterpret_cast<const T*>(&buf[t]);
#pragma unroll
      for (int j = 0; j < VW; ++j) acc[j] = any ? sf::add(acc[j], e[j]) : e[j];
      any = true;
    }
    V out;
    T* o = reinterpret_cast<T*>(&out);
#pragma unroll
    for (int j = 0; j < VW; ++j) o[j] = any ? acc[j] : T(0);
    reinterpret_cast<V*>(dx + (long long)pix * C)[cv] = out;
  }
}

static bool seg_ok(const ConvGeom& g, long long kp, int vw) {
  const long long rows = g.n * g.ho * g.wo, pix = g.n * g.h * g.w;
  return g.c % vw == 0 && kp % vw == 0 && rows * kp < (1ll << 31) &&
         pix * g.c < (1ll << 31) && rows * (g.kh * g.kw + 1) < (1ll << 31);
}

// cols[(n, oh, ow), (kh, kw, c)] = x[n, oh*s - p + kh, ow*s - p + kw, c] (0 outside)
template <class T>
__global__ void im2col_kernel(const T* __restrict__ x, T* __restrict__ cols, ConvGeom g) {
  const long long K = g.kh * g.kw * g.c;
  const long long total = g.n * g.ho * g.wo * K;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long k = i % K, m = i / K;
    const long long c = k % g.c, t = k / g.c;
    const long long kw = t % g.kw, kh = t / g.kw;
    const long long ow = m % g.wo, t2 = m / g.wo;
    const long long oh = t2 % g.ho, n = t2 / g.ho;
    const long long ih = oh * g.s - g.p + kh, iw = ow * g.s - g.p + kw;
    T v = T(0);
    if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w) v = x[((n * g.h + ih) * g.w + iw) * g.c + c];
    cols[i] = v;
  }
}

// im2col fused with the 3xTF32 hi/lo split and K padding (row stride kp):
// feeds the tcgen05 GEMM directly (csrc/sf_gemm_tc.cu)
// Raw im2col rows when C is not a multiple of 4 (the 3-channel stem): one
// warp per output row m, the row's pixel decoded once, lanes walk k so every
// store is a coalesced 128-byte line (the element-per-thread kernel below
// re-decoded m for every element and stored with a stride of kp).
__global__ void __launch_bounds__(256) im2col_rows_kernel(const float* __restrict__ x,
                                                          float* __restrict__ out, ConvGeom g,
                                                          int kp) {
  const int C = (int)g.c, KW = (int)g.kw, WO = (int)g.wo, HO = (int)g.ho;
  const int H = (int)g.h, W = (int)g.w, S = (int)g.s, P = (int)g.p;
  const int K = (int)g.kh * KW * C, M = (int)(g.n * g.ho * g.wo);
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int m = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; m < M; m += nwarps) {
    const int t2 = m / WO, ow = m - t2 * WO;
    const int n = t2 / HO, oh = t2 - n * HO;
    const int ih0 = oh * S - P, iw0 = ow * S - P;
    const float* xn = x + (long long)n * H * W * C;
    float* row = out + (long long)m * kp;
    for (int k = lane; k < kp; k += 32) {
      float v = 0.f;
      if (k < K) {
        const int t = k / C, c = k - t * C;
        const int kh = t / KW, kw = t - kh * KW;
        const int ih = ih0 + kh, iw = iw0 + kw;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = xn[(ih * W + iw) * C + c];
      }
      row[k] = v;
    }
  }
}

// I: index type — int (32-bit division, several times cheaper) whenever the
// matrix and the input have < 2^31 elements (every ResNet layer), else long long
template <class I>
__global__ void im2col_split_kernel(const float* __restrict__ x, float* __restrict__ hi,
                                    float* __restrict__ lo, ConvGeom g, long long kp_) {
  const I kp = (I)kp_, C = (I)g.c, KW = (I)g.kw, WO = (I)g.wo, HO = (I)g.ho;
  const I H = (I)g.h, W = (I)g.w, S = (I)g.s, P = (I)g.p;
  const I K = (I)g.kh * KW * C;
  const I total = (I)(g.n * g.ho * g.wo) * kp;
  const I stride = (I)gridDim.x * blockDim.x;
  for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const I m = i / kp, k = i - m * kp;
    float v = 0.f;
    if (k < K) {
      const I t = k / C, c = k - t * C;
      const I kh = t / KW, kw = t - kh * KW;
      const I t2 = m / WO, ow = m - t2 * WO;
      const I n = t2 / HO, oh = t2 - n * HO;
      const I ih = oh * S - P + kh, iw = ow * S - P + kw;
      if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = x[((n * H + ih) * W + iw) * C + c];
    }
    if (lo == nullptr) {  // raw padded cols (the GEMM derives lo in shared memory)
      hi[i] = v;
      continue;
    }
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    hi[i] = h;
    lo[i] = v - h;
  }
}

// dx[n, h, w, c] = sum over (kh, kw) (fixed order) of dcols[(n, oh, ow), (kh, kw, c)]
template <class T>
__global__ void col2im_kernel(const T* __restrict__ dcols, T* __restrict__ dx, ConvGeom g) {
  const long long K = g.kh * g.kw * g.c;
  const long long total = g.n * g.h * g.w * g.c;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long c = i % g.c, t = i / g.c;
    const long long w = t % g.w, t2 = t / g.w;
    const long long h = t2 % g.h, n = t2 / g.h;
    T acc = T(0);
    bool any = false;
    for (long long kh = 0; kh < g.kh; ++kh) {
      const long long y = h + g.p - kh;
      if (y < 0 || y % g.s) continue;
      const long long oh = y / g.s;
      if (oh >= g.ho) continue;
      for (long long kw = 0; kw < g.kw; ++kw) {
        const long long xx = w + g.p - kw;
        if (xx < 0 || xx % g.s) continue;
        const long long ow = xx / g.s;
        if (ow >= g.wo) continue;
        const T v = dcols[((n * g.ho + oh) * g.wo + ow) * K + (kh * g.kw + kw) * g.c + c];
        acc = any ? sf::add(acc, v) : v;
        any = true;
      }
    }
    dx[i] = acc;
  }
}

// max pool, window k x k, stride s, pad p (padding never wins); first max
// in (kh, kw) order is the argmax used by the gradient.
template <class T>
__global__ void maxpool_kernel(const T* __restrict__ x, T* __restrict__ y, ConvGeom g) {
  const long long total = g.n * g.ho * g.wo * g.c;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long c = i % g.c, t = i / g.c;
    const long long ow = t % g.wo, t2 = t / g.wo;
    const long long oh = t2 % g.ho, n = t2 / g.ho;
    T best = T(0);
    bool have = false;
    for (long long kh = 0; kh < g.kh; ++kh) {
      const long long ih = oh * g.s - g.p + kh;
      if (ih < 0 || ih >= g.h) continue;
      for (long long kw = 0; kw < g.kw; ++kw) {
        const long long iw = ow * g.s - g.p + kw;
        if (iw < 0 || iw >= g.w) continue;
        const T v = x[((n * g.h + ih) * g.w + iw) * g.c + c];
        if (!have || v > best || (v != v && best == best)) best = v;
        have = true;
      }
    }
    y[i] = best;
  }
}

// float32, C % 4 == 0, fewer than 2^31 elements: a thread owns 4 channels of
// one output pixel (float4 loads, 32-bit index math); each lane applies
// maxpool_kernel's rule (first maximum in kh, kw order; the first NaN wins),
// so the result is bit-identical.  With write_argmax it stores the window
// position of that maximum instead (maxpool_argmax_kernel's rule).
template <bool ARGMAX>
__global__ void __launch_bounds__(256) maxpool_f32x4_kernel(const float* __restrict__ x,
                                                            float* __restrict__ y,
                                                            signed char* __restrict__ am,
                                                            ConvGeom g) {
  const int C4 = (int)g.c / 4, W = (int)g.w, H = (int)g.h, WO = (int)g.wo, HO = (int)g.ho;
  const int S = (int)g.s, P = (int)g.p, KH = (int)g.kh, KW = (int)g.kw;
  const int total = (int)(g.n * g.ho * g.wo) * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c4 = i % C4, t = i / C4;
    const int ow = t % WO, t2 = t / WO;
    const int oh = t2 % HO, n = t2 / HO;
    float b[4] = {0.f, 0.f, 0.f, 0.f};
    int bi[4] = {-1, -1, -1, -1};
    for (int kh = 0; kh < KH; ++kh) {
      const int ih = oh * S - P + kh;
      if (ih < 0 || ih >= H) continue;
      for (int kw = 0; kw < KW; ++kw) {
        const int iw = ow * S - P + kw;
        if (iw < 0 || iw >= W) continue;
        const float4 v4 = reinterpret_cast<const float4*>(x)[((n * H + ih) * W + iw) * C4 + c4];
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float v = vv[e];
          if (bi[e] < 0 || v > b[e] || (v != v && b[e] == b[e])) {
            b[e] = v;
            bi[e] = kh * KW + kw;
          }
        }
      }
    }
    if (ARGMAX)
      reinterpret_cast<char4*>(am)[i] = make_char4((signed char)bi[0], (signed char)bi[1],
                                                   (signed char)bi[2], (signed char)bi[3]);
    else
      reinterpret_cast<float4*>(y)[i] = make_float4(b[0], b[1], b[2], b[3]);
  }
}

template <class T>
__device__ __forceinline__ bool is_argmax(const T* x, const ConvGeom& g, long long n, long long oh,
                                          long long ow, long long c, long long h, long long w) {
  // recompute the window's first max position and compare with (h, w)
  T best = T(0);
  long long bh = -1, bw = -1;
  for (long long kh = 0; kh < g.kh; ++kh) {
    const long long ih = oh * g.s - g.p + kh;
    if (ih < 0 || ih >= g.h) continue;
    for (long long kw = 0; kw < g.kw; ++kw) {
      const long long iw = ow * g.s - g.p + kw;
      if (iw < 0 || iw >= g.w) continue;
      const T v = x[((n * g.h + ih) * g.w + iw) * g.c + c];
      if (bh < 0 || v > best || (v != v && best == best)) {
        best = v;
        bh = ih;
        bw = iw;
      }
    }
  }
  return bh == h && bw == w;
}

template <class T>
__global__ void maxpool_grad_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                    T* __restrict__ dx, ConvGeom g) {
  const long long total = g.n * g.h * g.w * g.c;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long c = i % g.c, t = i / g.c;
    const long long w = t % g.w, t2 = t / g.w;
    const long long h = t2 % g.h, n = t2 / g.h;
    T acc = T(0);
    bool any = false;
    for (long long kh = 0; kh < g.kh; ++kh) {
      const long long y = h + g.p - kh;
      if (y < 0 || y % g.s) continue;
      const long long oh = y / g.s;
      if (oh >= g.ho) continue;
      for (long long kw = 0; kw < g.kw; ++kw) {
        const long long xx = w + g.p - kw;
        if (xx < 0 || xx % g.s) continue;
        const long long ow = xx / g.s;
        if (ow >= g.wo) continue;
        if (!is_argmax(x, g, n, oh, ow, c, h, w)) continue;
        const T v = dy[((n * g.ho + oh) * g.wo + ow) * g.c + c];
        acc = any ? sf::add(acc, v) : v;
        any = true;
      }
    }
    dx[i] = acc;
  }
}

// Two-phase max-pool gradient for tensors below 2^31 elements (32-bit
// index math).  Phase 1: one thread per window stores the position (kh*kw
// index, -1 if empty) of its first maximum — the same rule as is_argmax.
// Phase 2: one thread per input element gathers dy from the windows whose
// stored argmax is this element, in the same window order (and so the same
// sum) as maxpool_grad_kernel.  9 x-loads per window instead of 36 per
// input element, and no 64-bit divisions (ResNet-50 b32: 1.9 ms -> ~tens of µs).
template <class T>
__global__ void maxpool_argmax_kernel(const T* __restrict__ x, signed char* __restrict__ am,
                                      ConvGeom g) {
  const int C = (int)g.c, W = (int)g.w, H = (int)g.h, WO = (int)g.wo, HO = (int)g.ho;
  const int total = (int)(g.n * g.ho * g.wo * g.c);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % C, t = i / C;
    const int ow = t % WO, t2 = t / WO;
    const int oh = t2 % HO, n = t2 / HO;
    T best = T(0);
    int bi = -1;
    for (int kh = 0; kh < (int)g.kh; ++kh) {
      const int ih = oh * (int)g.s - (int)g.p + kh;
      if (ih < 0 || ih >= H) continue;
      for (int kw = 0; kw < (int)g.kw; ++kw) {
        const int iw = ow * (int)g.s - (int)g.p + kw;
        if (iw < 0 || iw >= W) continue;
        const T v = x[((n * H + ih) * W + iw) * C + c];
        if (bi < 0 || v > best || (v != v && best == best)) {
          best = v;
          bi = kh * (int)g.kw + kw;
        }
      }
    }
    am[i] = (signed char)bi;
  }
}

template <class T>
__global__ void maxpool_gather_kernel(const signed char* __restrict__ am,
                                      const T* __restrict__ dy, T* __restrict__ dx, ConvGeom g) {
  const int C = (int)g.c, W = (int)g.w, H = (int)g.h, WO = (int)g.wo, HO = (int)g.ho;
  const int S = (int)g.s, P = (int)g.p, KW = (int)g.kw;
  const int total = (int)(g.n * g.h * g.w * g.c);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % C, t = i / C;
    const int w = t % W, t2 = t / W;
    const int h = t2 % H, n = t2 / H;
    T acc = T(0);
    bool any = false;
    for (int kh = 0; kh < (int)g.kh; ++kh) {
      const int y = h + P - kh;
      if (y < 0 || y % S) continue;
      const int oh = y / S;
      if (oh >= HO) continue;
      for (int kw = 0; kw < KW; ++kw) {
        const int xx = w + P - kw;
        if (xx < 0 || xx % S) continue;
        const int ow = xx / S;
        if (ow >= WO) continue;
        const int o = ((n * HO + oh) * WO + ow) * C + c;
        if (am[o] != kh * KW + kw) continue;
        const T v = dy[o];
        acc = any ? sf::add(acc, v) : v;
        any = true;
      }
    }
    dx[i] = acc;
  }
}

// The same gather for float32 with C % 4 == 0: a thread owns 4 channels of
// one input pixel (char4 argmax / float4 gradient loads) and visits only the
// windows that contain the pixel, computed from the geometry instead of
// testing all K x K taps with divisions; windows are visited in the order of
// maxpool_gather_kernel (kh, then kw ascending), so sums are bit-identical.
__global__ void __launch_bounds__(256) maxpool_gather_f32x4_kernel(
    const signed char* __restrict__ am, const float* __restrict__ dy, float* __restrict__ dx,
    ConvGeom g) {
  const int C4 = (int)g.c / 4, W = (int)g.w, H = (int)g.h, WO = (int)g.wo, HO = (int)g.ho;
  const int S = (int)g.s, P = (int)g.p, KH = (int)g.kh, KW = (int)g.kw;
  const int total = (int)(g.n * g.h * g.w) * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c4 = i % C4, t = i / C4;
    const int w = t % W, t2 = t / W;
    const int h = t2 % H, n = t2 / H;
    // windows oh with oh*S - P <= h <= oh*S - P + KH - 1; kh = h + P - oh*S
    const int yh = h + P, xw = w + P;
    const int oh_hi = min(HO - 1, yh / S), ow_hi = min(WO - 1, xw / S);
    const int oh_lo = yh - KH + 1 <= 0 ? 0 : (yh - KH + S) / S;
    const int ow_lo = xw - KW + 1 <= 0 ? 0 : (xw - KW + S) / S;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    bool any[4] = {false, false, false, false};
    for (int oh = oh_hi; oh >= oh_lo; --oh) {  // kh ascending
      const int kh = yh - oh * S;
      for (int ow = ow_hi; ow >= ow_lo; --ow) {  // kw ascending
        const int kw = xw - ow * S;
        const int o4 = ((n * HO + oh) * WO + ow) * C4 + c4;
        const char4 m = reinterpret_cast<const char4*>(am)[o4];
        const signed char tap = (signed char)(kh * KW + kw);
        if (m.x != tap && m.y != tap && m.z != tap && m.w != tap) continue;
        const float4 v = reinterpret_cast<const float4*>(dy)[o4];
        const signed char mm[4] = {m.x, m.y, m.z, m.w};
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (mm[e] == tap) {
            a[e] = any[e] ? sf::add(a[e], vv[e]) : vv[e];
            any[e] = true;
          }
      }
    }
    reinterpret_cast<float4*>(dx)[i] = make_float4(a[0], a[1], a[2], a[3]);
  }
}

// softmax cross-entropy per row: loss = log(sum exp(x - m)) + m - x[label];
// one warp per row; the sum follows the canonical reduction order.
template <class T>
__global__ void xent_kernel(const T* __restrict__ logits, const int* __restrict__ labels,
                            long long rows, long long k, T* __restrict__ loss) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += warps) {
    const T* row = logits + r * k;
    T m = -INFINITY;
    for (long long j = lane; j < k; j += 32) m = sf::maximum(m, row[j]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = sf::maximum(m, __shfl_xor_sync(0xffffffffu, m, off));
    T acc = T(0);
    bool present = false;
    for (long long j = lane; j < k; j += 32) {
      const T e = sf::exp_(sf::sub(row[j], m));
      acc = present ? sf::add(acc, e) : e;
      present = true;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const T ov = __shfl_xor_sync(0xffffffffu, acc, off);
      const bool op = __shfl_xor_sync(0xffffffffu, present, off);
      if (present && op) acc = sf::add(acc, ov);
      else if (op) acc = ov;
      present = present || op;
    }
    if (lane == 0) {
      const int lab = labels[r];
      const T picked = (lab >= 0 && lab < k) ? row[lab] : T(NAN);
      loss[r] = sf::sub(sf::add(sf::log_(acc), m), picked);
    }
  }
}

// d logits = g[r] * (softmax - onehot(label))
template <class T>
__global__ void xent_grad_kernel(const T* __restrict__ logits, const int* __restrict__ labels,
                                 const T* __restrict__ g, long long rows, long long k,
                                 T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += warps) {
    const T* row = logits + r * k;
    T m = -INFINITY;
    for (long long j = lane; j < k; j += 32) m = sf::maximum(m, row[j]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = sf::maximum(m, __shfl_xor_sync(0xffffffffu, m, off));
    T acc = T(0);
    bool present = false;
    for (long long j = lane; j < k; j += 32) {
      const T e = sf::exp_(sf::sub(row[j], m));
      acc = present ? sf::add(acc, e) : e;
      present = true;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const T ov = __shfl_xor_sync(0xffffffffu, acc, off);
      const bool op = __shfl_xor_sync(0xffffffffu, present, off);
      if (present && op) acc = sf::add(acc, ov);
      else if (op) acc = ov;
      present = present || op;
    }
    const int lab = labels[r];
    const T gr = g ? g[r] : T(1);
    for (long long j = lane; j < k; j += 32) {
      const T p = sf::div(sf::exp_(sf::sub(row[j], m)), acc);
      out[r * k + j] = sf::mul(gr, j == lab ? sf::sub(p, T(1)) : p);
    }
  }
}

template <class F>
static int by_dtype(int dtype, F&& f) {
  if (dtype == SF_DTYPE_F32) return f(float());
  if (dtype == SF_DTYPE_F64) return f(double());
  set_error("nn ops require float tensors");
  return SF_ERR_INVALID;
}

}  // namespace sfrt

using namespace sfrt;

static ConvGeom geom(const int64_t* g) {
  ConvGeom c;
  c.n = g[0]; c.h = g[1]; c.w = g[2]; c.c = g[3]; c.kh = g[4]; c.kw = g[5]; c.s = g[6]; c.p = g[7];
  c.ho = (c.h + 2 * c.p - c.kh) / c.s + 1;
  c.wo = (c.w + 2 * c.p - c.kw) / c.s + 1;
  return c;
}

extern "C" {

// g = {N, H, W, C, KH, KW, stride, pad}
int sf_im2col(int dev, int dtype, const int64_t* g8, const void* x, void** cols) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  const ConvGeom g = geom(g8);
  const long long total = g.n * g.ho * g.wo * g.kh * g.kw * g.c;
  if (*cols == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)total * dtype_size(dtype), cols));
  if (total == 0) return SF_OK;
  count_launch(dev);
  return by_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    const long long K = g.kh * g.kw * g.c;
    if (seg_ok(g, K, 16 / (int)sizeof(T))) {
      const long long items = g.n * g.ho * g.wo * g.kh * g.kw * (g.c / (16 / (long long)sizeof(T)));
      im2col_vec_kernel<T, false, 4><<<grid_for_n(d, (items + 3) / 4), 256, 0, d->stream>>>(
          (const T*)x, (T*)*cols, nullptr, g, (int)K);
    } else {
      im2col_kernel<T><<<grid_for_n(d, total), 256, 0, d->stream>>>((const T*)x, (T*)*cols, g);
    }
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  });
}

int sf_im2col_split(int dev, const int64_t* g8, int64_t kp, const void* x, void** hi, void** lo) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  const ConvGeom g = geom(g8);
  const long long total = g.n * g.ho * g.wo * kp;
  if (*hi == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)total * 4, hi));
  // lo == NULL: raw fp32 cols, K padded to kp, no lo part (for GEMMs that
  // derive lo in shared memory)
  if (lo && *lo == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)total * 4, lo));
  if (total == 0) return SF_OK;
  count_launch(dev);
  if (seg_ok(g, kp, 4)) {
    const long long K = g.kh * g.kw * g.c;
    const long long taps = g.kh * g.kw + (kp > K ? 1 : 0);
    const long long sv = g.c / 4 > (kp - K) / 4 ? g.c / 4 : (kp - K) / 4;
    const long long items = g.n * g.ho * g.wo * taps * sv;
    const unsigned grid = grid_for_n(d, (items + 3) / 4);
    if (lo)
      im2col_vec_kernel<float, true, 4><<<grid, 256, 0, d->stream>>>(
          (const float*)x, (float*)*hi, (float*)*lo, g, (int)kp);
    else
      im2col_vec_kernel<float, false, 4><<<grid, 256, 0, d->stream>>>(
          (const float*)x, (float*)*hi, nullptr, g, (int)kp);
  } else if (!lo && total < (1ll << 31) - (1ll << 24) && g.n * g.h * g.w * g.c < (1ll << 31)) {
    im2col_rows_kernel<<<grid_for_n(d, g.n * g.ho * g.wo * 32), 256, 0, d->stream>>>(
        (const float*)x, (float*)*hi, g, (int)kp);
  } else if (total < (1ll << 31) - (1ll << 24) && g.n * g.h * g.w * g.c < (1ll << 31)) {
    im2col_split_kernel<int><<<grid_for_n(d, total), 256, 0, d->stream>>>(
        (const float*)x, (float*)*hi, lo ? (float*)*lo : nullptr, g, kp);
  } else {
    im2col_split_kernel<long long><<<grid_for_n(d, total), 256, 0, d->stream>>>(
        (const float*)x, (float*)*hi, lo ? (float*)*lo : nullptr, g, kp);
  }
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

int sf_col2im(int dev, int dtype, const int64_t* g8, const void* dcols, void** dx) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  const ConvGeom g = geom(g8);
  const long long total = g.n * g.h * g.w * g.c;
  if (*dx == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)total * dtype_size(dtype), dx));
  if (total == 0) return SF_OK;
  count_launch(dev);
  return by_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    constexpr int vw = 16 / (int)sizeof(T);
    if (seg_ok(g, g.kh * g.kw * g.c, vw)) {
      const unsigned grid = grid_for_n(d, total / vw);
      if (g.kh == 3 && g.kw == 3)
        col2im_small_kernel<T, 3, 3><<<grid, 256, 0, d->stream>>>((const T*)dcols, (T*)*dx, g);
      else if (g.kh == 1 && g.kw == 1)
        col2im_small_kernel<T, 1, 1><<<grid, 256, 0, d->stream>>>((const T*)dcols, (T*)*dx, g);
      else
        col2im_vec_kernel<T><<<grid, 256, 0, d->stream>>>((const T*)dcols, (T*)*dx, g);
    } else {
      col2im_kernel<T><<<grid_for_n(d, total), 256, 0, d->stream>>>((const T*)dcols, (T*)*dx, g);
    }
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  });
}

int sf_maxpool2d(int dev, int dtype, const int64_t* g8, const void* x, void** y) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  const ConvGeom g = geom(g8);
  const long long total = g.n * g.ho * g.wo * g.c;
  if (*y == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)total * dtype_size(dtype), y));
  if (total == 0) return SF_OK;
  count_launch(dev);
  return by_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    if (std::is_same<T, float>::value && g.c % 4 == 0 && g.n * g.h * g.w * g.c < (1ll << 31))
      maxpool_f32x4_kernel<false><<<grid_for_n(d, total / 4), 256, 0, d->stream>>>(
          (const float*)x, (float*)*y, nullptr, g);
    else
      maxpool_kernel<T><<<grid_for_n(d, total), 256, 0, d->stream>>>((const T*)x, (T*)*y, g);
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  });
}

int sf_maxpool2d_grad(int dev, int dtype, const int64_t* g8, const void* x, const void* dy,
                      void** dx) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  const ConvGeom g = geom(g8);
  const long long total = g.n * g.h * g.w * g.c;
  if (*dx == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)total * dtype_size(dtype), dx));
  if (total == 0) return SF_OK;
  const long long outs = g.n * g.ho * g.wo * g.c;
  if (total < (1ll << 31) && outs < (1ll << 31) && g.kh * g.kw <= 127) {
    signed char* am = nullptr;
    SF_TRY(d->alloc.alloc(dev, (size_t)outs, (void**)&am));
    count_launch(dev, 2);
    const int st = by_dtype(dtype, [&](auto t) {
      using T = decltype(t);
      if (std::is_same<T, float>::value && g.c % 4 == 0)
        maxpool_f32x4_kernel<true><<<grid_for_n(d, outs / 4), 256, 0, d->stream>>>(
            (const float*)x, nullptr, am, g);
      else
        maxpool_argmax_kernel<T><<<grid_for_n(d, outs), 256, 0, d->stream>>>((const T*)x, am, g);
      if (std::is_same<T, float>::value && g.c % 4 == 0)
        maxpool_gather_f32x4_kernel<<<grid_for_n(d, total / 4), 256, 0, d->stream>>>(
            am, (const float*)dy, (float*)*dx, g);
      else
        maxpool_gather_kernel<T><<<grid_for_n(d, total), 256, 0, d->stream>>>(
            am, (const T*)dy, (T*)*dx, g);
      SF_CHECK_CUDA(cudaGetLastError());
      return SF_OK;
    });
    d->alloc.release(am);  // stream-ordered reuse is safe
    return st;
  }
  count_launch(dev);
  return by_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    maxpool_grad_kernel<T><<<grid_for_n(d, total), 256, 0, d->stream>>>(
        (const T*)x, (const T*)dy, (T*)*dx, g);
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  });
}

int sf_softmax_xent(int dev, int dtype, int64_t rows, int64_t k, const void* logits,
                    const void* labels, void** loss) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (*loss == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)rows * dtype_size(dtype), loss));
  if (rows == 0) return SF_OK;
  count_launch(dev);
  return by_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    xent_kernel<T><<<grid_for_n(d, rows * 32), 256, 0, d->stream>>>(
        (const T*)logits, (const int*)labels, rows, k, (T*)*loss);
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  });
}

int sf_softmax_xent_grad(int dev, int dtype, int64_t rows, int64_t k, const void* logits,
                         const void* labels, const void* g, void** out) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (*out == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)(rows * k) * dtype_size(dtype), out));
  if (rows == 0) return SF_OK;
  count_launch(dev);
  return by_dtype(dtype, [&](auto t) {
    using T = decltype(t);
    xent_grad_kernel<T><<<grid_for_n(d, rows * 32), 256, 0, d->stream>>>(
        (const T*)logits, (const int*)labels, (const T*)g, rows, k, (T*)*out);
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  });
}

}  // extern "C"
