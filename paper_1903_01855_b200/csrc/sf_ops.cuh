// sf_ops.cuh — scalar semantics of every elementwise primitive.
//
// This header is the single definition of per-element arithmetic for the
// backend.  It is compiled twice: by nvcc into the ahead-of-time eager
// kernels (libsfb200.so) and, embedded as a string, by NVRTC into the fused
// kernels generated for staged graph functions.  Both compilations use the
// same IEEE flags (-fmad=false, -prec-div=true, -prec-sqrt=true, -ftz=false),
// which is what makes an eager op and the same op inside a fused staged
// kernel produce identical bits — the GPU restatement of the reference's
// "one kernel shared by both execution modes" rule
// (reference: stageflow/kernels.py:1-11).
//
// NumPy edge semantics mirrored here (reference kernels: stageflow/kernels.py):
//   relu      = np.maximum(x, 0): NaN propagates, -0.0 -> +0.0      (:176-177)
//   softplus  = np.logaddexp(0.0, x) incl. its x==0 branch           (:171-173)
//   step_pos  = (x > 0) as float                                     (:180-181)
//   int32 add/sub/mul/neg wrap modulo 2^32                           (:116-153)
//   exp overflow -> inf, log(0) -> -inf, log(<0) -> nan              (:161-168)
#pragma once

#ifndef SF_DEVFN
#define SF_DEVFN __device__ __forceinline__
#endif

// ---- dtype tags (same numbering as the reference wire tags, dtypes.py:63-69)
#define SF_F32 1
#define SF_F64 2
#define SF_I32 3
#define SF_BOOL 4

// ---- opcodes (mirrored in paper_1903_01855_b200/_native.py) ----------------
// unary
#define SF_OP_IDENTITY 0
#define SF_OP_NEG 1
#define SF_OP_EXP 2
#define SF_OP_LOG 3
#define SF_OP_SOFTPLUS 4
#define SF_OP_RELU 5
#define SF_OP_STEP_POS 6
#define SF_OP_TANH 7
#define SF_OP_SQRT 8
#define SF_OP_RSQRT 9
#define SF_OP_SIGMOID 10
#define SF_OP_ABS 11
#define SF_OP_SQUARE 12
#define SF_OP_ISFINITE 13
#define SF_OP_LOGICAL_NOT 14
#define SF_OP_RECIPROCAL 15
#define SF_OP_COS 16
#define SF_OP_SIN 17
// binary
#define SF_OP_ADD 32
#define SF_OP_SUB 33
#define SF_OP_MUL 34
#define SF_OP_DIV 35
#define SF_OP_GREATER 36
#define SF_OP_MAXIMUM 37
#define SF_OP_MINIMUM 38
#define SF_OP_LESS 39
#define SF_OP_EQUAL 40
#define SF_OP_GREATER_EQUAL 41
// ternary
#define SF_OP_SELECT 64

#define SF_OP_IS_BINARY(op) ((op) >= 32 && (op) < 64)
#define SF_OP_IS_TERNARY(op) ((op) >= 64)

namespace sf {

// ------------------------------------------------------------------ float32
SF_DEVFN float neg(float x) { return -x; }
SF_DEVFN float exp_(float x) { return expf(x); }
SF_DEVFN float log_(float x) { return logf(x); }
SF_DEVFN float softplus(float x) {
  // np.logaddexp(0.0, x) (npy_logaddexp with a = 0, b = x)
  if (x == 0.0f) return 0.0f + 0.693147180559945309417232121458176568f;
  const float t = 0.0f - x;
  if (t > 0.0f) return 0.0f + log1pf(expf(x));
  if (t <= 0.0f) return x + log1pf(expf(t));
  return t;  // NaN
}
SF_DEVFN float relu(float x) { return x > 0.0f ? x : (x != x ? x : 0.0f); }
SF_DEVFN float step_pos(float x) { return x > 0.0f ? 1.0f : 0.0f; }
SF_DEVFN float tanh_(float x) { return tanhf(x); }
SF_DEVFN float sqrt_(float x) { return sqrtf(x); }
SF_DEVFN float rsqrt_(float x) { return 1.0f / sqrtf(x); }
SF_DEVFN float sigmoid(float x) { return 1.0f / (1.0f + expf(-x)); }
SF_DEVFN float abs_(float x) { return fabsf(x); }
SF_DEVFN float square(float x) { return x * x; }
SF_DEVFN float recip(float x) { return 1.0f / x; }
SF_DEVFN float cos_(float x) { return cosf(x); }
SF_DEVFN float sin_(float x) { return sinf(x); }
SF_DEVFN bool isfinite_(float x) { return isfinite(x); }
SF_DEVFN float add(float a, float b) { return a + b; }
SF_DEVFN float sub(float a, float b) { return a - b; }
SF_DEVFN float mul(float a, float b) { return a * b; }
SF_DEVFN float div(float a, float b) { return a / b; }
// np.maximum / np.minimum propagate NaN from either side.
SF_DEVFN float maximum(float a, float b) { return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b)); }
SF_DEVFN float minimum(float a, float b) { return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b)); }

// ------------------------------------------------------------------ float64
SF_DEVFN double neg(double x) { return -x; }
SF_DEVFN double exp_(double x) { return exp(x); }
SF_DEVFN double log_(double x) { return log(x); }
SF_DEVFN double softplus(double x) {
  if (x == 0.0) return 0.0 + 0.693147180559945309417232121458176568;
  const double t = 0.0 - x;
  if (t > 0.0) return 0.0 + log1p(exp(x));
  if (t <= 0.0) return x + log1p(exp(t));
  return t;
}
SF_DEVFN double relu(double x) { return x > 0.0 ? x : (x != x ? x : 0.0); }
SF_DEVFN double step_pos(double x) { return x > 0.0 ? 1.0 : 0.0; }
SF_DEVFN double tanh_(double x) { return tanh(x); }
SF_DEVFN double sqrt_(double x) { return sqrt(x); }
SF_DEVFN double rsqrt_(double x) { return 1.0 / sqrt(x); }
SF_DEVFN double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }
SF_DEVFN double abs_(double x) { return fabs(x); }
SF_DEVFN double square(double x) { return x * x; }
SF_DEVFN double recip(double x) { return 1.0 / x; }
SF_DEVFN double cos_(double x) { return cos(x); }
SF_DEVFN double sin_(double x) { return sin(x); }
SF_DEVFN bool isfinite_(double x) { return isfinite(x); }
SF_DEVFN double add(double a, double b) { return a + b; }
SF_DEVFN double sub(double a, double b) { return a - b; }
SF_DEVFN double mul(double a, double b) { return a * b; }
SF_DEVFN double div(double a, double b) { return a / b; }
SF_DEVFN double maximum(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b)); }
SF_DEVFN double minimum(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b)); }

// ------------------------------------------------------------------ int32 (wrapping)
SF_DEVFN int neg(int x) { return (int)(0u - (unsigned)x); }
SF_DEVFN int add(int a, int b) { return (int)((unsigned)a + (unsigned)b); }
SF_DEVFN int sub(int a, int b) { return (int)((unsigned)a - (unsigned)b); }
SF_DEVFN int mul(int a, int b) { return (int)((unsigned)a * (unsigned)b); }
SF_DEVFN int abs_(int x) { return x < 0 ? neg(x) : x; }
SF_DEVFN int square(int x) { return mul(x, x); }
SF_DEVFN int maximum(int a, int b) { return a >= b ? a : b; }
SF_DEVFN int minimum(int a, int b) { return a <= b ? a : b; }
SF_DEVFN int relu(int x) { return x > 0 ? x : 0; }
SF_DEVFN int step_pos(int x) { return x > 0 ? 1 : 0; }
SF_DEVFN bool isfinite_(int) { return true; }

// ------------------------------------------------------------------ generic dispatch
// Used by the AOT eager kernels; the fused code generator calls the named
// functions above directly (same code, so the same bits).
template <class T>
SF_DEVFN T unary_f(int op, T x) {
  switch (op) {
    case SF_OP_IDENTITY: return x;
    case SF_OP_NEG: return neg(x);
    case SF_OP_EXP: return exp_(x);
    case SF_OP_LOG: return log_(x);
    case SF_OP_SOFTPLUS: return softplus(x);
    case SF_OP_RELU: return relu(x);
    case SF_OP_STEP_POS: return step_pos(x);
    case SF_OP_TANH: return tanh_(x);
    case SF_OP_SQRT: return sqrt_(x);
    case SF_OP_RSQRT: return rsqrt_(x);
    case SF_OP_SIGMOID: return sigmoid(x);
    case SF_OP_ABS: return abs_(x);
    case SF_OP_SQUARE: return square(x);
    case SF_OP_RECIPROCAL: return recip(x);
    case SF_OP_COS: return cos_(x);
    case SF_OP_SIN: return sin_(x);
    default: return x;
  }
}
template <>
SF_DEVFN int unary_f<int>(int op, int x) {
  switch (op) {
    case SF_OP_IDENTITY: return x;
    case SF_OP_NEG: return neg(x);
    case SF_OP_ABS: return abs_(x);
    case SF_OP_SQUARE: return square(x);
    case SF_OP_RELU: return relu(x);
    case SF_OP_STEP_POS: return step_pos(x);
    default: return x;
  }
}

template <class T>
SF_DEVFN T binary_f(int op, T a, T b) {
  switch (op) {
    case SF_OP_ADD: return add(a, b);
    case SF_OP_SUB: return sub(a, b);
    case SF_OP_MUL: return mul(a, b);
    case SF_OP_DIV: return div(a, b);
    case SF_OP_MAXIMUM: return maximum(a, b);
    case SF_OP_MINIMUM: return minimum(a, b);
    default: return a;
  }
}
template <>
SF_DEVFN int binary_f<int>(int op, int a, int b) {
  switch (op) {
    case SF_OP_ADD: return add(a, b);
    case SF_OP_SUB: return sub(a, b);
    case SF_OP_MUL: return mul(a, b);
    case SF_OP_MAXIMUM: return maximum(a, b);
    case SF_OP_MINIMUM: return minimum(a, b);
    default: return a;
  }
}

// boolean tensors only support identity/copy and equality
template <>
SF_DEVFN bool unary_f<bool>(int op, bool x) { return x; }
template <>
SF_DEVFN bool binary_f<bool>(int op, bool a, bool b) { return a; }

template <class T>
SF_DEVFN bool compare_f(int op, T a, T b) {
  switch (op) {
    case SF_OP_GREATER: return a > b;
    case SF_OP_LESS: return a < b;
    case SF_OP_EQUAL: return a == b;
    case SF_OP_GREATER_EQUAL: return a >= b;
    default: return false;
  }
}

// ------------------------------------------------------------------ reductions
// Canonical reduction order (CRO), shared by the eager reduce kernel and the
// fused row programs.  For n elements: lane l (0..31) folds x[l], x[l+32],
// x[l+64], ... left to right; the 32 partials are then combined by the xor
// butterfly (offsets 16, 8, 4, 2, 1) and lane 0's value is the result.  An
// empty partial is "absent" (not +0.0), so a single -0.0 sums to -0.0 like
// NumPy.  Longer reductions (n > SF_CRO_CHUNK) first reduce each
// SF_CRO_CHUNK-element chunk with the CRO, then reduce the chunk results
// with the CRO.  NumPy itself sums pairwise; the reference-vs-GPU contract
// for floats is therefore rtol-based (SURVEY.md §7 hard part (i)).
#define SF_CRO_CHUNK 1024

// ------------------------------------------------------------------ RNG
// Philox4x32-10, counter-based: element i of a draw with (seed, offset)
// uses counter (offset + i, 0, 0, 0) and key (seed_lo, seed_hi).  Eager and
// fused kernels evaluate the same function, so eager == staged for the
// device RNG mode.
struct u4 { unsigned x, y, z, w; };
SF_DEVFN u4 philox(unsigned long long ctr, unsigned long long seed) {
  unsigned c0 = (unsigned)ctr, c1 = (unsigned)(ctr >> 32), c2 = 0u, c3 = 0u;
  unsigned k0 = (unsigned)seed, k1 = (unsigned)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  u4 r;
  r.x = c0; r.y = c1; r.z = c2; r.w = c3;
  return r;
}
// uniform in [0, 1)
SF_DEVFN float uniform_f32(unsigned long long ctr, unsigned long long seed) {
  const u4 r = philox(ctr, seed);
  return (float)(r.x >> 8) * 5.9604644775390625e-08f;  // 2^-24
}
SF_DEVFN double uniform_f64(unsigned long long ctr, unsigned long long seed) {
  const u4 r = philox(ctr, seed);
  const unsigned long long m = ((unsigned long long)(r.x >> 5) << 26) | (r.y >> 6);
  return (double)m * 1.1102230246251565e-16;  // 2^-53
}
// standard normal via Box-Muller on two 53-bit uniforms (computed in f64,
// rounded once to the output dtype).
SF_DEVFN double normal_f64(unsigned long long ctr, unsigned long long seed) {
  const u4 r = philox(ctr, seed);
  const unsigned long long m1 = ((unsigned long long)(r.x >> 5) << 26) | (r.y >> 6);
  const unsigned long long m2 = ((unsigned long long)(r.z >> 5) << 26) | (r.w >> 6);
  const double u1 = ((double)m1 + 1.0) * 1.1102230246251565e-16;  // (0, 1]
  const double u2 = (double)m2 * 1.1102230246251565e-16;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// asynchronous global -> shared copy of one 4- or 8-byte element (LDGSTS):
// a row program's uniform operands are all put in flight at once instead of
// one dependent load/store pair per operand; sf::cp_wait() before the barrier.
template <int BYTES>
SF_DEVFN void cp_async(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gmem), "n"(BYTES)
               : "memory");
}
SF_DEVFN void cp_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// One G-byte chunk of a staged operand (elements of W bytes), copied with
// cp.async: a single 16-byte copy when the source is 16-byte aligned.
template <int G, int W>
SF_DEVFN void stage_chunk(unsigned char* dst, const unsigned char* src) {
  if (G == 16 && (((unsigned long long)src) & 15) == 0) {
    cp_async<16>(dst, src);
  } else {
#pragma unroll
    for (int e = 0; e < G / W; ++e) cp_async<W>(dst + W * e, src + W * e);
  }
}

// Volatile shared-memory reads of staged uniform operands.  A row program
// reads the same weights once per network evaluation; plain loads let ptxas
// merge every repeat into one register live across the whole chunk (hundreds
// of weights -> 255 registers + spills, 2 CTAs/SM).  Volatile loads are
// issued where they are used; the v4/v2 forms fetch a matvec weight row.
SF_DEVFN unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
SF_DEVFN float lds(const float* p) {
  float v;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr(p)));
  return v;
}
SF_DEVFN double lds(const double* p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(saddr(p)));
  return v;
}
SF_DEVFN int lds(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(saddr(p)));
  return v;
}
SF_DEVFN bool lds(const bool* p) { return *(const volatile bool*)p; }
SF_DEVFN float4 lds4(const float* p) {
  float4 v;
  asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(saddr(p)));
  return v;
}
SF_DEVFN double2 lds2(const double* p) {
  double2 v;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(saddr(p)));
  return v;
}

// Same loads from a row program's shared-memory pool: base register + a
// compile-time byte offset, so the address folds into the LDS instruction
// (no per-load integer add).
template <class T, int OFF> struct PoolLd;
template <int OFF> struct PoolLd<float, OFF> {
  static SF_DEVFN float ld(unsigned b) {
    float v;
    asm volatile("ld.volatile.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(b), "n"(OFF));
    return v;
  }
};
template <int OFF> struct PoolLd<double, OFF> {
  static SF_DEVFN double ld(unsigned b) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(b), "n"(OFF));
    return v;
  }
};
template <int OFF> struct PoolLd<int, OFF> {
  static SF_DEVFN int ld(unsigned b) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1+%2];" : "=r"(v) : "r"(b), "n"(OFF));
    return v;
  }
};
template <int OFF> struct PoolLd<bool, OFF> {
  static SF_DEVFN bool ld(unsigned b) {
    unsigned short v;
    asm volatile("ld.volatile.shared.u8 %0, [%1+%2];" : "=h"(v) : "r"(b), "n"(OFF));
    return v != 0;
  }
};
template <class T, int OFF>
SF_DEVFN T ldp(unsigned b) { return PoolLd<T, OFF>::ld(b); }
template <int OFF>
SF_DEVFN float4 ldp4(unsigned b) {
  float4 v;
  asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(b), "n"(OFF));
  return v;
}
template <int OFF>
SF_DEVFN double2 ldp2(unsigned b) {
  double2 v;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2+%3];"
               : "=d"(v.x), "=d"(v.y)
               : "r"(b), "n"(OFF));
  return v;
}

// Packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2): two independent IEEE
// round-to-nearest operations in one instruction, bit-identical to the
// scalar add / sub / mul / __fmaf_rn on each half (denormals kept).
// CAUTION: ptxas contracts mul2 followed by add2/sub2 into FFMA2 even under
// -fmad=false; generated code never feeds mul2 into an add (rowfuse.PACK).  Row programs keep adjacent elements of a chain's row in a float2;
// a scalar operand broadcast to both halves (make_float2(s, s)) becomes the
// instruction's .F32 operand form, not a register copy.
SF_DEVFN unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
SF_DEVFN float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
SF_DEVFN float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
SF_DEVFN float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
SF_DEVFN float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
SF_DEVFN float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}

// Row-kernel constant pool (rowfuse.CONST_POOL): a generated row kernel
// declares `__constant__ unsigned char cpool[]` holding its uniform operands
// (weights, biases, per-step stacked uniforms); the plan gathers them there
// before each launch (sf_plan.cpp).  Warp-uniform loads from the constant
// bank become uniform-datapath loads (LDCU) feeding FFMA/FFMA2 through
// uniform-register operands: no per-thread LSU traffic, no shared-memory
// staging prologue.  The loads are volatile asm (kept in program order:
// NVVM otherwise schedules them early and pins hundreds of weights in
// registers, 4.7 KB of spills measured); `dep` (the loop counter inside
// re-rolled loops) and `SITE` (unique per use) make every use distinct.
#ifdef SF_CPOOL
#define SF_CL(NAME, T, PTX, CON)                                                    \
  template <int OFF, int SITE>                                                      \
  SF_DEVFN T NAME(int dep) {                                                        \
    T v;                                                                            \
    asm volatile("ld.const." PTX " %0, [cpool+%1];" : "=" CON(v) : "n"(OFF), "r"(dep), "n"(SITE)); \
    return v;                                                                       \
  }                                                                                 \
  template <int OFF, int SITE>                                                      \
  SF_DEVFN T NAME##s(int stride) {                                                  \
    T v;                                                                            \
    unsigned long long b;                                                           \
    asm("mov.u64 %0, cpool;" : "=l"(b));                                            \
    asm volatile("ld.const." PTX " %0, [%1+%2];" : "=" CON(v) : "l"(b + (unsigned long long)stride), \
        "n"(OFF), "n"(SITE));                                                       \
    return v;                                                                       \
  }
SF_CL(clf, float, "f32", "f")
SF_CL(cld, double, "f64", "d")
SF_CL(cli, int, "s32", "r")
#undef SF_CL
template <int OFF, int SITE>
SF_DEVFN bool clb(int dep) {
  unsigned short v;
  asm volatile("ld.const.u8 %0, [cpool+%1];" : "=h"(v) : "n"(OFF), "r"(dep), "n"(SITE));
  return v != 0;
}
template <int OFF, int SITE>
SF_DEVFN bool clbs(int stride) {
  unsigned short v;
  unsigned long long b;
  asm("mov.u64 %0, cpool;" : "=l"(b));
  asm volatile("ld.const.u8 %0, [%1+%2];" : "=h"(v) : "l"(b + (unsigned long long)stride), "n"(OFF),
      "n"(SITE));
  return v != 0;
}
template <int OFF, int SITE>
SF_DEVFN float4 clf4(int dep) {
  float4 v;
  asm volatile("ld.const.v4.f32 {%0, %1, %2, %3}, [cpool+%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "n"(OFF), "r"(dep), "n"(SITE));
  return v;
}
template <int OFF, int SITE>
SF_DEVFN float4 clf4s(int stride) {
  float4 v;
  unsigned long long b;
  asm("mov.u64 %0, cpool;" : "=l"(b));
  asm volatile("ld.const.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(b + (unsigned long long)stride), "n"(OFF), "n"(SITE));
  return v;
}
template <int OFF, int SITE>
SF_DEVFN double2 cld2(int dep) {
  double2 v;
  asm volatile("ld.const.v2.f64 {%0, %1}, [cpool+%2];" : "=d"(v.x), "=d"(v.y) : "n"(OFF), "r"(dep), "n"(SITE));
  return v;
}
template <int OFF, int SITE>
SF_DEVFN double2 cld2s(int stride) {
  double2 v;
  unsigned long long b;
  asm("mov.u64 %0, cpool;" : "=l"(b));
  asm volatile("ld.const.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v.x), "=d"(v.y)
      : "l"(b + (unsigned long long)stride), "n"(OFF), "n"(SITE));
  return v;
}
#endif  // SF_CPOOL

}  // namespace sf
