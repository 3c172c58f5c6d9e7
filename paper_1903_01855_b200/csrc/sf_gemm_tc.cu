// sf_gemm_tc.cu — fp32-accurate GEMM on the 5th-generation tensor cores.
//
// C[M,N] (fp32, row-major) = A[M,K] . B[N,K]^T, computed as 3xTF32:
// A.B ~= Ahi.Bhi + Ahi.Blo + Alo.Bhi  where hi = x with the low 13 mantissa
// bits cleared (exactly representable in TF32) and lo = x - hi (exact in
// fp32).  Relative error ~2^-22, i.e. fp32 class — what the ResNet-50
// convolutions need to meet the rtol 1e-4 contract against the reference's
// numpy/OpenBLAS arithmetic.  The tensor cores ignore an fp32 operand's low
// 13 mantissa bits, so the unsplit matrix serves as hi; only lo is stored.
//
// gemm_tc_persistent: one CTA (6 warps) per SM walks the output tiles
//   warp 0 / lane 0 : TMA producer — 4 tiles (Ahi, Alo, Bhi, Blo) per k-block
//                     into a 3-stage ring of swizzled smem, mbarrier
//                     full/empty handshakes
//   warp 1 / lane 0 : MMA issuer — tcgen05.mma.cta_group::1.kind::tf32, 3
//                     passes x 4 k-steps per k-block into a double-buffered
//                     TMEM accumulator; tcgen05.commit releases smem slots
//   warps 2-5       : epilogue — tcgen05.ld 32x32b from their TMEM lane
//                     quarter, float4 stores to C, overlapping the next
//                     tile's MMAs
// Operands may be K-major (128B swizzle) or MN-major (128B swizzle with 32B
// atoms, the only MN-major tf32 layout UMMA accepts).
#include <cudaTypedefs.h>

#include "sf_internal.h"

namespace sfrt {

static constexpr int TC_BM = 128, TC_BK = 32, TC_STAGES = 3;
// smem ring depth: 64 KB stages (BN = 128) fit 3, 48 KB stages (BN = 64) fit 4
// (BN = 256: 96 KB stages, 2 fit; each 128x256x8 MMA reads 12 KB of shared
// memory per 128 tensor cycles vs 8 KB per 64 at BN = 128 — 25% less operand
// traffic per MAC on the pipe that bounds the 3xTF32 passes)
template <int BN>
struct TcStages {
  static constexpr int n = BN <= 64 ? 4 : (BN <= 128 ? 3 : 2);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "SF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra SF_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand tile, rows of 128 bytes (32 fp32), 128B swizzle: 8-row
// core groups 1024 bytes apart (SBO); LBO unused; descriptor version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// MN-major operand.  For 32-bit (tf32) MN-major operands the only smem
// layout UMMA accepts is "128B swizzle with 32B atoms" (descriptor layout
// type 1, SWIZZLE_128B_BASE32B; TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B):
// the plain 128B swizzle makes the MMA read zeros (measured,
// tools/dev/mn_mma_test.cu).  A tile is MN-chunks of 32 fp32 (128 B) by the
// k-block's 32 K rows, each chunk one 32x32 TMA box (4096 B): chunks LBO =
// 4096 B apart, 4-row K groups SBO = 512 B apart (CuTe canonical
// Swizzle<2,5,2> o ((8,n),(4,k)):((1,LBO),(4,SBO)) in 16-byte units).  One
// UMMA_K = 8 rows, so k-step j starts 1024 * j bytes in.
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(4096u >> 4) << 16;
  d |= (uint64_t)(512u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)1u << 61;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// tf32 split of 4 values: *h = x with the low 13 mantissa bits cleared
// (what the tensor core reads of x), returns lo = x - hi (exact in fp32)
__device__ __forceinline__ float4 tf32_lo4(float4 v, float4* h) {
  const unsigned m = 0xFFFFE000u;
  h->x = __uint_as_float(__float_as_uint(v.x) & m);
  h->y = __uint_as_float(__float_as_uint(v.y) & m);
  h->z = __uint_as_float(__float_as_uint(v.z) & m);
  h->w = __uint_as_float(__float_as_uint(v.w) & m);
  return make_float4(v.x - h->x, v.y - h->y, v.z - h->z, v.w - h->w);
}

// Persistent variant: one CTA per SM walks the output tiles (and split-K
// slices) round-robin.  Six warps:
//   warp 0 lane 0: TMA producer over a TC_STAGES ring shared by all tiles
//   warp 1 lane 0: MMA issuer; the accumulator is DOUBLE-BUFFERED in TMEM
//                  (2 x BN columns), so the MMAs of tile i+1 run while the
//                  epilogue drains tile i
//   warps 2-5    : epilogue; warp w reads TMEM lane quarter (w % 4)
// mbarriers: full/empty per smem stage; acc_full/acc_empty per TMEM buffer.
// Per tile the MMA sequence (3 passes x k-steps, in k order) is fixed, so a
// result does not depend on the tile schedule or the operand majorness.
// AMN / BMN: operand stored MN-major (the GEMM's M / N index contiguous,
// e.g. A = cols^T of a weight-gradient GEMM read straight from cols): it is
// loaded as 32x32 boxes and described with sw128_mn_desc, so no transposed
// copy is ever made.
// lo_a_smem / lo_b_smem: that operand's lo part is not read from HBM — the
// four converter warps (6-9) derive it in shared memory from the TMA-loaded
// fp32 tile (lo = x - tf32(x), elementwise, so the swizzled layout carries
// over unchanged), halving the operand bytes the TMA moves per k-block and
// making the separate split pass unnecessary.  The MMA issuer then waits on
// the converters' barrier instead of the TMA's.
// Implicit-GEMM convolution geometry (GATHER): A = im2col(x) of an NHWC
// input with C % 32 == 0 is never materialised — the producer warp gathers
// each 128-row x 32-k A tile (32 channels of one filter tap for 128 output
// pixels) straight from x with 16-byte cp.async into the same 128B-swizzled
// layout the TMA would have written (zero-filled outside the image).
struct GatherGeom {
  const float* x;
  int h, w, c, kw, s, p, wo, howo;
  int tma;    // 1: A tiles come from a TMA im2col map (passed as tAhi), one copy per k-block
  int n, kh;  // (host, for the im2col map)
};

__device__ __forceinline__ void tma_load_im2col(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c, int w, int h, int n, uint16_t ow,
                                                uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c), "r"(w), "r"(h), "r"(n), "r"(smem_u32(bar)), "h"(ow), "h"(oh)
      : "memory");
}

template <int BN, bool AMN, bool BMN, bool GATHER = false>
__global__ void __launch_bounds__(320, 1)
    gemm_tc_persistent(const __grid_constant__ CUtensorMap tAhi,
                       const __grid_constant__ CUtensorMap tAlo,
                       const __grid_constant__ CUtensorMap tBhi,
                       const __grid_constant__ CUtensorMap tBlo,
                       const __grid_constant__ CUtensorMap tC, float* __restrict__ C, int M,
                       int N, int K, int kb_per_split, int tiles_n, int tiles_mn, int n_tiles,
                       int lo_a_smem, int lo_b_smem, int tma_c, const GatherGeom gg) {
  constexpr int TC_STAGES = TcStages<BN>::n;  // shadows the default ring depth
  constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4, B_BYTES = BN * TC_BK * 4;
  constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + TC_STAGES * STAGE_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* acc_full = empty + TC_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* conv = acc_empty + 2;
  uint32_t* tmem_slot = (uint32_t*)(conv + TC_STAGES);
  const bool any_lo = lo_a_smem || lo_b_smem;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      // GATHER: the producer lane's expect_tx + one cp.async completion
      // arrival per producer lane
      mbar_init(&full[s], GATHER && !gg.tma ? 33 : 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int nk_all = (K + TC_BK - 1) / TC_BK;

  if (GATHER && gg.tma && warp == 0) {
    // TMA im2col: one 128-pixel x 32-channel box per k-block; the hardware
    // walks the output pixels (W, then H, then N) inside the bounding box
    // and zero-fills outside the image
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int z = t / tiles_mn, mn = t - z * tiles_mn;
        const int m0 = (mn / tiles_n) * TC_BM, n0 = (mn % tiles_n) * BN;
        const int kb0 = z * kb_per_split;
        const int kb1 = kb0 + kb_per_split < nk_all ? kb0 + kb_per_split : nk_all;
        const int n = m0 / gg.howo, rem = m0 - n * gg.howo;
        const int oh = rem / gg.wo, ow = rem - oh * gg.wo;
        const int w0 = ow * gg.s - gg.p, h0 = oh * gg.s - gg.p;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % TC_STAGES;
          if (g >= TC_STAGES) mbar_wait(&empty[s], ((g / TC_STAGES) & 1u) ^ 1u);
          uint8_t* st = smem + s * STAGE_BYTES;
          const int kx = kb * TC_BK;
          const int tap = kx / gg.c, c0 = kx - tap * gg.c;
          const int kh = tap / gg.kw, kw = tap - kh * gg.kw;
          mbar_expect_tx(&full[s], A_BYTES + (lo_b_smem ? B_BYTES : 2 * B_BYTES));
          tma_load_im2col(st, &tAhi, &full[s], c0, w0, h0, n, (uint16_t)kw, (uint16_t)kh);
          if constexpr (BMN) {
#pragma unroll
            for (int jj = 0; jj < BN / 32; ++jj) {
              tma_load_2d(st + 2 * A_BYTES + 4096 * jj, &tBhi, &full[s], n0 + 32 * jj, kx);
              if (!lo_b_smem)
                tma_load_2d(st + 2 * A_BYTES + B_BYTES + 4096 * jj, &tBlo, &full[s],
                            n0 + 32 * jj, kx);
            }
          } else {
            tma_load_2d(st + 2 * A_BYTES, &tBhi, &full[s], kx, n0);
            if (!lo_b_smem) tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tBlo, &full[s], kx, n0);
          }
        }
      }
    }
  } else if (GATHER && warp == 0) {
    // all 32 lanes gather A (lane l: 16-byte chunk l % 8 of rows l / 8 + 4 i);
    // lane 0 also loads B with the TMA
    uint32_t g = 0;
    const int j = lane & 7;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int z = t / tiles_mn, mn = t - z * tiles_mn;
      const int m0 = (mn / tiles_n) * TC_BM, n0 = (mn % tiles_n) * BN;
      const int kb0 = z * kb_per_split;
      const int kb1 = kb0 + kb_per_split < nk_all ? kb0 + kb_per_split : nk_all;
      int base[32], hw[32];  // pixel index of tap (0, 0); (ih0 << 16) | (iw0 & 0xffff)
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int m = m0 + (lane >> 3) + 4 * i;
        if (m < M) {
          const int n = m / gg.howo, rem = m - n * gg.howo;
          const int oh = rem / gg.wo, ow = rem - oh * gg.wo;
          const int ih0 = oh * gg.s - gg.p, iw0 = ow * gg.s - gg.p;
          base[i] = (n * gg.h + ih0) * gg.w + iw0;
          hw[i] = (ih0 << 16) | (iw0 & 0xffff);
        } else {
          base[i] = 0;
          hw[i] = (int)(0x80000000u);  // ih0 = -32768: never inside the image
        }
      }
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % TC_STAGES;
        if (g >= TC_STAGES) mbar_wait(&empty[s], ((g / TC_STAGES) & 1u) ^ 1u);
        uint8_t* st = smem + s * STAGE_BYTES;
        const int kx = kb * TC_BK;
        if (lane == 0) {
          mbar_expect_tx(&full[s], lo_b_smem ? B_BYTES : 2 * B_BYTES);
          if constexpr (BMN) {
#pragma unroll
            for (int jj = 0; jj < BN / 32; ++jj) {
              tma_load_2d(st + 2 * A_BYTES + 4096 * jj, &tBhi, &full[s], n0 + 32 * jj, kx);
              if (!lo_b_smem)
                tma_load_2d(st + 2 * A_BYTES + B_BYTES + 4096 * jj, &tBlo, &full[s],
                            n0 + 32 * jj, kx);
            }
          } else {
            tma_load_2d(st + 2 * A_BYTES, &tBhi, &full[s], kx, n0);
            if (!lo_b_smem) tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tBlo, &full[s], kx, n0);
          }
        }
        const int tap = kx / gg.c, c0 = kx - tap * gg.c;
        const int kh = tap / gg.kw, kw = tap - kh * gg.kw;
        const float* xs = gg.x + c0 + 4 * j;
        const int off = kh * gg.w + kw;
        const uint32_t sa = smem_u32(st);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int r = (lane >> 3) + 4 * i;
          const int ih = (hw[i] >> 16) + kh, iw = (int)(short)(hw[i] & 0xffff) + kw;
          const bool ok = (unsigned)ih < (unsigned)gg.h && (unsigned)iw < (unsigned)gg.w;
          const float* src = ok ? xs + (long long)(base[i] + off) * gg.c : gg.x;
          const uint32_t dst = sa + (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                       "r"(ok ? 16 : 0)
                       : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         smem_u32(&full[s]))
                     : "memory");
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      uint32_t g = 0;  // k-blocks issued so far (all tiles): ring position
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int z = t / tiles_mn, mn = t - z * tiles_mn;
        const int m0 = (mn / tiles_n) * TC_BM, n0 = (mn % tiles_n) * BN;
        const int kb0 = z * kb_per_split;
        const int kb1 = kb0 + kb_per_split < nk_all ? kb0 + kb_per_split : nk_all;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % TC_STAGES;
          if (g >= TC_STAGES) mbar_wait(&empty[s], ((g / TC_STAGES) & 1u) ^ 1u);
          uint8_t* st = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], (lo_a_smem ? A_BYTES : 2 * A_BYTES) +
                                       (lo_b_smem ? B_BYTES : 2 * B_BYTES));
          const int kx = kb * TC_BK;
          if constexpr (AMN) {
#pragma unroll
            for (int j = 0; j < TC_BM / 32; ++j) {
              tma_load_2d(st + 4096 * j, &tAhi, &full[s], m0 + 32 * j, kx);
              if (!lo_a_smem)
                tma_load_2d(st + A_BYTES + 4096 * j, &tAlo, &full[s], m0 + 32 * j, kx);
            }
          } else {
            tma_load_2d(st, &tAhi, &full[s], kx, m0);
            if (!lo_a_smem) tma_load_2d(st + A_BYTES, &tAlo, &full[s], kx, m0);
          }
          if constexpr (BMN) {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) {
              tma_load_2d(st + 2 * A_BYTES + 4096 * j, &tBhi, &full[s], n0 + 32 * j, kx);
              if (!lo_b_smem)
                tma_load_2d(st + 2 * A_BYTES + B_BYTES + 4096 * j, &tBlo, &full[s],
                            n0 + 32 * j, kx);
            }
          } else {
            tma_load_2d(st + 2 * A_BYTES, &tBhi, &full[s], kx, n0);
            if (!lo_b_smem) tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tBlo, &full[s], kx, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) |
                             ((BMN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);
      uint32_t g = 0;
      int i = 0;  // local tile count
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int z = t / tiles_mn;
        const int kb0 = z * kb_per_split;
        const int kb1 = kb0 + kb_per_split < nk_all ? kb0 + kb_per_split : nk_all;
        const int b = i & 1;
        if (i >= 2) mbar_wait(&acc_empty[b], ((uint32_t)(i >> 1) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + (uint32_t)(b * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % TC_STAGES;
          mbar_wait(&full[s], (g / TC_STAGES) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t a_hi = base, a_lo = base + A_BYTES;
          const uint32_t b_hi = base + 2 * A_BYTES, b_lo = base + 2 * A_BYTES + B_BYTES;
          const uint32_t pa[3] = {a_hi, a_hi, a_lo};
          const uint32_t pb[3] = {b_hi, b_lo, b_hi};
          if (GATHER) {
            // the A tile came through cp.async (generic proxy; its completion
            // is observed through the full barrier): order it before this
            // thread's async-proxy (tensor core) reads
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          }
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            if (pass == 1 && any_lo) {
              // hi.hi needs only the TMA'd tiles and is already issued; the
              // passes reading lo wait for the converters (their work hides
              // behind the tensor core's pass 0)
              mbar_wait(&conv[s], (g / TC_STAGES) & 1u);
              asm volatile("tcgen05.fence::after_thread_sync;");
            }
#pragma unroll
            for (int j = 0; j < TC_BK / 8; ++j) {
              const uint64_t da = AMN ? sw128_mn_desc(pa[pass] + 1024u * j)
                                      : sw128_desc(pa[pass] + 32u * j);
              const uint64_t db = BMN ? sw128_mn_desc(pb[pass] + 1024u * j)
                                      : sw128_desc(pb[pass] + 32u * j);
              mma_tf32(acc, da, db, idesc, ((kb - kb0) | pass | j) != 0);
            }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[b]);
      }
    }
  } else if (warp >= 6) {
    // converter warps 6..9: lo parts of the stage's tiles, in ring order
    if (any_lo) {
      const int ct = threadIdx.x - 192;  // 0..127
      uint32_t g = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int z = t / tiles_mn;
        const int kb0 = z * kb_per_split;
        const int kb1 = kb0 + kb_per_split < nk_all ? kb0 + kb_per_split : nk_all;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % TC_STAGES;
          mbar_wait(&full[s], (g / TC_STAGES) & 1u);
          uint8_t* st = smem + s * STAGE_BYTES;
          // shared-window addressing (ld/st.shared, not generic LD/ST)
          if (lo_a_smem) {
            const uint32_t hi = smem_u32(st), lo = hi + A_BYTES;
            float4 v[A_BYTES / 16 / 128];
#pragma unroll
            for (int i = 0; i < (int)(A_BYTES / 16 / 128); ++i) v[i] = lds128(hi + (ct + 128 * i) * 16);
#pragma unroll
            for (int i = 0; i < (int)(A_BYTES / 16 / 128); ++i) {
              float4 h;
              sts128(lo + (ct + 128 * i) * 16, tf32_lo4(v[i], &h));
            }
          }
          if (lo_b_smem) {
            const uint32_t hi = smem_u32(st + 2 * A_BYTES), lo = hi + B_BYTES;
            float4 v[B_BYTES / 16 / 128];
#pragma unroll
            for (int i = 0; i < (int)(B_BYTES / 16 / 128); ++i) v[i] = lds128(hi + (ct + 128 * i) * 16);
#pragma unroll
            for (int i = 0; i < (int)(B_BYTES / 16 / 128); ++i) {
              float4 h;
              sts128(lo + (ct + 128 * i) * 16, tf32_lo4(v[i], &h));
            }
          }
          // generic-proxy smem writes -> visible to the tensor core (async proxy)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[s]);
        }
      }
    }
  } else {
    // epilogue warps 2..5: TMEM lane quarter q = warp % 4 -> tile rows [32q, 32q + 32)
    const int q = warp & 3;
    int i = 0;
    if (tma_c) {
      // 32x32 sub-tiles: tcgen05.ld (thread = row), registers -> a 128B-
      // swizzled 4 KB smem box (two per warp, alternating), TMA store of the
      // box (rows >= M / columns >= N clipped by the tensor map); the TMEM
      // buffer is released as soon as its last columns are in registers
      uint8_t* ebuf = smem + TC_STAGES * STAGE_BYTES + 1024 + q * 8192;
      uint32_t chunk = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
        const int z = t / tiles_mn, mn = t - z * tiles_mn;
        const int m0 = (mn / tiles_n) * TC_BM, n0 = (mn % tiles_n) * BN;
        const int b = i & 1;
        mbar_wait(&acc_full[b], (uint32_t)(i >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32, ++chunk) {
          uint32_t r[32];
          const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
              "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, "
              "%26, %27, %28, %29, %30, %31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),
                "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
                "=r"(r[30]), "=r"(r[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c0 + 32 >= BN) {
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
          }
          uint8_t* box = ebuf + (chunk & 1u) * 4096;
          // the store issued from this box two chunks ago must have read it
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          const uint32_t rowa = smem_u32(box) + (uint32_t)lane * 128u;
#pragma unroll
          for (int v = 0; v < 8; ++v)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             rowa + (uint32_t)((v ^ (lane & 7)) * 16)),
                         "r"(r[4 * v]), "r"(r[4 * v + 1]), "r"(r[4 * v + 2]), "r"(r[4 * v + 3])
                         : "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                ::"l"(&tC), "r"(n0 + c0), "r"(m0 + q * 32), "r"(z), "r"(smem_u32(box))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else {
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int z = t / tiles_mn, mn = t - z * tiles_mn;
      const int m0 = (mn / tiles_n) * TC_BM, n0 = (mn % tiles_n) * BN;
      const int b = i & 1;
      mbar_wait(&acc_full[b], (uint32_t)(i >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = m0 + q * 32 + lane;
      float* Cz = C + (long long)z * M * N;
      const bool vec = (N & 3) == 0;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
            "%10, %11, %12, %13, %14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
              "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
              "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M) {
          float* out = Cz + (long long)row * N + n0 + c0;
          if (vec && n0 + c0 + 16 <= N) {
#pragma unroll
            for (int v = 0; v < 4; ++v)
              reinterpret_cast<float4*>(out)[v] =
                  make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                              __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (n0 + c0 + e < N) out[e] = __uint_as_float(r[e]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * BN));
  }
}

// split-K epilogue, 16-byte accesses (mn % 4 == 0): same split order
__global__ void splitk_reduce_x4(const float4* __restrict__ W, float4* __restrict__ C,
                                 long long mn4, int splits) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mn4; i += stride) {
    // partials added in split order; 8 splits' loads in flight per round
    float4 acc = __ldcs(W + i);
    int s = 1;
    for (; s + 8 <= splits; s += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(W + (long long)(s + u) * mn4 + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x = acc.x + v[u].x;
        acc.y = acc.y + v[u].y;
        acc.z = acc.z + v[u].z;
        acc.w = acc.w + v[u].w;
      }
    }
    for (; s < splits; ++s) {
      const float4 v = __ldcs(W + (long long)s * mn4 + i);
      acc.x = acc.x + v.x;
      acc.y = acc.y + v.y;
      acc.z = acc.z + v.z;
      acc.w = acc.w + v.w;
    }
    C[i] = acc;
  }
}

// split-K epilogue: sum of the partial tiles in split order (deterministic)
__global__ void splitk_reduce(const float* __restrict__ W, float* __restrict__ C, long long mn,
                              int splits) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mn; i += stride) {
    float acc = W[i];
    for (int s = 1; s < splits; ++s) acc = acc + W[(long long)s * mn + i];
    C[i] = acc;
  }
}

// hi = x with the low 13 mantissa bits cleared, lo = x - hi; optionally
// transposing an (R, Ccols) row-major matrix into (Ccols, R).
__global__ void split_tf32_kernel(const float* __restrict__ x, float* __restrict__ hi,
                                  float* __restrict__ lo, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = x[i];
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    if (hi) hi[i] = h;  // hi may be skipped: tcgen05 kind::tf32 ignores the low
    lo[i] = v - h;      // 13 mantissa bits, so the raw fp32 operand IS hi
  }
}

// Same split with 16-byte accesses, two vectors in flight per thread and
// iteration (HBM-bound: 4 B read + 4 B written per element when hi is skipped).
__global__ void __launch_bounds__(256) split_tf32_x4_kernel(const float* __restrict__ x,
                                                            float* __restrict__ hi,
                                                            float* __restrict__ lo, long long n) {
  const long long n4 = n >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* lo4 = reinterpret_cast<float4*>(lo);
  float4* hi4 = reinterpret_cast<float4*>(hi);
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + stride < n4; i += 2 * stride) {
    const float4 a = x4[i], b = x4[i + stride];
    float4 ha, hb;
    const float4 la = tf32_lo4(a, &ha), lb = tf32_lo4(b, &hb);
    lo4[i] = la;
    lo4[i + stride] = lb;
    if (hi) {
      hi4[i] = ha;
      hi4[i + stride] = hb;
    }
  }
  for (; i < n4; i += stride) {
    float4 h;
    lo4[i] = tf32_lo4(x4[i], &h);
    if (hi) hi4[i] = h;
  }
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long j = (n4 << 2) + t;
  if (t < 4 && j < n) {
    const float v = x[j];
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    if (hi) hi[j] = h;
    lo[j] = v - h;
  }
}

// (R x Cc) row-major -> hi/lo of its transpose (Cc x ldo), rows padded to ldo
__global__ void split_tf32_transpose_kernel(const float* __restrict__ x, float* __restrict__ hi,
                                            float* __restrict__ lo, long long R, long long Cc,
                                            long long ldo) {
  __shared__ float tile[32][33];
  const long long bx = (long long)blockIdx.x * 32, by = (long long)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long r = by + j, c = bx + threadIdx.x;
    tile[j][threadIdx.x] = (r < R && c < Cc) ? x[r * Cc + c] : 0.f;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long c = bx + j, r = by + threadIdx.x;  // output row c, column r
    if (c < Cc && r < ldo) {
      const float v = r < R ? tile[threadIdx.x][j] : 0.f;
      const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
      hi[c * ldo + r] = h;
      lo[c * ldo + r] = v - h;
    }
  }
}

// mn_major: 32x32 boxes in the 128B-swizzle-with-32B-atoms layout that
// MN-major tf32 UMMA operands require (see sw128_mn_desc)
static int encode_map(CUtensorMap* map, const float* ptr, long long rows, long long cols,
                      int box_rows, bool mn_major = false) {
  if (!drv.tensorMapEncodeTiled) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SF_ERR_CUDA;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  const cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  SF_CHECK_CU(drv.tensorMapEncodeTiled(
      map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE,
      mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return SF_OK;
}

// GEMM output (Z split slices of M x N, row-major) for the TMA-store
// epilogue: 32 x 32 boxes, 128B swizzle (the epilogue's smem box layout)
static int encode_out_map(CUtensorMap* map, float* ptr, long long M, long long N, long long Z) {
  if (!drv.tensorMapEncodeTiled) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SF_ERR_CUDA;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)Z};
  const cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)(M * N * 4)};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  SF_CHECK_CU(drv.tensorMapEncodeTiled(
      map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)ptr, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return SF_OK;
}

static bool no_tma_store() {
  static const bool off = getenv("SF_GEMM_NO_TMA_STORE") != nullptr;
  return off;
}

// TMA im2col map of an NHWC float32 input for a KH x KW (stride s, pad p)
// convolution: 32 channels x 128 output pixels per box, 128B swizzle (the
// K-major A-tile layout the MMA descriptors expect)
static int encode_im2col_map(CUtensorMap* map, const GatherGeom& g) {
  if (!drv.tensorMapEncodeIm2col) {
    set_error("cuTensorMapEncodeIm2col unavailable");
    return SF_ERR_CUDA;
  }
  const int kh = g.kh;
  const cuuint64_t dims[4] = {(cuuint64_t)g.c, (cuuint64_t)g.w, (cuuint64_t)g.h, (cuuint64_t)g.n};
  const cuuint64_t strides[3] = {(cuuint64_t)g.c * 4, (cuuint64_t)g.c * g.w * 4,
                                 (cuuint64_t)g.c * g.w * g.h * 4};
  const int lower[2] = {-g.p, -g.p};                                   // W, H
  const int upper[2] = {g.p - (g.kw - 1), g.p - (kh - 1)};
  const cuuint32_t estr[4] = {1, (cuuint32_t)g.s, (cuuint32_t)g.s, 1};
  SF_CHECK_CU(drv.tensorMapEncodeIm2col(
      map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)g.x, dims, strides, lower, upper, 32,
      TC_BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return SF_OK;
}

// ak / bk: the contraction extent each operand actually stores (<= K; the
// TMA boxes zero-fill beyond it).  K-major: the row length (leading
// dimension); MN-major: the number of rows.
template <int BN, bool AMN, bool BMN, bool GATHER = false>
static int run_tc(Device* d, long long M, long long N, long long K, long long ak, long long bk,
                  const float* ahi, const float* alo, const float* bhi, const float* blo,
                  float* c, const GatherGeom* gat = nullptr) {
  // a null lo pointer: that operand's lo part is derived in shared memory
  const int lo_a_smem = alo == nullptr, lo_b_smem = blo == nullptr;
  if (lo_a_smem) alo = ahi;  // the (unused) lo map still needs a valid encoding
  if (lo_b_smem) blo = bhi;
  CUtensorMap ta, tal, tb, tbl;
  if (GATHER && gat && gat->tma) {
    SF_TRY(encode_im2col_map(&ta, *gat));
    tal = ta;
  } else if (GATHER) {
    // A is gathered by the producer warp; its maps are unused (any valid map)
    if (BMN) {
      SF_TRY(encode_map(&ta, bhi, bk, N, 32, true));
    } else {
      SF_TRY(encode_map(&ta, bhi, N, bk, BN));
    }
    tal = ta;
  } else if (AMN) {
    SF_TRY(encode_map(&ta, ahi, ak, M, 32, true));
    SF_TRY(encode_map(&tal, alo, ak, M, 32, true));
  } else {
    SF_TRY(encode_map(&ta, ahi, M, ak, TC_BM));
    SF_TRY(encode_map(&tal, alo, M, ak, TC_BM));
  }
  if (BMN) {
    SF_TRY(encode_map(&tb, bhi, bk, N, 32, true));
    SF_TRY(encode_map(&tbl, blo, bk, N, 32, true));
  } else {
    SF_TRY(encode_map(&tb, bhi, N, bk, BN));
    SF_TRY(encode_map(&tbl, blo, N, bk, BN));
  }
  // + 4 epilogue warps x two 4 KB output boxes (TMA-store epilogue)
  const int smem = TcStages<BN>::n * (2 * TC_BM * TC_BK * 4 + 2 * BN * TC_BK * 4) + 1024 + 1024 +
                   4 * 8192;
  static bool configured[64] = {};
  if (!configured[d->id]) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc_persistent<BN, AMN, BMN, GATHER>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured[d->id] = true;
  }
  const long long tiles_n = (N + BN - 1) / BN, tiles_m = (M + TC_BM - 1) / TC_BM;
  const long long nk = (K + TC_BK - 1) / TC_BK;
  const long long tiles = tiles_n * tiles_m;
  long long splits = 1;
  if (tiles < d->sm_count && nk >= 64) {  // long contraction, few tiles
    splits = (2LL * d->sm_count + tiles - 1) / tiles;
    if (splits > nk / 16) splits = nk / 16;
    if (splits > 128) splits = 128;
    if (splits < 1) splits = 1;
  }
  const long long per = (nk + splits - 1) / splits;
  splits = (nk + per - 1) / per;
  const long long n_tiles = tiles * splits;
  const unsigned grid = (unsigned)(n_tiles < d->sm_count ? n_tiles : d->sm_count);
  static const bool log_shapes = getenv("SF_GEMM_LOG") != nullptr;
  if (log_shapes)
    fprintf(stderr, "gemm_tc BN=%d amn=%d bmn=%d M=%lld N=%lld K=%lld tiles=%lld splits=%lld lo=%d%d\n",
            BN, (int)AMN, (int)BMN, M, N, K, tiles, splits, lo_a_smem, lo_b_smem);
  float* out = c;
  float* work = nullptr;
  if (splits > 1)
    SF_TRY(d->alloc.alloc(d->id, sizeof(float) * (size_t)(splits * M * N), (void**)&work));
  if (work) out = work;
  // output through TMA stores when the rows are 16-byte multiples
  CUtensorMap tc;
  int tma_c = 0;
  if (N % 4 == 0 && (uintptr_t)out % 16 == 0 && !no_tma_store()) {
    SF_TRY(encode_out_map(&tc, out, M, N, splits));
    tma_c = 1;
  } else {
    tc = ta;  // unused
  }
  GatherGeom gg{};
  if (gat) gg = *gat;
  gemm_tc_persistent<BN, AMN, BMN, GATHER><<<grid, 320, smem, d->stream>>>(
      ta, tal, tb, tbl, tc, out, (int)M, (int)N, (int)K, (int)per, (int)tiles_n, (int)tiles,
      (int)n_tiles, GATHER ? 1 : lo_a_smem, lo_b_smem, tma_c, gg);
  if (splits == 1) {
    count_launch(d->id);
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  }
  if ((M * N) % 4 == 0 && (uintptr_t)c % 16 == 0) {
    long long blocks = (M * N / 4 + 255) / 256;
    if (blocks > d->sm_count * 16LL) blocks = d->sm_count * 16LL;
    splitk_reduce_x4<<<(unsigned)blocks, 256, 0, d->stream>>>(
        (const float4*)work, (float4*)c, M * N / 4, (int)splits);
  } else {
    long long blocks = (M * N + 255) / 256;
    if (blocks > d->sm_count * 16LL) blocks = d->sm_count * 16LL;
    splitk_reduce<<<(unsigned)blocks, 256, 0, d->stream>>>(work, c, M * N, (int)splits);
  }
  count_launch(d->id, 2);
  d->alloc.release(work);  // stream-ordered reuse is safe
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

template <int BN>
static int run_tc_major(Device* d, long long M, long long N, long long K, bool amn, bool bmn,
                        long long ak, long long bk, const float* ahi, const float* alo,
                        const float* bhi, const float* blo, float* c) {
  if (amn && bmn) return run_tc<BN, true, true>(d, M, N, K, ak, bk, ahi, alo, bhi, blo, c);
  if (amn) return run_tc<BN, true, false>(d, M, N, K, ak, bk, ahi, alo, bhi, blo, c);
  if (bmn) return run_tc<BN, false, true>(d, M, N, K, ak, bk, ahi, alo, bhi, blo, c);
  return run_tc<BN, false, false>(d, M, N, K, ak, bk, ahi, alo, bhi, blo, c);
}

int launch_gemm_tc_ex(Device* d, int64_t M, int64_t N, int64_t K, bool amn, bool bmn, int64_t ak,
                      int64_t bk, const float* ahi, const float* alo, const float* bhi,
                      const float* blo, float* c) {
  if (M == 0 || N == 0) return SF_OK;
  // every TMA row stride must be a multiple of 16 bytes
  const long long a_ld = amn ? M : ak, b_ld = bmn ? N : bk;
  if (a_ld % 4 != 0 || b_ld % 4 != 0 || ak > K || bk > K || ak <= 0 || bk <= 0) {
    set_error("gemm_tc: operand leading dimensions must be multiples of 4 and extents <= k");
    return SF_ERR_INVALID;
  }
  if (N <= 64) return run_tc_major<64>(d, M, N, K, amn, bmn, ak, bk, ahi, alo, bhi, blo, c);
  // 256-wide tiles where they still give every SM a tile
  static const int bn256 = [] {
    const char* e = getenv("SF_GEMM_BN256");
    return e ? atoi(e) : 1;
  }();
  const long long tiles256 = ((N + 255) / 256) * ((M + TC_BM - 1) / TC_BM);
  // (bn256 >= 2: also for long contractions, where split-K fills the SMs)
  const bool long_k = (K + TC_BK - 1) / TC_BK >= 64;
  if (bn256 && N >= 256 && (tiles256 >= d->sm_count || (bn256 >= 2 && long_k)))
    return run_tc_major<256>(d, M, N, K, amn, bmn, ak, bk, ahi, alo, bhi, blo, c);
  return run_tc_major<128>(d, M, N, K, amn, bmn, ak, bk, ahi, alo, bhi, blo, c);
}

// Implicit-GEMM convolution: out[N*HO*WO, co] = im2col(x) . W, W (kh*kw*c, co)
// row-major read MN-major; x NHWC with c % 32 == 0 (one filter tap per
// 32-wide k-block).  Same tiles, passes and k order as the explicit
// im2col + GEMM path, so the result is bit-identical to it.
int launch_conv_tc(Device* d, const int64_t* g8, int64_t co, const float* x, const float* w,
                   float* out) {
  const long long n = g8[0], h = g8[1], wd = g8[2], c = g8[3], kh = g8[4], kw = g8[5];
  const long long st = g8[6], pd = g8[7];
  const long long ho = (h + 2 * pd - kh) / st + 1, wo = (wd + 2 * pd - kw) / st + 1;
  const long long M = n * ho * wo, K = kh * kw * c;
  if (c % 32 != 0 || co % 4 != 0 || (uintptr_t)x % 16 != 0 || n * h * wd >= (1ll << 31) ||
      M >= (1ll << 31) || h >= 32768 || wd >= 32768 || pd >= 16384) {
    set_error("conv_tc: needs C % 32 == 0, Cout % 4 == 0, a 16-byte aligned input and "
              "32-bit pixel indices");
    return SF_ERR_INVALID;
  }
  if (M == 0 || co == 0) return SF_OK;
  // A tiles through TMA im2col boxes (one copy per k-block; the hardware
  // walks the output pixels and zero-fills the padding) when the driver
  // offers im2col maps, else the producer warp's cp.async gathers.  B200,
  // ResNet-50 b32 forward (tools/conv_time.py): layer1 3x3 141 -> 77 us,
  // layer2 92 -> 59 us, layer3 78 -> 54 us, layer4 73 -> 62 us, strided
  // 1x1 52 -> 40 us (explicit im2col + GEMM: 161 / 106 / 77 / 73 / 52 us)
  static const int im2col_tma = getenv("SF_CONV_TMA") ? atoi(getenv("SF_CONV_TMA")) : 1;
  GatherGeom gg{x, (int)h, (int)wd, (int)c, (int)kw, (int)st, (int)pd, (int)wo, (int)(ho * wo),
                im2col_tma && drv.tensorMapEncodeIm2col ? 1 : 0, (int)n, (int)kh};
  if (co <= 64) return run_tc<64, false, true, true>(d, M, co, K, K, K, nullptr, nullptr, w,
                                                     nullptr, out, &gg);
  const long long tiles256 = ((co + 255) / 256) * ((M + TC_BM - 1) / TC_BM);
  if (co >= 256 && tiles256 >= d->sm_count)
    return run_tc<256, false, true, true>(d, M, co, K, K, K, nullptr, nullptr, w, nullptr, out,
                                          &gg);
  return run_tc<128, false, true, true>(d, M, co, K, K, K, nullptr, nullptr, w, nullptr, out,
                                        &gg);
}

int launch_gemm_tc(Device* d, int64_t M, int64_t N, int64_t K, const float* ahi, const float* alo,
                   const float* bhi, const float* blo, float* c) {
  return launch_gemm_tc_ex(d, M, N, K, false, false, K, K, ahi, alo, bhi, blo, c);
}

int launch_split_tf32(Device* d, int64_t n, const float* x, float* hi, float* lo) {
  if (n == 0) return SF_OK;
  if (((uintptr_t)x | (uintptr_t)hi | (uintptr_t)lo) % 16 == 0 && n >= 4096) {
    long long blocks = (n / 4 + 255) / 256;
    if (blocks > d->sm_count * 8LL) blocks = d->sm_count * 8LL;
    split_tf32_x4_kernel<<<(unsigned)blocks, 256, 0, d->stream>>>(x, hi, lo, n);
    count_launch(d->id);
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  }
  long long blocks = (n + 255) / 256;
  if (blocks > d->sm_count * 16LL) blocks = d->sm_count * 16LL;
  split_tf32_kernel<<<(unsigned)blocks, 256, 0, d->stream>>>(x, hi, lo, n);
  count_launch(d->id);
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

int launch_split_tf32_t(Device* d, int64_t R, int64_t Cc, int64_t ldo, const float* x, float* hi,
                        float* lo) {
  if (R == 0 || Cc == 0) return SF_OK;
  dim3 grid((unsigned)((Cc + 31) / 32), (unsigned)((ldo + 31) / 32));
  split_tf32_transpose_kernel<<<grid, dim3(32, 8), 0, d->stream>>>(x, hi, lo, R, Cc, ldo);
  count_launch(d->id);
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

extern "C" {

int sf_gemm_tf32x3(int dev, int64_t m, int64_t n, int64_t k, const void* a_hi, const void* a_lo,
                   const void* b_hi, const void* b_lo, void** c) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (*c == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)(m * n) * 4, c));
  return launch_gemm_tc(d, m, n, k, (const float*)a_hi, (const float*)a_lo, (const float*)b_hi,
                        (const float*)b_lo, (float*)*c);
}

int sf_gemm_tf32x3_ex(int dev, int64_t m, int64_t n, int64_t k, int a_mn, int b_mn, int64_t ak,
                      int64_t bk, const void* a_hi, const void* a_lo, const void* b_hi,
                      const void* b_lo, void** c) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (*c == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)(m * n) * 4, c));
  return launch_gemm_tc_ex(d, m, n, k, a_mn != 0, b_mn != 0, ak, bk, (const float*)a_hi,
                           (const float*)a_lo, (const float*)b_hi, (const float*)b_lo,
                           (float*)*c);
}

int sf_conv2d_tc(int dev, const int64_t* g8, int64_t co, const void* x, const void* w,
                 void** out) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  const long long ho = (g8[1] + 2 * g8[7] - g8[4]) / g8[6] + 1;
  const long long wo = (g8[2] + 2 * g8[7] - g8[5]) / g8[6] + 1;
  if (*out == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)(g8[0] * ho * wo * co) * 4, out));
  return launch_conv_tc(d, g8, co, (const float*)x, (const float*)w, (float*)*out);
}

int sf_split_tf32(int dev, int64_t rows, int64_t cols, int64_t ldo, int transpose, const void* x,
                  void** hi, void** lo) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  const int64_t n = transpose ? cols * ldo : rows * ldo;
  if (hi == nullptr && transpose) {
    set_error("sf_split_tf32: the hi part may only be skipped without transpose");
    return SF_ERR_INVALID;
  }
  if (hi && *hi == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)n * 4, hi));
  if (*lo == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)n * 4, lo));
  if (transpose)
    return launch_split_tf32_t(d, rows, cols, ldo, (const float*)x, (float*)*hi, (float*)*lo);
  if (ldo != cols) {
    set_error("sf_split_tf32: padding only supported with transpose");
    return SF_ERR_INVALID;
  }
  return launch_split_tf32(d, rows * cols, (const float*)x, hi ? (float*)*hi : nullptr,
                           (float*)*lo);
}

}  // extern "C"
