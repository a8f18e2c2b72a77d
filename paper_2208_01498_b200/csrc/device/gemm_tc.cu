// Tensor-core path for the large, GEMM-shaped steps of the contraction tree
// (complex64 amplitudes).  PAPER.md Eq. (3) (l.82-86): a step contracting the two
// child tensors costs M multiply-adds, the product of all index dimensions -- for
// the top levels of the separator hierarchy this is a dense complex GEMM
//   C[b][m][n] = sum_k A[b][m][k] * B[b][k][n].
//
// Precision scheme: every fp32 component x of A and B
// is split into three bf16 pieces x = x0 + x1 + x2 (each the bf16 rounding of the
// remainder); the six products x_i y_j with i + j <= 2 are accumulated in fp32 on
// tcgen05 (kind::f16, bf16 inputs, fp32 accumulators in TMEM).  Complex arithmetic
// is planar: Cr += Ar.Br + (-Ai).Bi, Ci += Ar.Bi + Ai.Br, the minus sign taken by
// the instruction descriptor's negate-A bit, so no operand is ever expanded.
//
// Pipeline: pack kernel (fused permutation to matricised [b][rows][k] form + bf16x3
// split, one HBM pass) -> TMA (SWIZZLE_64B, 3-D maps over planes) into a 2/3-stage
// mbarrier ring -> one elected thread issues tcgen05.mma into ping-pong TMEM buffers
// -> epilogue warps promote each stage into fp32 registers (tcgen05.ld) and finally
// write interleaved complex64 C (or a split-K partial).
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace tnd {

// ------------------------------------------------------------------- pack ----
struct PackDesc {
  int32_t src;                      // node id in the pointer table
  int32_t nb_bits, r_bits, k_bits;
  GroupMap gb, gr, gk;              // element offsets of (batch, row, k) in the source
};

__device__ __forceinline__ void split3(float x, __nv_bfloat16& p0, __nv_bfloat16& p1, __nv_bfloat16& p2) {
  p0 = __float2bfloat16_rn(x);
  float r = x - __bfloat162float(p0);
  p1 = __float2bfloat16_rn(r);
  r = r - __bfloat162float(p1);
  p2 = __float2bfloat16_rn(r);
}

// out: 6 planes (piece * 2 + {re, im}) of [b][r][k] bf16; each thread packs 8
// consecutive k of one (b, r) row: 8 complex loads, 6 x 16-byte stores.
__global__ void __launch_bounds__(256) pack_bf16x3_kernel(const void* const* __restrict__ ptrs, PackDesc d,
                                                          const int64_t* __restrict__ tab,
                                                          __nv_bfloat16* __restrict__ out) {
  const float2* __restrict__ src = reinterpret_cast<const float2*>(ptrs[d.src]);
  const int64_t plane = int64_t(1) << (d.nb_bits + d.r_bits + d.k_bits);
  const int64_t nvec = plane >> 3;
  const int64_t kmask8 = (int64_t(1) << (d.k_bits - 3)) - 1;
  const int64_t rmask = (int64_t(1) << d.r_bits) - 1;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < nvec; v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k0 = (v & kmask8) << 3;
    const int64_t row = (v >> (d.k_bits - 3)) & rmask;
    const int64_t b = v >> (d.k_bits - 3 + d.r_bits);
    const int64_t base = gmap(tab, d.gb, b) + gmap(tab, d.gr, row);
    __align__(16) __nv_bfloat16 pc[6][8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float2 x = src[base + gmap(tab, d.gk, k0 + j)];
      split3(x.x, pc[0][j], pc[2][j], pc[4][j]);
      split3(x.y, pc[1][j], pc[3][j], pc[5][j]);
    }
#pragma unroll
    for (int p = 0; p < 6; ++p)
      *reinterpret_cast<uint4*>(out + p * plane + (v << 3)) = *reinterpret_cast<const uint4*>(pc[p]);
  }
}

// ------------------------------------------------------------- tcgen05 -------
namespace tc {

constexpr int BM = 128;   // rows per tile (TMEM lanes)
constexpr int BK = 32;    // bf16 elements of K per stage (64-byte rows, SWIZZLE_64B)

template <int BN>
struct Cfg {
  static constexpr int A_PLANE = BM * BK * 2;
  static constexpr int B_PLANE = BN * BK * 2;
  static constexpr int STAGE = 6 * A_PLANE + 6 * B_PLANE;
  static constexpr int STAGES = (3 * STAGE + 2048 <= 227 * 1024) ? 3 : 2;
  static constexpr int ACC_COLS = 2 * BN;                  // re + im of one accumulator buffer
  static constexpr int TMEM_COLS = 2 * ACC_COLS;           // ping-pong buffers
  static constexpr int EPI_WARPS = 4 * (BN / 64);          // each owns 32 rows x 64 columns
  static constexpr int THREADS = 32 * (EPI_WARPS + 2);     // + TMA warp + MMA warp
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, void* smem, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// K-major operand tile with 64-byte rows, SWIZZLE_64B: 8-row atoms of 512 B.
__device__ __forceinline__ uint64_t make_desc_sw64(const void* smem) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;            // start address
  d |= (uint64_t)(0) << 16;                // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;         // SBO: 8 rows * 64 B
  d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;                  // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// Precision: the tensor core's fp32 accumulation
// truncates, so an accumulator updated T times drifts by ~T/4 ulp toward zero.  Each
// 32-wide K stage is therefore accumulated in a fresh TMEM buffer (24 MMA updates per
// element) and promoted by the epilogue warps into fp32 registers with round-to-
// nearest adds; two TMEM buffers ping-pong so promotion overlaps the next stage.
template <int BN>
__global__ void __launch_bounds__(Cfg<BN>::THREADS, 1)
    cgemm_bf16x6_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        void* const* __restrict__ ptrs, int32_t c_node, int32_t M, int32_t N, int32_t K,
                        int32_t nb, int32_t kc_per_split, float2* __restrict__ partial) {
  using CF = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::STAGES * CF::STAGE);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* tfull = empty + CF::STAGES;     // [2] MMA -> epilogue: buffer holds a finished stage
  uint64_t* tempty = tfull + 2;             // [2] epilogue -> MMA: buffer promoted
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TMA_WARP = CF::EPI_WARPS, MMA_WARP = CF::EPI_WARPS + 1;
  // split-K: blockIdx.z = split * nb + batch; this CTA covers K chunks [kc0, kc0 + nk)
  const int n_blk = blockIdx.x, m_blk = blockIdx.y, b = blockIdx.z % nb, split = blockIdx.z / nb;
  const int nk_all = (K + BK - 1) / BK;
  const int kc0 = split * kc_per_split;
  const int nk = min(nk_all, kc0 + kc_per_split) - kc0;

  if (warp == TMA_WARP && lane == 0) {
    for (int s = 0; s < CF::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], CF::EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == TMA_WARP) {
    if (lane == 0) {
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % CF::STAGES;
        const uint32_t ph = (kc / CF::STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], CF::STAGE);
        uint8_t* st = smem + s * CF::STAGE;
        for (int p = 0; p < 6; ++p)
          tma_load_3d(&tmA, st + p * CF::A_PLANE, &full[s], (kc0 + kc) * BK, m_blk * BM, p * nb + b);
        for (int p = 0; p < 6; ++p)
          tma_load_3d(&tmB, st + 6 * CF::A_PLANE + p * CF::B_PLANE, &full[s], (kc0 + kc) * BK, n_blk * BN, p * nb + b);
      }
    }
  } else if (warp == MMA_WARP) {
    if (lane == 0) {
      // idesc: F32 accumulate, BF16 A/B, K-major both, N = BN, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      const uint32_t idesc_negA = idesc | (1u << 13);
      const int PA[6] = {0, 0, 1, 0, 1, 2};
      const int PB[6] = {0, 1, 0, 2, 1, 0};
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % CF::STAGES;
        const uint32_t ph = (kc / CF::STAGES) & 1;
        const int buf = kc & 1;
        const uint32_t tph = (kc >> 1) & 1;
        mbar_wait(&tempty[buf], tph ^ 1);       // epilogue has drained this buffer
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t t_re = tmem + buf * CF::ACC_COLS, t_im = t_re + BN;
        uint8_t* st = smem + s * CF::STAGE;
#pragma unroll
        for (int ks = 0; ks < BK / 16; ++ks) {
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const uint64_t a_re = make_desc_sw64(st + (2 * PA[q] + 0) * CF::A_PLANE) + (uint64_t)(ks * 2);
            const uint64_t a_im = make_desc_sw64(st + (2 * PA[q] + 1) * CF::A_PLANE) + (uint64_t)(ks * 2);
            const uint64_t b_re = make_desc_sw64(st + 6 * CF::A_PLANE + (2 * PB[q] + 0) * CF::B_PLANE) + (uint64_t)(ks * 2);
            const uint64_t b_im = make_desc_sw64(st + 6 * CF::A_PLANE + (2 * PB[q] + 1) * CF::B_PLANE) + (uint64_t)(ks * 2);
            const uint32_t acc = (ks | q) != 0;   // fresh accumulator every stage
            mma_bf16(t_re, a_re, b_re, idesc, acc);
            mma_bf16(t_re, a_im, b_im, idesc_negA, 1);
            mma_bf16(t_im, a_re, b_im, idesc, acc);
            mma_bf16(t_im, a_im, b_re, idesc, 1);
          }
        }
        mma_commit(&empty[s]);     // smem stage free once these MMAs have read it
        mma_commit(&tfull[buf]);   // accumulator buffer ready for promotion
      }
    }
  } else {
    // ---- epilogue warps: promote every stage into fp32 registers ----
    const int lg = warp & 3;                 // TMEM lane group (rows 32 lg .. 32 lg + 31)
    const int ch = warp >> 2;                // column half: columns [64 ch, 64 ch + 64)
    const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
    float ar[64], ai[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) { ar[j] = 0.f; ai[j] = 0.f; }
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      const uint32_t tph = (kc >> 1) & 1;
      mbar_wait(&tfull[buf], tph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t t_re = tmem + buf * CF::ACC_COLS + lane_base + ch * 64, t_im = t_re + BN;
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        uint32_t vr[16], vi[16];
        tmem_ld16(t_re + c, vr);
        tmem_ld16(t_im + c, vi);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          ar[c + j] = __fadd_rn(ar[c + j], __uint_as_float(vr[j]));
          ai[c + j] = __fadd_rn(ai[c + j], __uint_as_float(vi[j]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
    // single split: write C; several: this split's fp32 partial (reduced in fp64 later)
    float2* C = partial ? partial + (int64_t)split * nb * M * (int64_t)N : reinterpret_cast<float2*>(ptrs[c_node]);
    const int row = m_blk * BM + lg * 32 + lane;
    const int col0 = n_blk * BN + ch * 64;
    if (row < M && col0 < N) {
      float2* crow = C + ((int64_t)b * M + row) * (int64_t)N + col0;
      if (N - col0 >= 64) {
#pragma unroll
        for (int j = 0; j < 64; j += 2) *reinterpret_cast<float4*>(crow + j) = make_float4(ar[j], ai[j], ar[j + 1], ai[j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (j < N - col0) crow[j] = make_float2(ar[j], ai[j]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS));
}

}  // namespace tc

// C[i] = sum_s partial[s][i], summed in fp64 (split-K epilogue)
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float2* __restrict__ partial, int32_t S,
                                                            int64_t n, void* const* __restrict__ ptrs, int32_t c_node) {
  float2* C = reinterpret_cast<float2*>(ptrs[c_node]);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int s = 0; s < S; ++s) {
      const float2 v = partial[(int64_t)s * n + i];
      re += v.x;
      im += v.y;
    }
    C[i] = make_float2((float)re, (float)im);
  }
}
}  // namespace tnd
