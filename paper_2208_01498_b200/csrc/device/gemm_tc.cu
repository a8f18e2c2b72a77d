// Tensor-core path for the large, GEMM-shaped steps of the contraction tree
// (complex64 amplitudes).  PAPER.md Eq. (3) (l.82-86): a step contracting the two
// child tensors costs M multiply-adds, the product of all index dimensions -- for
// the top levels of the separator hierarchy this is a dense complex GEMM
//   C[b][m][n] = sum_k A[b][m][k] * B[b][k][n].
//
// Precision scheme: every fp32 component x of A and B
// is scaled by a power of two per (row, 128-element K chunk) so the chunk maximum lies
// just below 2^14, then split into two fp16 pieces x = x0 + x1 (x0 = fp16(x),
// x1 = fp16(x - x0)): 22 significand bits, the representation error is
// <= 2^-24 |x| + 2^-38 max|chunk|.  The three products x0 y0, x0 y1, x1 y0 are
// accumulated in fp32 on tcgen05 (kind::f16, fp16 inputs, fp32 accumulators in TMEM);
// the dropped x1 y1 is <= 2^-24 |x y|.  That is fp32-level accuracy at 3 MMAs per real
// product (bf16x3 splitting needs 6).  Complex arithmetic is planar:
// Cr += Ar.Br + (-Ai).Bi, Ci += Ar.Bi + Ai.Br, the minus sign taken by the instruction
// descriptor's negate-A bit, so no operand is ever expanded.
//
// Pipeline: pack kernel (fused permutation to matricised [b][rows][k] form + scale +
// fp16x2 split, one HBM pass) -> TMA (SWIZZLE_64B, 3-D maps over the 4 planes) and bulk
// copies of the chunk scales into mbarrier rings -> one elected thread issues
// tcgen05.mma into ping-pong TMEM buffers -> epilogue warps promote each stage, scaled,
// into fp32 registers (tcgen05.ld) and finally write interleaved complex64 C (or a
// split-K partial).
#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace tnd {

// ------------------------------------------------------------------- pack ----
// Fused permutation + split of one operand into the tensor-core layout.
// The operand's stored order and the matricised order [b][rows][k] are both
// row-major over power-of-two dimensions, so the permutation is a permutation of the
// bits of the element index.  One CTA handles a tile of 2^t_bits elements whose bits
// T contain the source's 4 lowest bits (coalesced 128-byte reads of complex64) and the
// destination's lowest bits (coalesced 16-byte writes); the tile is transposed
// through shared memory.
struct PackDesc {
  int32_t src;                      // node id in the pointer table
  int32_t nb_bits, r_bits, k_bits;
  int32_t t_bits;                   // |T|
  int32_t ld;                       // lowest destination bits inside T (contiguous runs)
  int32_t tile_bits;                // bits enumerating tiles
  int32_t pad;
  int64_t e_src;                    // tab[e_src + e]: source offset of local element e
  int64_t e_q;                      // tab[e_q + e]: compact destination index of e
  GroupMap tile_src, tile_dst;      // tile id -> source / destination element offset
  GroupMap q_hi;                    // (q >> ld) -> destination offset
  int64_t plane;                    // rows * K: elements per plane
};

constexpr int PACK_MAX_T = 11;
constexpr int PACK_THREADS = 256;
constexpr int PACK_PER_THREAD = (1 << PACK_MAX_T) / PACK_THREADS;   // 8

// smem slot of compact destination index q: XOR-swizzle bits 1-3 by higher bits so the
// scattered 8-byte stores of phase 1 spread over banks; pairs (bit 0) stay adjacent
// for the 16-byte loads of phase 2.
__device__ __forceinline__ int pack_slot(int q) { return q ^ ((((q >> 4) ^ (q >> 7) ^ (q >> 10)) & 7) << 1); }

// Block scaling: every chunk of 2^SCALE_LOG2 consecutive K
// elements of one row (re and im together) gets a power-of-two scale 2^(e-14), e the
// exponent with max|x| < 2^e, so the scaled chunk lies in (-2^14, 2^14): the top of the
// fp16 range, which keeps the second piece of elements far below the chunk maximum out
// of the fp16 subnormals (absolute error floor 2^-25 in the scaled unit, i.e. at most
// 2^-38 of the chunk maximum, which is >= 2^13 after scaling).
constexpr int SCALE_LOG2 = 7;   // 128-element K chunks = 4 GEMM stages per TMEM promotion
// a chunk (2^SCALE_LOG2 destination elements, 8 per thread) must lie within one warp for
// the shuffle max, and the tile must hold the chunk's destination bits plus the 4 lowest
// source bits (make_pack)
static_assert(SCALE_LOG2 <= 3 + 5, "scale chunk wider than one warp of pack threads");
static_assert(SCALE_LOG2 + 4 <= PACK_MAX_T, "pack tile too small for a scale chunk plus 4 source bits");

// split two scaled floats into two fp16x2 pieces: hi = fp16(x), lo = fp16(x - hi)
__device__ __forceinline__ void split2x2(float a, float b, uint32_t& p0, uint32_t& p1) {
  __half2 h = __floats2half2_rn(a, b);
  p0 = *reinterpret_cast<uint32_t*>(&h);
  const float2 f = __half22float2(h);
  h = __floats2half2_rn(a - f.x, b - f.y);
  p1 = *reinterpret_cast<uint32_t*>(&h);
}

// out planes, layout [b][4][r][k] fp16, plane = 2 * piece + {0: re, 1: im}; scales
// [b][K / 128][r] fp32 (one per row and 128-element K chunk; one per row if K < 128).
// Tiles have 2^t_bits elements, 8 <= t_bits <= PACK_MAX_T, destination bits 0..6 always
// inside the tile, so every K chunk is held by 2-16 adjacent threads of one warp.
// 4 CTAs per SM (64 registers, a few spilled) beat 3 without spills in the configs[1]
// step: 0.73 vs 0.70 of the copy peak (more bytes in flight; scripts/gpu_pack_ab.sh)
__global__ void __launch_bounds__(PACK_THREADS, 4) pack_f16x2s_kernel(const void* const* __restrict__ ptrs, PackDesc d,
                                                                   const int64_t* __restrict__ tab,
                                                                   __half* __restrict__ out, float* __restrict__ scales,
                                                                   int64_t src_base) {
  __shared__ __align__(16) float2 s[1 << PACK_MAX_T];
  const float2* __restrict__ src = reinterpret_cast<const float2*>(ptrs[d.src]) + src_base;
  const int64_t n_tiles = int64_t(1) << d.tile_bits;
  const int64_t lmask = (int64_t(1) << d.ld) - 1;
  const int T = 1 << d.t_bits;
  const int RK = d.r_bits + d.k_bits;
  const int chunk_log2 = min(d.k_bits, SCALE_LOG2);    // log2 elements per scale
  const int nch_log2 = max(d.k_bits - SCALE_LOG2, 0);  // log2 chunks per row
  int64_t so[PACK_PER_THREAD];
  int sl[PACK_PER_THREAD];
#pragma unroll
  for (int i = 0; i < PACK_PER_THREAD; ++i) {
    const int e = threadIdx.x + i * PACK_THREADS;
    so[i] = e < T ? __ldg(tab + d.e_src + e) : 0;
    sl[i] = e < T ? pack_slot((int)__ldg(tab + d.e_q + e)) : 0;
  }
  const int q0 = threadIdx.x * 8;                       // this thread's 8 destination elements
  const bool writer = q0 < T;                           // uniform per warp (T >= 256)
  const int64_t dq = writer ? (q0 & lmask) + gmap(tab, d.q_hi, q0 >> d.ld) : 0;
  // software pipeline: the next tile's loads are in flight while this tile goes through
  // shared memory and out (twice the bytes in flight per thread)
  float2 v[PACK_PER_THREAD];
  if ((int64_t)blockIdx.x < n_tiles) {
    const int64_t sb = gmap(tab, d.tile_src, blockIdx.x);
#pragma unroll
    for (int i = 0; i < PACK_PER_THREAD; ++i)
      if (threadIdx.x + i * PACK_THREADS < T) v[i] = __ldg(src + sb + so[i]);
  }
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t db = gmap(tab, d.tile_dst, tile) + dq;
#pragma unroll
    for (int i = 0; i < PACK_PER_THREAD; ++i)
      if (threadIdx.x + i * PACK_THREADS < T) s[sl[i]] = v[i];
    __syncthreads();
    if (tile + gridDim.x < n_tiles) {
      const int64_t sb = gmap(tab, d.tile_src, tile + gridDim.x);
#pragma unroll
      for (int i = 0; i < PACK_PER_THREAD; ++i)
        if (threadIdx.x + i * PACK_THREADS < T) v[i] = __ldg(src + sb + so[i]);
    }
    float4 w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = writer ? *reinterpret_cast<const float4*>(&s[pack_slot(q0 + 2 * j)]) : float4{};
    __syncthreads();
    if (!writer) continue;
    // chunk maximum over |re|, |im| (chunk = 2^chunk_log2 elements = 2^(chunk_log2-3) threads)
    float m = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) m = fmaxf(m, fmaxf(fmaxf(fabsf(w[j].x), fabsf(w[j].y)), fmaxf(fabsf(w[j].z), fabsf(w[j].w))));
    for (int o = 1; o < (1 << (chunk_log2 - 3)); o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    int e = 0;
    frexpf(m, &e);                                       // m < 2^e (e = 0 for m = 0)
    // scale up by 2^(14-e), exact; a second factor only when 14-e exceeds the fp32
    // exponent range (chunk maxima below 2^-113: a warp-uniform, practically never taken
    // branch -- the pack is issue-bound at the power-capped clock)
    const float upc = ldexpf(1.f, min(14 - e, 127));
    if (14 - e > 127) {
      const float up2 = ldexpf(1.f, 14 - e - 127);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        w[j].x *= up2; w[j].y *= up2; w[j].z *= up2; w[j].w *= up2;
      }
    }
    uint4 o[4];
    uint32_t* op = reinterpret_cast<uint32_t*>(o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t r0, r1, i0, i1;
      split2x2(w[j].x * upc, w[j].z * upc, r0, r1);
      split2x2(w[j].y * upc, w[j].w * upc, i0, i1);
      op[0 * 4 + j] = r0; op[1 * 4 + j] = i0; op[2 * 4 + j] = r1; op[3 * 4 + j] = i1;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) *reinterpret_cast<uint4*>(out + db + p * d.plane) = o[p];
    if ((threadIdx.x & ((1 << (chunk_log2 - 3)) - 1)) == 0) {
      const int64_t bb = db >> (RK + 2), rk = db & (d.plane - 1);
      const int64_t r = rk >> d.k_bits, kc = (rk & ((int64_t(1) << d.k_bits) - 1)) >> SCALE_LOG2;
      scales[(((bb << nch_log2) + kc) << d.r_bits) + r] = ldexpf(1.f, e - 14);
    }
  }
}

// ------------------------------------------------------------- tcgen05 -------
namespace tc {

constexpr int BM = 128;    // rows per tile (TMEM lanes)
constexpr int BK = 32;     // fp16 elements of K per smem stage (64-byte rows, SWIZZLE_64B)
constexpr int PROMO = 4;   // stages per TMEM accumulation = one 128-element scale chunk

// Debiasing of the truncating TMEM accumulation: tcgen05
// adds each MMA's products to the fp32 accumulator rounding toward zero, so a chunk sum
// built by T MMA updates comes out shrunk by ~beta(T) 2^-24 of itself -- coherently,
// and the amplitude is multilinear in every step's result, so the shrinks of all
// tensor-core steps multiply (measured 3-4e-5 on one configs[1] slice without this).
// beta measured on dense random operands (scripts/diag_bias2.py; Gaussian / unit-phase /
// log-normal: T = 6, 12, 24, 48 -> 3.1, 4.7, 8.0, 13-14.6; 70%-sparse: 2.6 .. 10.8).  The
// promotion scales the chunk by 1 + beta 2^-24 with beta rounded to an even number of
// units, so the factor is exact in fp32 and the per-chunk power-of-two scale stays exact.
// T = 12 MMA updates per 32-element stage of K (2 k16 blocks x 3 fp16x2 products x 2
// complex terms); 6 when K = 16 (half a stage).
__device__ __forceinline__ float rz_debias(int stages, int K) {
  const int T = K < BK ? 6 : 12 * stages;
  const int beta = T >= 48 ? 14 : T >= 36 ? 12 : T >= 24 ? 8 : T >= 12 ? 4 : 2;
  return 1.0f + (float)(beta >> 1) * 0x1p-23f;
}
// CTA rasterization: GROUP_M M-tiles sweep the N tiles together (panels shared in L2).
// Measured with scripts/raster_sweep.sh (DRAM traffic costs clock under the power cap):
// pair kernel 4 (DRAM reads 67 -> 55 GB on a (2^18, 2^12, 2^12) step, 1-2% faster);
// persistent short-K pair kernel 32 (69 -> 40 GB on (2^18, 2^16, 2^8), 0.5-1.3% faster);
// single-CTA kernel 8.
constexpr int GROUP_M = 8, GROUP_M_PAIR = 4, GROUP_M_PERSIST = 32;
__device__ int d_group_m = 0;   // > 0: TN_GEMM_GROUP_M override (raster experiments)
// pair kernel: odd raster groups sweep the N tiles backwards, so the B panels the last
// wave read are still in L2 when the next group starts (DRAM reads 57 -> 51 GB on the
// bench's dominant slab, ~1% faster); TN_GEMM_SERP=0 turns it off
__device__ int d_serp = 1;

template <int BN>
struct Cfg {
  static constexpr int A_PLANE = BM * BK * 2;              // one fp16 plane tile
  static constexpr int B_PLANE = BN * BK * 2;
  static constexpr int A_BYTES = 4 * A_PLANE;              // 2 pieces x (re, im)
  static constexpr int B_BYTES = 4 * B_PLANE;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SLOTS = 8;                          // scale ring (epilogue lags the MMA)
  static constexpr int SC_BYTES = (BM + BN) * 4;           // A and B chunk scales of one stage
  static constexpr int STAGES = (4 * STAGE + SLOTS * SC_BYTES + 2048 <= 227 * 1024) ? 4 : 3;
  static constexpr int ACC_COLS = 2 * BN;                  // [re | im] of one accumulator buffer
  static constexpr int TMEM_COLS = 2 * ACC_COLS;           // ping-pong buffers
  static constexpr int EPI_WARPS = 4 * (BN / 64);          // each owns 32 rows x 64 columns
  static constexpr int THREADS = 32 * (EPI_WARPS + 2);     // + TMA warp + MMA warp
  static constexpr int SMEM = STAGES * STAGE + SLOTS * SC_BYTES + 1024 /*align*/ + 512 /*barriers*/;
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
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// explicit shared / global vector accesses for the C staging (a generic pointer into the
// dynamic smem window compiles to generic LD.E / ST.E)
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void stg128(void* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 ldg128(const void* p) {
  float4 v;
  asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
// TMA tensor store / reduce-add of a staged smem box (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t smem, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(smem), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, uint32_t smem, int x, int y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(smem), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// plain bulk copy global -> shared (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(reinterpret_cast<uint64_t>(gmem)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// cta_group::2 helpers: shared::cluster address of the same location in CTA rank 0 of the
// cluster (the pair's leader), remote arrive, 2-SM TMA / MMA / commit
__device__ __forceinline__ uint32_t mapa_rank0(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-SM TMA: data into this CTA's shared memory, completion bytes to the leader's barrier
__device__ __forceinline__ void tma_load_3d_pair(const CUtensorMap* map, void* smem, uint32_t bar_cluster, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// arrive once on the barrier at this offset in both CTAs of the pair when the MMAs issued
// so far complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
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
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
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
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// Epilogue warps of both GEMM kernels: promote every TMEM accumulation (one 128-wide
// scale chunk) into fp32 registers, scaled by sA[row] * sB[col], then write C rows
// [row0, row0 + 128) x columns [col0, col0 + BN) (C += when `acc_c`); C is addressed as
// [b][c_rows][N] with this launch's rows at c_row_off (row slabs of a larger C).  kPair: the
// tempty barrier lives in the leader CTA of a cta_group::2 pair (remote arrive).
constexpr int EPI_PITCH = 132;   // floats per staged C row (64 complex + 16 B pad: conflict-free)
template <int BN, bool kPair>
__device__ __forceinline__ void epilogue(float* stage_smem, int warp, int lane, uint32_t tmem, const float* sc, uint64_t* sfull,
                                         uint64_t* sempty, uint64_t* tfull, uint64_t* tempty, int nk, int K,
                                         float2* C, int b, int M, int N, int row0, int col0_blk, bool acc_c,
                                         int c_rows, int c_row_off, const CUtensorMap* tmC = nullptr) {
  using CF = Cfg<BN>;
  const int lg = warp & 3;                 // TMEM lane group (rows 32 lg .. 32 lg + 31)
  const int ch = warp >> 2;                // column half: columns [64 ch, 64 ch + 64)
  const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
  float ar[64], ai[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) { ar[j] = 0.f; ai[j] = 0.f; }
  const int n_promo = (nk + PROMO - 1) / PROMO;
  for (int pi = 0; pi < n_promo; ++pi) {
    const int buf = pi & 1, slot = pi % CF::SLOTS;
    mbar_wait(&sfull[slot], (pi / CF::SLOTS) & 1);
    mbar_wait(&tfull[buf], (pi >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t scs = smem_u32(sc + slot * (BM + BN));
    const float sa = lds_f32(scs + 4 * (lg * 32 + lane)) * rz_debias(min(PROMO, nk - pi * PROMO), K);
    // column scales: one conflict-free load per lane, broadcast by shuffles (broadcast
    // LDS.128s cost 4 shared wavefronts each, competing with the MMA operand reads)
    const float sb_lo = lds_f32(scs + 4 * (BM + ch * 64 + lane));
    const float sb_hi = lds_f32(scs + 4 * (BM + ch * 64 + 32 + lane));
    const uint32_t t_re = tmem + buf * CF::ACC_COLS + lane_base + ch * 64, t_im = t_re + BN;
#pragma unroll
    for (int c = 0; c < 64; c += 8) {
      uint32_t vr[8], vi[8];
      tmem_ld8(t_re + c, vr);
      tmem_ld8(t_im + c, vi);
      float sbl[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) sbl[j] = __shfl_sync(0xffffffffu, (c + j) < 32 ? sb_lo : sb_hi, (c + j) & 31);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float s = sa * sbl[j];
        ar[c + j] = __fmaf_rn(__uint_as_float(vr[j]), s, ar[c + j]);
        ai[c + j] = __fmaf_rn(__uint_as_float(vi[j]), s, ai[c + j]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    if (lane == 0) {
      if (kPair) mbar_arrive_cluster(mapa_rank0(&tempty[buf]));
      else mbar_arrive(&tempty[buf]);
      mbar_arrive(&sempty[slot]);
    }
  }
  const int col0 = col0_blk + ch * 64;
  if (tmC) {
    // TMA tensor stores (reduce-add for C += of K-slabs): the warp's 32 x 64 complex block
    // goes to the (idle) operand stages as 4 boxes of 32 rows x 16 complex in the
    // SWIZZLE_128B layout of the C map (16-byte chunk j of row r at j ^ (r & 7)); one lane
    // issues the 4 stores.  Full tiles only (pair kernel: M % 256 == 0, N % 128 == 0).
    const uint32_t stg = smem_u32(stage_smem) + warp * (4 * 32 * 128);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        sts128(stg + q * (32 * 128) + lane * 128 + ((j ^ (lane & 7)) << 4),
               make_float4(ar[16 * q + 2 * j], ai[16 * q + 2 * j], ar[16 * q + 2 * j + 1], ai[16 * q + 2 * j + 1]));
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      const int y = b * c_rows + c_row_off + row0 + lg * 32;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (acc_c) tma_reduce_add_2d(tmC, stg + q * (32 * 128), 2 * (col0 + 16 * q), y);
        else tma_store_2d(tmC, stg + q * (32 * 128), 2 * (col0 + 16 * q), y);
      }
      bulk_commit();
      bulk_wait_all();
    }
    __syncwarp();
    return;
  }
  if (col0 + 64 <= N) {
    // Coalesced C: the warp's 32 x 64 complex block goes through shared memory (the
    // operand stages: every MMA has completed, so they are free) and leaves one 512-byte
    // row per instruction (thread-per-row stores would scatter 32 rows per instruction).
    const uint32_t stg = smem_u32(stage_smem + warp * (32 * EPI_PITCH));
#pragma unroll
    for (int j = 0; j < 32; ++j)
      sts128(stg + 4 * (lane * EPI_PITCH + 4 * j), make_float4(ar[2 * j], ai[2 * j], ar[2 * j + 1], ai[2 * j + 1]));
    __syncwarp();
    const int rbase = row0 + lg * 32;
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      if (rbase + r >= M) break;
      float4 v = lds128(stg + 4 * (r * EPI_PITCH + 4 * lane));
      float4* dst = reinterpret_cast<float4*>(C + ((int64_t)b * c_rows + c_row_off + rbase + r) * (int64_t)N + col0) + lane;
      if (acc_c) {
        const float4 o = ldg128(dst);
        v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
      }
      stg128(dst, v);
    }
    return;
  }
  const int row = row0 + lg * 32 + lane;
  if (row < M && col0 < N) {
    float2* crow = C + ((int64_t)b * c_rows + c_row_off + row) * (int64_t)N + col0;
    if (acc_c) {        // K-slab > 0: C += this slab's product
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        ar[j] += (j < N - col0) ? crow[j].x : 0.f;
        ai[j] += (j < N - col0) ? crow[j].y : 0.f;
      }
    }
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

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// MMA issue loop of the GEMM below (whole warp; one elected lane issues).  kTmem0: TMEM
// base known to be 0.
template <int BN, bool kTmem0>
__device__ __forceinline__ void mma_loop(uint8_t* smem, uint64_t* full, uint64_t* empty, uint64_t* tfull,
                                         uint64_t* tempty, uint32_t tmem_rt, int nk) {
  using CF = Cfg<BN>;
  const uint32_t tmem = kTmem0 ? 0u : tmem_rt;
  // idesc: F32 accumulate, F16 A/B, K-major both, N = BN, M = 128
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  constexpr uint32_t idesc_negA = idesc | (1u << 13);
  constexpr int PA[3] = {0, 0, 1};
  constexpr int PB[3] = {0, 1, 0};
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % CF::STAGES;
    const uint32_t ph = (kc / CF::STAGES) & 1;
    const int pi = kc / PROMO;
    const int buf = pi & 1;
    const bool first = (kc % PROMO) == 0;
    const bool last = (kc % PROMO) == PROMO - 1 || kc == nk - 1;
    if (first) mbar_wait(&tempty[buf], ((pi >> 1) & 1) ^ 1);   // epilogue drained this buffer
    mbar_wait(&full[s], ph);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t_re = tmem + buf * CF::ACC_COLS, t_im = t_re + BN;
    uint8_t* st = smem + s * CF::STAGE;
    if (elect_one()) {
#pragma unroll
    for (int ks = 0; ks < BK / 16; ++ks) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const uint64_t a_re = make_desc_sw64(st + (2 * PA[q] + 0) * CF::A_PLANE) + (uint64_t)(ks * 2);
        const uint64_t a_im = make_desc_sw64(st + (2 * PA[q] + 1) * CF::A_PLANE) + (uint64_t)(ks * 2);
        const uint64_t b_re = make_desc_sw64(st + CF::A_BYTES + (2 * PB[q] + 0) * CF::B_PLANE) + (uint64_t)(ks * 2);
        const uint64_t b_im = make_desc_sw64(st + CF::A_BYTES + (2 * PB[q] + 1) * CF::B_PLANE) + (uint64_t)(ks * 2);
        const uint32_t acc = (first && (ks | q) == 0) ? 0u : 1u;   // fresh accumulator per promotion
        mma_f16(t_re, a_re, b_re, idesc, acc);
        mma_f16(t_re, a_im, b_im, idesc_negA, 1u);
        mma_f16(t_im, a_re, b_im, idesc, acc);
        mma_f16(t_im, a_im, b_re, idesc, 1u);
      }
    }
    mma_commit(&empty[s]);                 // smem stage free once these MMAs have read it
    if (last) mma_commit(&tfull[buf]);     // accumulator buffer ready for promotion
    }
    __syncwarp();
  }
}

// Complex GEMM C[b][m][n] (+)= sum_k A[b][m][k] B[b][n][k] on block-scaled fp16x2
// operands.  Per 32-wide K stage the MMA warp issues
// 2 (k16) x 3 piece pairs (hi.hi, hi.lo, lo.hi) x 4 real products = 24 MMAs; every
// 4 stages (one 128-wide scale chunk) go into a fresh TMEM buffer, which the epilogue
// warps promote into fp32 registers, multiplying by the chunk scales sA[row] * sB[col]
// (round-to-nearest; tcgen05 fp32 accumulation truncates, so no accumulator sees more
// than 48 updates).  Two TMEM buffers ping-pong.
template <int BN>
__global__ void __launch_bounds__(Cfg<BN>::THREADS, 1)
    cgemm_f16x2s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const float* __restrict__ scA, const float* __restrict__ scB,
                        void* const* __restrict__ ptrs, int32_t c_node, int32_t M, int32_t N, int32_t K,
                        int32_t nb, int32_t kc_per_split, float2* __restrict__ partial, int32_t accumulate,
                        int32_t m_off, int32_t M_c) {
  using CF = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* sc = reinterpret_cast<float*>(smem + CF::STAGES * CF::STAGE);   // [SLOTS][BM + BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::STAGES * CF::STAGE + CF::SLOTS * CF::SC_BYTES);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* tfull = empty + CF::STAGES;     // [2] MMA -> epilogue: buffer holds a finished stage
  uint64_t* tempty = tfull + 2;             // [2] epilogue -> MMA: buffer promoted
  uint64_t* sfull = tempty + 2;             // [SLOTS] scales landed
  uint64_t* sempty = sfull + CF::SLOTS;     // [SLOTS] scales consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + CF::SLOTS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TMA_WARP = CF::EPI_WARPS, MMA_WARP = CF::EPI_WARPS + 1;
  // tile rasterization: groups of GROUP_M M-tiles sweep the N-tiles together (L2 reuse)
  const int n_tiles_m = (M + BM - 1) / BM, n_tiles_n = (N + BN - 1) / BN;
  const int pid = blockIdx.x;
  const int group_m = d_group_m > 0 ? d_group_m : GROUP_M;
  const int group = pid / (group_m * n_tiles_n);
  const int first_m = group * group_m;
  const int gm = min(n_tiles_m - first_m, group_m);
  const int m_blk = first_m + (pid % (group_m * n_tiles_n)) % gm;
  const int n_blk = (pid % (group_m * n_tiles_n)) / gm;
  // split-K: blockIdx.z = split * nb + batch; this CTA covers K chunks [kc0, kc0 + nk)
  const int b = blockIdx.z % nb, split = blockIdx.z / nb;
  const int nk_all = (K + BK - 1) / BK;
  const int kc0 = split * kc_per_split;
  const int nk = min(nk_all, kc0 + kc_per_split) - kc0;
  const int nch_all = (nk_all + PROMO - 1) / PROMO;     // scale chunks of the whole K

  if (warp == TMA_WARP && lane == 0) {
    for (int s = 0; s < CF::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], CF::EPI_WARPS); }
    for (int s = 0; s < CF::SLOTS; ++s) { mbar_init(&sfull[s], 1); mbar_init(&sempty[s], CF::EPI_WARPS); }
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
      const float* sa = scA + ((int64_t)b * nch_all) * M + m_blk * BM;
      const float* sb = scB + ((int64_t)b * nch_all) * N + n_blk * BN;
      for (int kc = 0; kc < nk; ++kc) {
        if (kc % PROMO == 0) {                  // chunk scales of this promotion
          const int pi = kc / PROMO, slot = pi % CF::SLOTS, cg = (kc0 + kc) / PROMO;
          mbar_wait(&sempty[slot], ((pi / CF::SLOTS) & 1) ^ 1);
          mbar_expect_tx(&sfull[slot], CF::SC_BYTES);
          float* d = sc + slot * (BM + BN);
          bulk_load(d, sa + (int64_t)cg * M, BM * 4, &sfull[slot]);
          bulk_load(d + BM, sb + (int64_t)cg * N, BN * 4, &sfull[slot]);
        }
        const int s = kc % CF::STAGES;
        const uint32_t ph = (kc / CF::STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], CF::STAGE);
        uint8_t* st = smem + s * CF::STAGE;
        tma_load_3d(&tmA, st, &full[s], (kc0 + kc) * BK, m_blk * BM, b * 4);               // 4 planes
        tma_load_3d(&tmB, st + CF::A_BYTES, &full[s], (kc0 + kc) * BK, n_blk * BN, b * 4); // 4 planes
      }
    }
  } else if (warp == MMA_WARP) {
    // The whole warp runs the issue loop; one elected lane issues the MMAs and commits.
    // With the whole TMEM allocated to this CTA its base is column 0: issuing with the
    // literal base keeps every MMA operand in uniform registers (no per-MMA R2UR).
    if (tmem == 0) mma_loop<BN, true>(smem, full, empty, tfull, tempty, 0u, nk);
    else mma_loop<BN, false>(smem, full, empty, tfull, tempty, tmem, nk);
  } else {
    // ---- epilogue warps: promote every stage, scaled, into fp32 registers ----
    float2* C = partial ? partial + (int64_t)split * nb * M * (int64_t)N : reinterpret_cast<float2*>(ptrs[c_node]);
    epilogue<BN, false>(reinterpret_cast<float*>(smem), warp, lane, tmem, sc, sfull, sempty, tfull, tempty, nk, K, C, b, M, N, m_blk * BM,
                        n_blk * BN, accumulate && !partial, partial ? M : M_c, partial ? 0 : m_off);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS));
}

// ------------------------------------------------------- cta_group::2 GEMM ----
// The same GEMM on CTA pairs (cluster of 2 on one TPC): the leader issues
// tcgen05.mma.cta_group::2 with M = 256 (each CTA holds 128 rows of A) and N = 128 (each
// CTA holds 64 rows of B, read by both tensor cores), so each SM streams 6 KB of
// operands per 64-cycle MMA instead of 8 KB -- the single-CTA kernel is bound by the
// shared-memory pipe (tensor reads + TMA writes), not the tensor core.  Both CTAs' TMA
// loads complete on the leader's `full` barrier; the leader's commits arrive on `empty`
// and `tfull` in both CTAs; both epilogues arrive on the leader's `tempty`.
static_assert(8 * 32 * 132 * 4 <= 3 * (4 * 128 * 32 * 2 + 4 * 128 * 32 * 2), "C staging must fit the operand stages");
struct Cfg2 {
  static constexpr int BN = 128, BNH = 64;
  static constexpr int A_PLANE = BM * BK * 2, B_PLANE = BNH * BK * 2;
  static constexpr int A_BYTES = 4 * A_PLANE, B_BYTES = 4 * B_PLANE;
  static constexpr int STAGE = A_BYTES + B_BYTES;            // 48 KB per CTA
  static constexpr int STAGES = 4;
  static constexpr int SLOTS = Cfg<128>::SLOTS, SC_BYTES = Cfg<128>::SC_BYTES;
  static constexpr int TMEM_COLS = Cfg<128>::TMEM_COLS, ACC_COLS = Cfg<128>::ACC_COLS;
  static constexpr int EPI_WARPS = 8, THREADS = 32 * (EPI_WARPS + 2);
  static constexpr int SMEM = STAGES * STAGE + SLOTS * SC_BYTES + 1024 + 512;
};

template <bool kTmem0>
__device__ __forceinline__ void mma_loop_pair(uint8_t* smem, uint64_t* full, uint64_t* empty, uint64_t* tfull,
                                              uint64_t* tempty, uint32_t tmem_rt, int nk) {
  using CF = Cfg2;
  const uint32_t tmem = kTmem0 ? 0u : tmem_rt;
  // idesc: F32 accumulate, F16 A/B, K-major both, N = 128, M = 256 (pair)
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(CF::BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  constexpr uint32_t idesc_negA = idesc | (1u << 13);
  constexpr int PA[3] = {0, 0, 1};
  constexpr int PB[3] = {0, 1, 0};
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % CF::STAGES;
    const uint32_t ph = (kc / CF::STAGES) & 1;
    const int pi = kc / PROMO;
    const int buf = pi & 1;
    const bool first = (kc % PROMO) == 0;
    const bool last = (kc % PROMO) == PROMO - 1 || kc == nk - 1;
    if (first) mbar_wait(&tempty[buf], ((pi >> 1) & 1) ^ 1);   // both epilogues drained this buffer
    mbar_wait(&full[s], ph);                                     // both CTAs' halves landed
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t_re = tmem + buf * CF::ACC_COLS, t_im = t_re + CF::BN;
    uint8_t* st = smem + s * CF::STAGE;
    if (elect_one()) {
#pragma unroll
      for (int ks = 0; ks < BK / 16; ++ks) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const uint64_t a_re = make_desc_sw64(st + (2 * PA[q] + 0) * CF::A_PLANE) + (uint64_t)(ks * 2);
          const uint64_t a_im = make_desc_sw64(st + (2 * PA[q] + 1) * CF::A_PLANE) + (uint64_t)(ks * 2);
          const uint64_t b_re = make_desc_sw64(st + CF::A_BYTES + (2 * PB[q] + 0) * CF::B_PLANE) + (uint64_t)(ks * 2);
          const uint64_t b_im = make_desc_sw64(st + CF::A_BYTES + (2 * PB[q] + 1) * CF::B_PLANE) + (uint64_t)(ks * 2);
          const uint32_t acc = (first && (ks | q) == 0) ? 0u : 1u;
          mma_f16_pair(t_re, a_re, b_re, idesc, acc);
          mma_f16_pair(t_re, a_im, b_im, idesc_negA, 1u);
          mma_f16_pair(t_im, a_re, b_im, idesc, acc);
          mma_f16_pair(t_im, a_im, b_re, idesc, 1u);
        }
      }
      mma_commit_pair(&empty[s]);                 // both CTAs' stage s free
      if (last) mma_commit_pair(&tfull[buf]);     // both CTAs' accumulators ready
    }
    __syncwarp();
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2::THREADS, 1)
    cgemm2_f16x2s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const float* __restrict__ scA, const float* __restrict__ scB,
                         void* const* __restrict__ ptrs, int32_t c_node, int32_t M, int32_t N, int32_t K,
                         int32_t nb, int32_t kc_per_split, float2* __restrict__ partial, int32_t accumulate,
                         int32_t m_off, int32_t M_c, const __grid_constant__ CUtensorMap tmC, int32_t k_base) {
  using CF = Cfg2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* sc = reinterpret_cast<float*>(smem + CF::STAGES * CF::STAGE);   // [SLOTS][BM + BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::STAGES * CF::STAGE + CF::SLOTS * CF::SC_BYTES);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* tfull = empty + CF::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + CF::SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + CF::SLOTS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TMA_WARP = CF::EPI_WARPS, MMA_WARP = CF::EPI_WARPS + 1;
  const uint32_t rank = cluster_ctarank();
  // pair rasterization: groups of GROUP_M 256-row tiles sweep the N tiles together
  const int n_tiles_m = (M + 255) / 256, n_tiles_n = N / CF::BN;
  const int pid = blockIdx.x >> 1;
  const int group_m = d_group_m > 0 ? d_group_m : GROUP_M_PAIR;
  const int group = pid / (group_m * n_tiles_n);
  const int first_m = group * group_m;
  const int gm = min(n_tiles_m - first_m, group_m);
  const int m_blk = first_m + (pid % (group_m * n_tiles_n)) % gm;
  const int n_fwd = (pid % (group_m * n_tiles_n)) / gm;
  const int n_blk = (d_serp && (group & 1)) ? n_tiles_n - 1 - n_fwd : n_fwd;
  const int row0 = m_blk * 256 + (int)rank * BM;
  const int b = blockIdx.z % nb, split = blockIdx.z / nb;
  const int nk_all = (K + BK - 1) / BK;
  const int kc0 = k_base + split * kc_per_split;     // k_base: K-chunk of a long-K step (stages)
  const int nk = min(nk_all, kc0 + kc_per_split) - kc0;
  const int nch_all = (nk_all + PROMO - 1) / PROMO;

  if (warp == TMA_WARP && lane == 0) {
    for (int s = 0; s < CF::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * CF::EPI_WARPS); }
    for (int s = 0; s < CF::SLOTS; ++s) { mbar_init(&sfull[s], 1); mbar_init(&sempty[s], CF::EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();          // the peer's barriers are initialised before any remote use
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == TMA_WARP) {
    if (lane == 0) {
      const float* sa = scA + ((int64_t)b * nch_all) * M + row0;
      const float* sb = scB + ((int64_t)b * nch_all) * N + n_blk * CF::BN;
      for (int kc = 0; kc < nk; ++kc) {
        if (kc % PROMO == 0) {                  // this CTA's rows' and the tile's column scales
          const int pi = kc / PROMO, slot = pi % CF::SLOTS, cg = (kc0 + kc) / PROMO;
          mbar_wait(&sempty[slot], ((pi / CF::SLOTS) & 1) ^ 1);
          mbar_expect_tx(&sfull[slot], CF::SC_BYTES);
          float* d = sc + slot * (BM + CF::BN);
          bulk_load(d, sa + (int64_t)cg * M, BM * 4, &sfull[slot]);
          bulk_load(d + BM, sb + (int64_t)cg * N, CF::BN * 4, &sfull[slot]);
        }
        const int s = kc % CF::STAGES;
        const uint32_t ph = (kc / CF::STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        if (rank == 0) mbar_expect_tx(&full[s], 2 * CF::STAGE);     // both CTAs' bytes
        const uint32_t fb = mapa_rank0(&full[s]);
        uint8_t* st = smem + s * CF::STAGE;
        tma_load_3d_pair(&tmA, st, fb, (kc0 + kc) * BK, row0, b * 4);
        tma_load_3d_pair(&tmB, st + CF::A_BYTES, fb, (kc0 + kc) * BK, n_blk * CF::BN + (int)rank * CF::BNH, b * 4);
      }
    }
  } else if (warp == MMA_WARP) {
    if (rank == 0) {
      if (tmem == 0) mma_loop_pair<true>(smem, full, empty, tfull, tempty, 0u, nk);
      else mma_loop_pair<false>(smem, full, empty, tfull, tempty, tmem, nk);
    }
  } else {
    float2* C = partial ? partial + (int64_t)split * nb * M * (int64_t)N : reinterpret_cast<float2*>(ptrs[c_node]);
    epilogue<128, true>(reinterpret_cast<float*>(smem), warp, lane, tmem, sc, sfull, sempty, tfull, tempty, nk, K, C, b, M, N, row0,
                        n_blk * CF::BN, accumulate && !partial, partial ? M : M_c, partial ? 0 : m_off,
                        partial ? nullptr : &tmC);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();          // no CTA leaves while its peer may still signal or read it
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS));
  }
}

// ------------------------------------------------ persistent CTA-pair GEMM ----
// cgemm2 as a persistent kernel: one CTA pair per TPC loops over the output tiles
// (batch, split, 256 x 128 tile), so the TMA producer prefetches tile i + 1 while the
// epilogue of tile i runs, and the MMA warp starts tile i + 1 in the TMEM buffer the
// epilogue has released -- the per-CTA prologue/fill/drain of the one-tile-per-CTA
// kernel (a third of the time of a K = 256 step) disappears.  All three roles walk the
// same tile sequence with global stage / promotion counters.  C leaves through a
// dedicated 64 KB staging area by TMA tensor stores (reduce-add for C += of K-slabs): each
// epilogue warp stages 32 rows x 16 complex per box (SWIZZLE_128B, conflict-free) in two
// alternating buffers and one lane issues the store, so the warps return to promoting
// the next tile while the TMA engine drains C (thread stores of C cost a third of a
// K = 256 step).  3 operand stages instead of 4 make room for the staging.
struct Cfg2P {
  static constexpr int STAGES = 3;                                     // short-K tiles: 3 operand stages
  static constexpr int STG_WARP = 2 * 32 * 128;                        // 2 TMA-store boxes of 32 rows x 16 complex
  static constexpr int STG_BYTES = Cfg2::EPI_WARPS * STG_WARP;         // 64 KB
  static constexpr int STG_PITCH = 68;                                 // split-K partial path: 8 rows x 32 complex + pad
  static constexpr int SMEM = STAGES * Cfg2::STAGE + Cfg2::SLOTS * Cfg2::SC_BYTES + STG_BYTES + 1024 + 512;
};

template <bool kTmem0>
__device__ __forceinline__ void mma_tiles_pair(uint8_t* smem, uint64_t* full, uint64_t* empty, uint64_t* tfull,
                                               uint64_t* tempty, uint32_t tmem_rt, int pair, int n_pairs, int total,
                                               int tiles_per_z, int nb, int nk_all, int kc_per_split) {
  using CF = Cfg2;
  const uint32_t tmem = kTmem0 ? 0u : tmem_rt;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(CF::BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  constexpr uint32_t idesc_negA = idesc | (1u << 13);
  constexpr int PA[3] = {0, 0, 1};
  constexpr int PB[3] = {0, 1, 0};
  int g = 0, gp = 0;                      // global stage / promotion counters
  for (int tile = pair; tile < total; tile += n_pairs) {
    const int split = (tile / tiles_per_z) / nb;
    const int kc0 = split * kc_per_split;
    const int nk = min(nk_all, kc0 + kc_per_split) - kc0;
    for (int kc = 0; kc < nk; ++kc, ++g) {
      const int s = g % Cfg2P::STAGES;
      const uint32_t ph = (g / Cfg2P::STAGES) & 1;
      const bool first = (kc % PROMO) == 0;
      const bool last = (kc % PROMO) == PROMO - 1 || kc == nk - 1;
      const int buf = gp & 1;
      if (first) mbar_wait(&tempty[buf], ((gp >> 1) & 1) ^ 1);
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t t_re = tmem + buf * CF::ACC_COLS, t_im = t_re + CF::BN;
      uint8_t* st = smem + s * CF::STAGE;
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < BK / 16; ++ks) {
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const uint64_t a_re = make_desc_sw64(st + (2 * PA[q] + 0) * CF::A_PLANE) + (uint64_t)(ks * 2);
            const uint64_t a_im = make_desc_sw64(st + (2 * PA[q] + 1) * CF::A_PLANE) + (uint64_t)(ks * 2);
            const uint64_t b_re = make_desc_sw64(st + CF::A_BYTES + (2 * PB[q] + 0) * CF::B_PLANE) + (uint64_t)(ks * 2);
            const uint64_t b_im = make_desc_sw64(st + CF::A_BYTES + (2 * PB[q] + 1) * CF::B_PLANE) + (uint64_t)(ks * 2);
            const uint32_t acc = (first && (ks | q) == 0) ? 0u : 1u;
            mma_f16_pair(t_re, a_re, b_re, idesc, acc);
            mma_f16_pair(t_re, a_im, b_im, idesc_negA, 1u);
            mma_f16_pair(t_im, a_re, b_im, idesc, acc);
            mma_f16_pair(t_im, a_im, b_re, idesc, 1u);
          }
        }
        mma_commit_pair(&empty[s]);
        if (last) mma_commit_pair(&tfull[buf]);
      }
      __syncwarp();
      if (last) ++gp;
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2::THREADS, 1)
    cgemm2p_f16x2s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const float* __restrict__ scA, const float* __restrict__ scB,
                          void* const* __restrict__ ptrs, int32_t c_node, int32_t M, int32_t N, int32_t K,
                          int32_t nb, int32_t S, int32_t kc_per_split, float2* __restrict__ partial,
                          int32_t accumulate, int32_t m_off, int32_t M_c, const __grid_constant__ CUtensorMap tmC) {
  using CF = Cfg2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* sc = reinterpret_cast<float*>(smem + Cfg2P::STAGES * CF::STAGE);   // [SLOTS][BM + BN]
  float* stg = sc + CF::SLOTS * (BM + CF::BN);                          // [EPI_WARPS][STG_WARP bytes]
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + Cfg2P::STG_BYTES);
  uint64_t* empty = full + Cfg2P::STAGES;
  uint64_t* tfull = empty + Cfg2P::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + CF::SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + CF::SLOTS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TMA_WARP = CF::EPI_WARPS, MMA_WARP = CF::EPI_WARPS + 1;
  const uint32_t rank = cluster_ctarank();
  const int n_tiles_m = (M + 255) / 256, n_tiles_n = N / CF::BN;
  const int tiles_per_z = n_tiles_m * n_tiles_n;
  const int total = tiles_per_z * nb * S;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int nk_all = (K + BK - 1) / BK;
  const int nch_all = (nk_all + PROMO - 1) / PROMO;
  // tile -> (batch, split, m_blk, n_blk): groups of GROUP_M 256-row tiles sweep the N tiles
  auto tile_coords = [&](int tile, int& b, int& split, int& m_blk, int& n_blk) {
    const int z = tile / tiles_per_z, pid = tile % tiles_per_z;
    b = z % nb;
    split = z / nb;
    const int group_m = d_group_m > 0 ? d_group_m : GROUP_M_PERSIST;
    const int group = pid / (group_m * n_tiles_n);
    const int first_m = group * group_m;
    const int gm = min(n_tiles_m - first_m, group_m);
    m_blk = first_m + (pid % (group_m * n_tiles_n)) % gm;
    n_blk = (pid % (group_m * n_tiles_n)) / gm;
  };

  if (warp == TMA_WARP && lane == 0) {
    for (int s = 0; s < Cfg2P::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * CF::EPI_WARPS); }
    for (int s = 0; s < CF::SLOTS; ++s) { mbar_init(&sfull[s], 1); mbar_init(&sempty[s], CF::EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == TMA_WARP) {
    if (lane == 0) {
      int g = 0, gp = 0;
      for (int tile = pair; tile < total; tile += n_pairs) {
        int b, split, m_blk, n_blk;
        tile_coords(tile, b, split, m_blk, n_blk);
        const int row0 = m_blk * 256 + (int)rank * BM;
        const int kc0 = split * kc_per_split;
        const int nk = min(nk_all, kc0 + kc_per_split) - kc0;
        const float* sa = scA + ((int64_t)b * nch_all) * M + row0;
        const float* sb = scB + ((int64_t)b * nch_all) * N + n_blk * CF::BN;
        for (int kc = 0; kc < nk; ++kc, ++g) {
          if (kc % PROMO == 0) {
            const int slot = gp % CF::SLOTS, cg = (kc0 + kc) / PROMO;
            mbar_wait(&sempty[slot], ((gp / CF::SLOTS) & 1) ^ 1);
            mbar_expect_tx(&sfull[slot], CF::SC_BYTES);
            float* d = sc + slot * (BM + CF::BN);
            bulk_load(d, sa + (int64_t)cg * M, BM * 4, &sfull[slot]);
            bulk_load(d + BM, sb + (int64_t)cg * N, CF::BN * 4, &sfull[slot]);
            ++gp;
          }
          const int s = g % Cfg2P::STAGES;
          const uint32_t ph = (g / Cfg2P::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * CF::STAGE);
          const uint32_t fb = mapa_rank0(&full[s]);
          uint8_t* st = smem + s * CF::STAGE;
          tma_load_3d_pair(&tmA, st, fb, (kc0 + kc) * BK, row0, b * 4);
          tma_load_3d_pair(&tmB, st + CF::A_BYTES, fb, (kc0 + kc) * BK, n_blk * CF::BN + (int)rank * CF::BNH, b * 4);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    if (rank == 0) {
      if (tmem == 0) mma_tiles_pair<true>(smem, full, empty, tfull, tempty, 0u, pair, n_pairs, total, tiles_per_z, nb, nk_all, kc_per_split);
      else mma_tiles_pair<false>(smem, full, empty, tfull, tempty, tmem, pair, n_pairs, total, tiles_per_z, nb, nk_all, kc_per_split);
    }
  } else {
    // ---- epilogue warps ----
    const int lg = warp & 3, ch = warp >> 2;
    const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
    float* my_stg = stg + warp * (Cfg2P::STG_WARP / 4);
    int sb = 0;                                // TMA-store boxes issued by this warp
    int gp = 0;
    for (int tile = pair; tile < total; tile += n_pairs) {
      int b, split, m_blk, n_blk;
      tile_coords(tile, b, split, m_blk, n_blk);
      const int row0 = m_blk * 256 + (int)rank * BM;
      const int kc0 = split * kc_per_split;
      const int nk = min(nk_all, kc0 + kc_per_split) - kc0;
      const int n_promo = (nk + PROMO - 1) / PROMO;
      float ar[64], ai[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) { ar[j] = 0.f; ai[j] = 0.f; }
      for (int p = 0; p < n_promo; ++p, ++gp) {
        const int buf = gp & 1, slot = gp % CF::SLOTS;
        mbar_wait(&sfull[slot], (gp / CF::SLOTS) & 1);
        mbar_wait(&tfull[buf], (gp >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t scs = smem_u32(sc + slot * (BM + CF::BN));
        const float sa = lds_f32(scs + 4 * (lg * 32 + lane)) * rz_debias(min(PROMO, nk - p * PROMO), K);
        const float sb_lo = lds_f32(scs + 4 * (BM + ch * 64 + lane));
        const float sb_hi = lds_f32(scs + 4 * (BM + ch * 64 + 32 + lane));
        const uint32_t t_re = tmem + buf * CF::ACC_COLS + lane_base + ch * 64, t_im = t_re + CF::BN;
#pragma unroll
        for (int c = 0; c < 64; c += 8) {
          uint32_t vr[8], vi[8];
          tmem_ld8(t_re + c, vr);
          tmem_ld8(t_im + c, vi);
          float sbl[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) sbl[j] = __shfl_sync(0xffffffffu, (c + j) < 32 ? sb_lo : sb_hi, (c + j) & 31);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float sv = sa * sbl[j];
            ar[c + j] = __fmaf_rn(__uint_as_float(vr[j]), sv, ar[c + j]);
            ai[c + j] = __fmaf_rn(__uint_as_float(vi[j]), sv, ai[c + j]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(mapa_rank0(&tempty[buf]));
          mbar_arrive(&sempty[slot]);
        }
      }
      // C tile rows [row0 + 32 lg, +32) x columns [n_blk 128 + 64 ch, +64) in 8 rounds of
      // 8 rows x 32 complex: the 8 lanes owning the rows stage 256 B each, then 16 lanes
      // per row store whole 256-byte row segments (2 rows, 4 full lines per instruction)
      float2* C;
      int c_rows, c_row_off;
      if (partial) { C = partial + (int64_t)split * nb * M * (int64_t)N; c_rows = M; c_row_off = 0; }
      else { C = reinterpret_cast<float2*>(ptrs[c_node]); c_rows = M_c; c_row_off = m_off; }
      const bool acc_c = accumulate && !partial;
      const int rbase = row0 + lg * 32, col0 = n_blk * CF::BN + ch * 64;
      const uint32_t stg_u = smem_u32(my_stg);
      if (!partial) {
        // 4 boxes of 32 rows x 16 complex (128-byte rows, 16-byte chunk j of row r at
        // j ^ (r & 7): the SWIZZLE_128B layout of the C tensor map)
        const int y = b * c_rows + c_row_off + rbase;
#pragma unroll
        for (int q = 0; q < 4; ++q, ++sb) {
          const uint32_t buf = stg_u + (sb & 1) * (32 * 128);
          if (lane == 0) bulk_wait_read1();        // the box stored from this buffer 2 rounds ago is read
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            sts128(buf + lane * 128 + ((j ^ (lane & 7)) << 4),
                   make_float4(ar[16 * q + 2 * j], ai[16 * q + 2 * j], ar[16 * q + 2 * j + 1], ai[16 * q + 2 * j + 1]));
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (acc_c) tma_reduce_add_2d(&tmC, buf, 2 * (col0 + 16 * q), y);
            else tma_store_2d(&tmC, buf, 2 * (col0 + 16 * q), y);
            bulk_commit();
          }
        }
        continue;
      }
      // split-K partials: thread stores through the staging area
      constexpr int P = Cfg2P::STG_PITCH;
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if ((lane >> 3) == g) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            sts128(stg_u + 4 * ((lane & 7) * P + 4 * j),
                   make_float4(ar[32 * h + 2 * j], ai[32 * h + 2 * j], ar[32 * h + 2 * j + 1], ai[32 * h + 2 * j + 1]));
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = 2 * i + (lane >> 4), r = 8 * g + rr;
          if (rbase + r < M) {
            float4 v = lds128(stg_u + 4 * (rr * P + 4 * (lane & 15)));
            float4* dst = reinterpret_cast<float4*>(C + ((int64_t)b * c_rows + c_row_off + rbase + r) * (int64_t)N +
                                                    col0 + 32 * h) + (lane & 15);
            if (acc_c) {
              const float4 o = ldg128(dst);
              v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
            }
            stg128(dst, v);
          }
        }
        __syncwarp();
      }
    }
    if (lane == 0) bulk_wait_all();              // C fully written before the CTA exits
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS));
  }
}

}  // namespace tc

// C[i] = sum_s partial[s][i], summed in fp64 (split-K epilogue)
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float2* __restrict__ partial, int32_t S,
                                                            int64_t n, void* const* __restrict__ ptrs, int32_t c_node,
                                                            int32_t accumulate) {
  float2* C = reinterpret_cast<float2*>(ptrs[c_node]);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double re = 0.0, im = 0.0;
    if (accumulate) {
      const float2 c = C[i];
      re = c.x;
      im = c.y;
    }
    for (int s = 0; s < S; ++s) {
      const float2 v = partial[(int64_t)s * n + i];
      re += v.x;
      im += v.y;
    }
    C[i] = make_float2((float)re, (float)im);
  }
}
}  // namespace tnd
