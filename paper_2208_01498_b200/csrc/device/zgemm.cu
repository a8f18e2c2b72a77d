// complex128 GEMM-shaped steps on the FP64 tensor pipe (DMMA).
//   C[b][m][n] = sum_k A[b][m][k] * B[b][k][n]     (Eq. (3), l.82-86)
// tcgen05 has no f64 kind; sm_100a's FP64 tensor instructions are mma.sync
// m16n8k4 f64 (SASS DMMA.8x8x4).  Operands come from the fp64 variant of the tiled
// transpose pack: 2 planes (re, im) of [b][rows][K]; complex arithmetic is planar,
// Cr += Ar.Br + (-Ai).Bi, Ci += Ar.Bi + Ai.Br, accumulated in fp64 registers.
// CTA tile 64 x 64 complex, 8 warps of 32 x 16, K staged 16 at a time through a
// 2-stage cp.async ring with an XOR swizzle of 16-byte chunks (conflict-free-ish
// fragment loads).
#include "common.cuh"

namespace tnd {

// DMMA operands are packed by pack_planar_kernel<double> (skinny.cu): planes
// [b][2][rows][K] (re plane, im plane) of fp64.

// ------------------------------------------------------------------ DMMA -----
namespace zg {
constexpr int BM = 64, BN = 64, BK = 16, THREADS = 256, STAGES = 3;
constexpr int PLANE_TILE = BM * BK;                       // doubles per plane per tile (BM == BN)
constexpr int STAGE_DOUBLES = 4 * PLANE_TILE;             // A re, A im, B re, B im
constexpr int SMEM = STAGES * STAGE_DOUBLES * 8;          // 96 KB (2 CTAs per SM)
constexpr int GROUP_M = 8;

__device__ __forceinline__ int swz(int row, int col) {      // col in doubles (0..15)
  return row * BK + ((((col >> 1) ^ (row & 7)) << 1) | (col & 1));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// A planes: [b][2][M][K], B planes: [b][2][N][K] (fp64, K contiguous)
__global__ void __launch_bounds__(THREADS, 2) zgemm_dmma_kernel(const double* __restrict__ Ap, const double* __restrict__ Bp,
                                                             void* const* __restrict__ ptrs, int32_t c_node, int32_t M,
                                                             int32_t N, int32_t K) {
  extern __shared__ __align__(16) double sm[];
  const int n_tiles_m = (M + BM - 1) / BM, n_tiles_n = (N + BN - 1) / BN;
  const int pid = blockIdx.x;
  const int group = pid / (GROUP_M * n_tiles_n);
  const int first_m = group * GROUP_M;
  const int gm = min(n_tiles_m - first_m, GROUP_M);
  const int m_blk = first_m + (pid % (GROUP_M * n_tiles_n)) % gm;
  const int n_blk = (pid % (GROUP_M * n_tiles_n)) / gm;
  const int b = blockIdx.z;
  const double* A = Ap + (int64_t)b * 2 * M * (int64_t)K;
  const double* B = Bp + (int64_t)b * 2 * N * (int64_t)K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;   // 8 warps of 32 x 16
  const int g = lane >> 2, t = lane & 3;

  auto load_stage = [&](int stage, int k0) {
    double* st = sm + stage * STAGE_DOUBLES;
    // 4 planes x 64 rows x 8 chunks of 16 B = 2048 chunks, 8 per thread
#pragma unroll
    for (int i = 0; i < 2048 / THREADS; ++i) {
      const int c = threadIdx.x + i * THREADS;
      const int plane = c >> 9;                  // 0: A re, 1: A im, 2: B re, 3: B im
      const int row = (c >> 3) & 63;
      const int ch = c & 7;
      const bool isA = plane < 2;
      const int grow = (isA ? m_blk * BM : n_blk * BN) + row;
      const int gk = k0 + ch * 2;
      const bool valid = grow < (isA ? M : N) && gk < K;
      const double* base = isA ? A + (int64_t)(plane & 1) * M * K : B + (int64_t)(plane & 1) * N * K;
      const double* src = valid ? base + (int64_t)grow * K + gk : base;
      cp_async16(st + plane * PLANE_TILE + row * BK + ((ch ^ (row & 7)) << 1), src, valid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  double cr[2][2][4], ci[2][2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) { cr[i][j][r] = 0.0; ci[i][j][r] = 0.0; }

  const int nk = (K + BK - 1) / BK;
  // STAGES-deep cp.async ring: stages kc + 1 .. kc + STAGES - 1 are in flight while stage
  // kc is consumed (one commit group per stage, empty groups past the end keep the count)
#pragma unroll
  for (int p = 0; p < STAGES - 1; ++p) {
    if (p < nk) load_stage(p, p * BK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kc = 0; kc < nk; ++kc) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    if (kc + STAGES - 1 < nk) load_stage((kc + STAGES - 1) % STAGES, (kc + STAGES - 1) * BK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const double* st = sm + (kc % STAGES) * STAGE_DOUBLES;
    const double* sAr = st;
    const double* sAi = st + PLANE_TILE;
    const double* sBr = st + 2 * PLANE_TILE;
    const double* sBi = st + 3 * PLANE_TILE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[2][2], ai[2][2], nai[2][2], br[2], bi[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r0 = wm + i * 16 + g;
        ar[i][0] = sAr[swz(r0, kk + t)];
        ar[i][1] = sAr[swz(r0 + 8, kk + t)];
        ai[i][0] = sAi[swz(r0, kk + t)];
        ai[i][1] = sAi[swz(r0 + 8, kk + t)];
        nai[i][0] = -ai[i][0];
        nai[i][1] = -ai[i][1];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n0 = wn + j * 8 + g;
        br[j] = sBr[swz(n0, kk + t)];
        bi[j] = sBi[swz(n0, kk + t)];
      }
      // the two products into one accumulator are 2 * 4 DMMAs apart (one pass per
      // product term over every accumulator): back-to-back dependent DMMAs would stall
      // each warp for the pipe's full latency
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(cr[i][j], ar[i][0], ar[i][1], br[j]);
          dmma(ci[i][j], ar[i][0], ar[i][1], bi[j]);
        }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(cr[i][j], nai[i][0], nai[i][1], bi[j]);
          dmma(ci[i][j], ai[i][0], ai[i][1], br[j]);
        }
    }
  }
  double2* C = reinterpret_cast<double2*>(ptrs[c_node]) + (int64_t)b * M * (int64_t)N;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = m_blk * BM + wm + i * 16 + g + 8 * h;
        const int col = n_blk * BN + wn + j * 8 + 2 * t;
        if (row < M && col < N) {
          double2* cp = C + (int64_t)row * N + col;
          cp[0] = double2{cr[i][j][2 * h], ci[i][j][2 * h]};
          if (col + 1 < N) cp[1] = double2{cr[i][j][2 * h + 1], ci[i][j][2 * h + 1]};
        }
      }
}

// ----------------------------------------------------------- DMMA, gathered ----
// The same GEMM reading the raw operands (interleaved complex128, any stored index order)
// straight from the producing steps: the permutation to matricised form is folded into
// the cp.async tile loads through GroupMap offset tables (as the small path does), so the
// step has no pack pass (configs[3]: the planar packs were 28% of an amplitude).  Per CTA
// the 64 row offsets of A and of B are computed once into shared memory; per stage each
// thread gathers 16-byte complex elements, row-fastest or K-fastest along whichever is
// contiguous in the operand's stored layout (kfast flags, chosen on the host) so a warp's
// requests stay coalesced.  Tiles are interleaved [row][k] complex in shared memory with
// the 16-byte column XOR-swizzled by (row & 7): the DMMA fragment loads (8 rows x 4 k per
// warp, one LDS.128 = re + im) are conflict-free.
using tnd::GatherMaps;
constexpr int G_KTAB = 1024;                              // K offsets tabulated per CTA up to this K
// tiles of 64 x BNT complex (BNT = 64, or 32 when a step's 64-wide tiles would leave a
// partial last wave: configs[3]'s dominant step, 1024 tiles = 3.46 waves of 296 slots)
template <int BNT>
__host__ __device__ constexpr int g_stage() { return (BM + BNT) * BK; }      // complex128 per stage (A and B tiles)
template <int BNT>
__host__ __device__ constexpr int g_smem() { return STAGES * g_stage<BNT>() * 16 + (BM + BNT) * 8 + 2 * G_KTAB * 8; }

// ksplit in {2, 4} (the tail launch of a step whose tiles leave a partial last wave): the
// ksplit CTAs of one tile form a cluster along y, each contracts a contiguous 1/ksplit of K,
// and the leader (cluster rank 0) adds the others' accumulators from their shared memory
// (DSMEM) in rank order -- deterministic, no zeroing pass, no atomics, no extra C traffic.
// tile0: first linear tile (batch-major) of this launch; grid.x tiles, grid.y = ksplit.
template <int BNT>
__global__ void __launch_bounds__(THREADS, 2) zgemm_dmma_gather_kernel(const GatherMaps gm_, const int64_t* __restrict__ tab,
                                                                    void* const* __restrict__ ptrs, int32_t c_node,
                                                                    int32_t M, int32_t N, int32_t K, int32_t ksplit,
                                                                    int64_t tile0) {
  constexpr int G_STAGE = g_stage<BNT>();
  constexpr int WN = BNT / 16, WM = 8 / WN;              // warp grid (N x M), warp tile 16 x (BM / WM)
  constexpr int MI = BM / WM / 16;                        // 16-row fragments per warp
  extern __shared__ __align__(16) double2 smz[];
  int64_t* rowA = reinterpret_cast<int64_t*>(smz + STAGES * G_STAGE);
  int64_t* rowB = rowA + BM;
  int64_t* kA = rowB + BNT;                     // K offsets of A and B (K <= G_KTAB)
  int64_t* kB = kA + G_KTAB;
  const bool ktab = K <= G_KTAB;
  if (ktab)
    for (int k = threadIdx.x; k < K; k += THREADS) {
      kA[k] = gmap(tab, gm_.Ak, k);
      kB[k] = gmap(tab, gm_.Bk, k);
    }
  const int n_tiles_m = (M + BM - 1) / BM, n_tiles_n = (N + BNT - 1) / BNT;
  const int64_t lt = tile0 + blockIdx.x;                 // linear tile: batch-major
  const int b = (int)(lt / (n_tiles_m * n_tiles_n));
  const int pid = (int)(lt % (n_tiles_m * n_tiles_n));
  const int group = pid / (GROUP_M * n_tiles_n);
  const int first_m = group * GROUP_M;
  const int gmr = min(n_tiles_m - first_m, GROUP_M);
  const int m_blk = first_m + (pid % (GROUP_M * n_tiles_n)) % gmr;
  const int n_blk = (pid % (GROUP_M * n_tiles_n)) / gmr;
  const double2* __restrict__ A = reinterpret_cast<const double2*>(ptrs[gm_.a_node]);
  const double2* __restrict__ B = reinterpret_cast<const double2*>(ptrs[gm_.b_node]);
  if (threadIdx.x < BM) {
    const int r = m_blk * BM + threadIdx.x;
    rowA[threadIdx.x] = r < M ? gmap(tab, gm_.Ab, b) + gmap(tab, gm_.Am, r) : -1;
  } else if (threadIdx.x < BM + BNT) {
    const int r = n_blk * BNT + threadIdx.x - BM;
    rowB[threadIdx.x - BM] = r < N ? gmap(tab, gm_.Bb, b) + gmap(tab, gm_.Bn, r) : -1;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp / WN) * (BM / WM), wn = (warp % WN) * 16;
  const int g = lane >> 2, t = lane & 3;

  auto load_stage = [&](int stage, int k0) {
    double2* st = smz + stage * G_STAGE;
    // (64 + BNT) rows x 16 k complex: A then B, (64 + BNT) * 16 / 256 per thread
#pragma unroll
    for (int i = 0; i < (BM + BNT) * BK / THREADS; ++i) {
      const int c = threadIdx.x + i * THREADS;
      const int op = c >= BM * BK, e = op ? c - BM * BK : c;
      const int rows = op ? BNT : BM;
      const bool kf = op ? gm_.b_kfast : gm_.a_kfast;
      const int row = kf ? e >> 4 : e & (rows - 1);
      const int kk = kf ? e & 15 : e / rows;
      const int gk = k0 + kk;
      const int64_t ro = op ? rowB[row] : rowA[row];
      const bool valid = ro >= 0 && gk < K;
      const double2* base = op ? B : A;
      const double2* src = !valid ? base
                           : base + ro + (ktab ? (op ? kB[gk] : kA[gk]) : gmap(tab, op ? gm_.Bk : gm_.Ak, gk));
      cp_async16(st + op * BM * BK + row * BK + (kk ^ (row & 7)), src, valid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  double cr[MI][2][4], ci[MI][2][4];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) { cr[i][j][r] = 0.0; ci[i][j][r] = 0.0; }

  const int kbeg = ksplit > 1 ? (int)blockIdx.y * (K / ksplit) : 0;
  const int nk = ((ksplit > 1 ? K / ksplit : K) + BK - 1) / BK;
#pragma unroll
  for (int p = 0; p < STAGES - 1; ++p) {
    if (p < nk) load_stage(p, kbeg + p * BK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kc = 0; kc < nk; ++kc) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    if (kc + STAGES - 1 < nk) load_stage((kc + STAGES - 1) % STAGES, kbeg + (kc + STAGES - 1) * BK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const double2* sA = smz + (kc % STAGES) * G_STAGE;
    const double2* sB = sA + BM * BK;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[MI][2], ai[MI][2], nai[MI][2], br[2], bi[2];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r0 = wm + i * 16 + g;
        const double2 v0 = sA[r0 * BK + ((kk + t) ^ (r0 & 7))];
        const double2 v1 = sA[(r0 + 8) * BK + ((kk + t) ^ ((r0 + 8) & 7))];
        ar[i][0] = v0.x; ai[i][0] = v0.y; ar[i][1] = v1.x; ai[i][1] = v1.y;
        nai[i][0] = -ai[i][0];
        nai[i][1] = -ai[i][1];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n0 = wn + j * 8 + g;
        const double2 w = sB[n0 * BK + ((kk + t) ^ (n0 & 7))];
        br[j] = w.x;
        bi[j] = w.y;
      }
      // the two products into one accumulator are MI * 4 DMMAs apart (one pass per
      // product term over every accumulator): back-to-back dependent DMMAs would stall
      // each warp for the pipe's full latency
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(cr[i][j], ar[i][0], ar[i][1], br[j]);
          dmma(ci[i][j], ar[i][0], ar[i][1], bi[j]);
        }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(cr[i][j], nai[i][0], nai[i][1], bi[j]);
          dmma(ci[i][j], ai[i][0], ai[i][1], br[j]);
        }
    }
  }
  if (ksplit > 1) {
    // K-split cluster: the other ranks park their accumulators in their (now idle) stage
    // buffers, the leader adds them in rank order over DSMEM
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    uint32_t crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    double* red = reinterpret_cast<double*>(smz);           // [2 * MI * 2 * 4][THREADS]
    static_assert(2 * MI * 2 * 4 * THREADS * 8 <= STAGES * G_STAGE * 16, "reduction buffer");
    if (crank != 0) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            red[((i * 2 + j) * 8 + r) * THREADS + threadIdx.x] = cr[i][j][r];
            red[((i * 2 + j) * 8 + 4 + r) * THREADS + threadIdx.x] = ci[i][j][r];
          }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (crank == 0) {
      for (int q = 1; q < ksplit; ++q) {
        uint32_t base;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(base)
                     : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(red + threadIdx.x))), "r"(q));
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              double vr, vi;
              asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(vr) : "r"(base + ((i * 2 + j) * 8 + r) * THREADS * 8));
              asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(vi) : "r"(base + ((i * 2 + j) * 8 + 4 + r) * THREADS * 8));
              cr[i][j][r] += vr;
              ci[i][j][r] += vi;
            }
      }
    }
    // no rank leaves (its shared memory) before the leader has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (crank != 0) return;
  }
  double2* C = reinterpret_cast<double2*>(ptrs[c_node]) + (int64_t)b * M * (int64_t)N;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = m_blk * BM + wm + i * 16 + g + 8 * h;
        const int col = n_blk * BNT + wn + j * 8 + 2 * t;
        if (row < M && col < N) {
          double2* cp = C + (int64_t)row * N + col;
          cp[0] = double2{cr[i][j][2 * h], ci[i][j][2 * h]};
          if (col + 1 < N) cp[1] = double2{cr[i][j][2 * h + 1], ci[i][j][2 * h + 1]};
        }
      }
}
}  // namespace zg
}  // namespace tnd
