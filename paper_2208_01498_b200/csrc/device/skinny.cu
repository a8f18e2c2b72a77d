// CUDA-core paths for the large steps that are not GEMM-shaped enough for the tensor
// cores (Eq. (3), l.82-86: a step costs M = prod of all its index dimensions):
//   * skinny: few outputs (M, N <= 64, M N <= 256 per batch) and a long contraction
//     (K >= 2^10) -- HBM-bound on READING the operands once;
//   * wide:   short contraction (K <= 16) and a large output -- HBM-bound on WRITING C.
// Both read operands that the planar pack (pack_planar_kernel, the same smem-tiled
// bit-permutation transpose as the tensor-core packs) has put in [b][re|im][rows][K]
// layout, K contiguous, so every load is coalesced; accumulation is fp64.
#include <type_traits>

#include "common.cuh"

namespace tnd {

// ------------------------------------------------------------ planar pack ----
// Output planes [b][2][rows][K] of R: (re plane, im plane); the host built tile_dst /
// q_hi for 2 planes per batch (see PackDesc).
template <typename R>
__global__ void __launch_bounds__(PACK_THREADS, sizeof(R) == 4 ? 4 : 3) pack_planar_kernel(const void* const* __restrict__ ptrs, PackDesc d,
                                                                   const int64_t* __restrict__ tab,
                                                                   R* __restrict__ out, int64_t src_base) {
  using C2 = typename cplx_t<R>::type;
  __shared__ __align__(16) C2 s[1 << PACK_MAX_T];
  const C2* __restrict__ src = reinterpret_cast<const C2*>(ptrs[d.src]) + src_base;
  const int64_t n_tiles = int64_t(1) << d.tile_bits;
  const int64_t lmask = (int64_t(1) << d.ld) - 1;
  const int T = 1 << d.t_bits;
  int64_t so[PACK_PER_THREAD];
  int sl[PACK_PER_THREAD];
#pragma unroll
  for (int i = 0; i < PACK_PER_THREAD; ++i) {
    const int e = threadIdx.x + i * PACK_THREADS;
    so[i] = e < T ? __ldg(tab + d.e_src + e) : 0;
    sl[i] = e < T ? pack_slot((int)__ldg(tab + d.e_q + e)) : 0;
  }
  const int q0 = threadIdx.x * 8;
  const bool writer = q0 < T;
  const int64_t dq = writer ? (q0 & lmask) + gmap(tab, d.q_hi, q0 >> d.ld) : 0;
  // software pipeline (as pack_f16x2s_kernel): the next tile's loads are in flight while
  // this tile goes through shared memory and out
  C2 v[PACK_PER_THREAD];
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
    // 8 consecutive elements per plane leave as two float4 / four double2 stores; the
    // barrier that frees s for the next tile comes after them
    constexpr int V = 16 / sizeof(R);
    using V4 = typename std::conditional<sizeof(R) == 4, float4, double2>::type;
    if (writer) {
#pragma unroll
      for (int j = 0; j < 8; j += V) {
        V4 re, im;
        R* rp = reinterpret_cast<R*>(&re);
        R* ip = reinterpret_cast<R*>(&im);
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const C2 w = s[pack_slot(q0 + j + u)];
          rp[u] = w.x;
          ip[u] = w.y;
        }
        *reinterpret_cast<V4*>(out + db + j) = re;
        *reinterpret_cast<V4*>(out + db + d.plane + j) = im;
      }
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------- skinny ----
// X [b][2][M][K], Y [b][2][N][K] (planar, K contiguous).  The M N outputs of a batch are
// cut into groups of GM x GN <= 16 (GM = min(M, 4) rows of X, GN = min(N, 16 / GM) rows
// of Y).  CTA (s, b) covers K range [s kc, (s + 1) kc); each of its 8 warps takes one
// group (several warps per group interleave the range) and streams the group's rows
// straight from HBM, lanes on consecutive k (coalesced row segments, no shared memory,
// no barriers), accumulating GM GN complex fp64 sums per lane (complex64: fp32 blocks of
// 8 k per lane folded into the fp64 sums).  Warp sums go to
// partial[b][s * WS + w][o] (WS warps per group), summed in order by
// skinny_reduce_kernel -- deterministic.
constexpr int SK_THREADS = 256, SK_WARPS = SK_THREADS / 32;

__host__ __device__ inline void skinny_groups(int m_bits, int n_bits, int& gm_bits, int& gn_bits, int& ng, int& ws) {
  gm_bits = m_bits < 2 ? m_bits : 2;
  gn_bits = n_bits < 4 - gm_bits ? n_bits : 4 - gm_bits;
  ng = 1 << (m_bits - gm_bits + n_bits - gn_bits);
  ws = ng >= SK_WARPS ? 1 : SK_WARPS / ng;
}

template <typename R, int GM, int GN>
__global__ void __launch_bounds__(SK_THREADS) skinny_kernel(const R* __restrict__ X, const R* __restrict__ Y,
                                                            double2* __restrict__ partial, int32_t m_bits,
                                                            int32_t n_bits, int64_t K, int64_t kc, int32_t S,
                                                            void* const* __restrict__ ptrs, int32_t c_node,
                                                            int32_t accumulate) {
  using C2 = typename cplx_t<R>::type;
  int gm_bits, gn_bits, ng, ws;
  skinny_groups(m_bits, n_bits, gm_bits, gn_bits, ng, ws);
  const int M = 1 << m_bits, N = 1 << n_bits;
  const int b = blockIdx.y, s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k_begin = (int64_t)s * kc, k_end = min(K, k_begin + kc);
  const R* __restrict__ xb = X + (int64_t)b * 2 * M * K;
  const R* __restrict__ yb = Y + (int64_t)b * 2 * N * K;
  for (int g = warp % ng; g < ng; g += SK_WARPS) {
    const int wsub = (ng >= SK_WARPS) ? 0 : warp / ng;
    const int m0 = (g >> (n_bits - gn_bits)) << gm_bits, n0 = (g & ((1 << (n_bits - gn_bits)) - 1)) << gn_bits;
    double ar[GM][GN], ai[GM][GN];
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int j = 0; j < GN; ++j) { ar[i][j] = 0.0; ai[i][j] = 0.0; }
    const R* xr_p = xb + (int64_t)m0 * K;
    const R* xi_p = xb + (int64_t)(M + m0) * K;
    const R* yr_p = yb + (int64_t)n0 * K;
    const R* yi_p = yb + (int64_t)(N + n0) * K;
    if constexpr (sizeof(R) == 4) {
      // complex64: each lane takes 4 consecutive k (16-byte loads, 512-byte warp segments);
      // products accumulate in fp32 over blocks of 8 k per lane, each block then added to
      // the fp64 sums (the FP64 pipe bounded the all-fp64 loop at ~1 TB/s)
      float br[GM][GN], bi[GM][GN];
#pragma unroll
      for (int i = 0; i < GM; ++i)
#pragma unroll
        for (int j = 0; j < GN; ++j) { br[i][j] = 0.f; bi[i][j] = 0.f; }
      int cnt = 0;
      for (int64_t k = k_begin + (int64_t)(wsub * 32 + lane) * 4; k < k_end; k += 128 * ws) {
        float4 xr[GM], xi[GM], yr[GN], yi[GN];
#pragma unroll
        for (int i = 0; i < GM; ++i) {
          xr[i] = __ldg(reinterpret_cast<const float4*>(xr_p + (int64_t)i * K + k));
          xi[i] = __ldg(reinterpret_cast<const float4*>(xi_p + (int64_t)i * K + k));
        }
#pragma unroll
        for (int j = 0; j < GN; ++j) {
          yr[j] = __ldg(reinterpret_cast<const float4*>(yr_p + (int64_t)j * K + k));
          yi[j] = __ldg(reinterpret_cast<const float4*>(yi_p + (int64_t)j * K + k));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int i = 0; i < GM; ++i)
#pragma unroll
            for (int j = 0; j < GN; ++j) {
              const float a_r = (&xr[i].x)[u], a_i = (&xi[i].x)[u], b_r = (&yr[j].x)[u], b_i = (&yi[j].x)[u];
              br[i][j] = fmaf(a_r, b_r, br[i][j]);
              br[i][j] = fmaf(-a_i, b_i, br[i][j]);
              bi[i][j] = fmaf(a_r, b_i, bi[i][j]);
              bi[i][j] = fmaf(a_i, b_r, bi[i][j]);
            }
        if (++cnt == 2) {
          cnt = 0;
#pragma unroll
          for (int i = 0; i < GM; ++i)
#pragma unroll
            for (int j = 0; j < GN; ++j) {
              ar[i][j] += (double)br[i][j]; ai[i][j] += (double)bi[i][j];
              br[i][j] = 0.f; bi[i][j] = 0.f;
            }
        }
      }
#pragma unroll
      for (int i = 0; i < GM; ++i)
#pragma unroll
        for (int j = 0; j < GN; ++j) { ar[i][j] += (double)br[i][j]; ai[i][j] += (double)bi[i][j]; }
    } else {
      for (int64_t k = k_begin + wsub * 32 + lane; k < k_end; k += 32 * ws) {
        double xr[GM], xi[GM], yr[GN], yi[GN];
#pragma unroll
        for (int i = 0; i < GM; ++i) { xr[i] = xr_p[(int64_t)i * K + k]; xi[i] = xi_p[(int64_t)i * K + k]; }
#pragma unroll
        for (int j = 0; j < GN; ++j) { yr[j] = yr_p[(int64_t)j * K + k]; yi[j] = yi_p[(int64_t)j * K + k]; }
#pragma unroll
        for (int i = 0; i < GM; ++i)
#pragma unroll
          for (int j = 0; j < GN; ++j) {
            ar[i][j] = fma(xr[i], yr[j], ar[i][j]);
            ar[i][j] = fma(-xi[i], yi[j], ar[i][j]);
            ai[i][j] = fma(xr[i], yi[j], ai[i][j]);
            ai[i][j] = fma(xi[i], yr[j], ai[i][j]);
          }
      }
    }
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int j = 0; j < GN; ++j) {
        double re = ar[i][j], im = ai[i][j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          re += __shfl_xor_sync(0xffffffffu, re, off);
          im += __shfl_xor_sync(0xffffffffu, im, off);
        }
        if (lane == 0) {
          if (S * ws == 1) {        // one partial per output: write C directly
            C2* C = reinterpret_cast<C2*>(ptrs[c_node]) + (int64_t)b * M * N + (m0 + i) * N + n0 + j;
            if (accumulate) { re += C->x; im += C->y; }
            *C = C2{(R)re, (R)im};
          } else {
            partial[(((int64_t)b * S + s) * ws + wsub) * (M * N) + (m0 + i) * N + n0 + j] = make_double2(re, im);
          }
        }
      }
  }
}

// --------------------------------------------------------------- skinny v2 ----
// The same contraction with the operand rows staged through shared memory by TMA: a
// persistent CTA walks work items (batch, K range[, half of X's rows]); one producer lane
// loads every stage -- the item's X rows (re and im planes) and Y rows x KS elements of K
// -- as two 3-D tensor boxes {KS, rows, 2 planes} into a ring of STAGES buffers (mbarrier
// full / empty), so each byte of X and Y is read from HBM once and enough bytes are in
// flight to cover the latency (v1 read every X row from 2 warps and every Y row from 4,
// straight from global, at 12% warp occupancy: 0.44-0.59 of HBM; per-row bulk copies of
// 512 bytes were issue-bound at ~1 copy per 80 cycles per SM).  Sixteen consumer warps
// (8 warps with 4 x 4 groups were issue / latency bound at 0.6 of HBM): each output group
// (GM x GN <= 4 x 2, at most 16 groups per item) has WPG = 16 / groups warps, which take
// its stages in turn; lanes take 16-byte vectors of consecutive k (conflict-free
// LDS.128).  Complex64 products accumulate in fp32 over a stage (KS / 32 terms per lane,
// <= 8) and fold into fp64 (the fp32-path bound with K = 8 holds: DESIGN.md
// "Tolerances"); complex128 in fp64.  Per item the warp sums go to partial[b][s][wsub][o] (then the in-order
// skinny_reduce_kernel: deterministic) or, with one item per batch and one warp per group,
// straight to C.
constexpr int SK2_WARPS = 16, SK2_THREADS = 32 * SK2_WARPS;

// producer cursor over this CTA's stages (items blockIdx.x, + gridDim.x, ...; stages of KS)
struct Sk2Cursor {
  int64_t it, k, k1;
  int b, h;
};
__device__ __forceinline__ bool sk2_item(Sk2Cursor& c, int64_t n_items, int m_split, int S, int64_t kc, int64_t K) {
  if (c.it >= n_items) return false;
  c.h = (int)(c.it % m_split);
  const int64_t bs = c.it / m_split;
  c.b = (int)(bs / S);
  c.k = (bs % S) * kc;
  c.k1 = min(K, c.k + kc);
  return true;
}

template <typename R, int GM, int GN>
__global__ void __launch_bounds__(SK2_THREADS, 1) skinny2_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                const __grid_constant__ CUtensorMap tmY,
                                                                double2* __restrict__ partial, int32_t m_bits,
                                                                int32_t n_bits, int64_t K, int64_t kc, int32_t S,
                                                                int32_t nb, int32_t m_split, int32_t ks,
                                                                int32_t stages, void* const* __restrict__ ptrs,
                                                                int32_t c_node, int32_t accumulate) {
  using C2 = typename cplx_t<R>::type;
  constexpr int VEC = 16 / sizeof(R);
  extern __shared__ __align__(128) uint8_t sk_smem[];
  const int M = 1 << m_bits, N = 1 << n_bits;
  const int Mh = M / m_split;
  const int rows = 2 * (Mh + N);
  const int64_t stage_elems = (int64_t)rows * ks;
  R* st_base = reinterpret_cast<R*>(sk_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(sk_smem + (size_t)stages * stage_elems * sizeof(R));
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ngn = N / GN, n_groups = (Mh / GM) * ngn;
  const int wpg = SK2_WARPS / n_groups;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], n_groups); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmY)) : "memory");
  }
  __syncthreads();
  const int64_t n_items = (int64_t)nb * S * m_split;
  // The producer is lane 0 of warp 0: before consuming stage g it tops the ring up to stage
  // g + stages - 1 (whose slot frees when every group's warp has finished stage g - 1).
  const bool producer = threadIdx.x == 0;
  const uint32_t stage_bytes = (uint32_t)(stage_elems * sizeof(R));
  Sk2Cursor pc{(int64_t)blockIdx.x, 0, 0, 0, 0};
  bool p_more = producer && sk2_item(pc, n_items, m_split, S, kc, K);
  int64_t g_p = 0;                               // next stage the producer loads
  int p_slot = 0;
  uint32_t p_phase = 0;
  auto top_up = [&](int64_t g_limit) {
    while (p_more && g_p < g_limit) {
      tc::mbar_wait(&empty[p_slot], p_phase ^ 1);
      tc::mbar_expect_tx(&full[p_slot], stage_bytes);
      R* d = st_base + p_slot * stage_elems;
      tc::tma_load_3d(&tmX, d, &full[p_slot], (int)pc.k, pc.h * Mh, 2 * pc.b);                    // [2][Mh][ks]
      tc::tma_load_3d(&tmY, d + (int64_t)2 * Mh * ks, &full[p_slot], (int)pc.k, 0, 2 * pc.b);      // [2][N][ks]
      ++g_p;
      if (++p_slot == stages) { p_slot = 0; p_phase ^= 1; }
      pc.k += ks;
      if (pc.k >= pc.k1) {
        pc.it += gridDim.x;
        p_more = sk2_item(pc, n_items, m_split, S, kc, K);
      }
    }
  };
  // consumers: warp -> (group grp, sub-warp wsub of the WPG warps taking its stages in turn)
  const int grp = warp % n_groups, wsub = warp / n_groups;
  const int gm0 = (grp / ngn) * GM, gn0 = (grp % ngn) * GN;
  const int iters = ks / (32 * VEC);
  int64_t g = 0;
  int slot = 0;
  uint32_t phase = 0;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int h = (int)(it % m_split);
    const int64_t bs = it / m_split;
    const int b = (int)(bs / S), s = (int)(bs % S);
    const int64_t k0 = (int64_t)s * kc, k1 = min(K, k0 + kc);
    double ar[GM][GN], ai[GM][GN];
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int j = 0; j < GN; ++j) { ar[i][j] = 0.0; ai[i][j] = 0.0; }
    int turn = 0;                                  // stage of this item modulo WPG
    float br[GM][GN], bi[GM][GN];                  // complex64: fp32 sums since the last fold
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int j = 0; j < GN; ++j) { br[i][j] = 0.f; bi[i][j] = 0.f; }
    int unfolded = 0;                              // stages summed into br / bi
    for (int64_t k = k0; k < k1; k += ks, ++g) {
      if (producer) top_up(g + stages);
      const int cur = slot;
      const uint32_t cph = phase;
      if (++slot == stages) { slot = 0; phase ^= 1; }
      const bool mine = turn == wsub;
      if (++turn == wpg) turn = 0;
      // every warp waits for every stage in order, owner or not: a warp that skipped ahead
      // could otherwise wait on a slot whose previous phase is still pending -- a parity
      // wait cannot tell the two phases apart, it would read the slot early and arrive on
      // the wrong phase of `empty` (a hang on K = 2^20 scalar steps)
      tc::mbar_wait(&full[cur], cph);
      if (!mine) continue;
      const R* st = st_base + cur * stage_elems;
      for (int itr = 0; itr < iters; ++itr) {
        const int kk = (itr * 32 + lane) * VEC;
        if constexpr (sizeof(R) == 4) {
          // all the iteration's loads first (16 warps x 128 registers hold them), then the FMAs
          float4 yr[GN], yi[GN], xr4[GM], xi4[GM];
#pragma unroll
          for (int j = 0; j < GN; ++j) {
            yr[j] = *reinterpret_cast<const float4*>(st + (int64_t)(2 * Mh + gn0 + j) * ks + kk);
            yi[j] = *reinterpret_cast<const float4*>(st + (int64_t)(2 * Mh + N + gn0 + j) * ks + kk);
          }
#pragma unroll
          for (int i = 0; i < GM; ++i) {
            xr4[i] = *reinterpret_cast<const float4*>(st + (int64_t)(gm0 + i) * ks + kk);
            xi4[i] = *reinterpret_cast<const float4*>(st + (int64_t)(Mh + gm0 + i) * ks + kk);
          }
#pragma unroll
          for (int i = 0; i < GM; ++i) {
            const float4 xr = xr4[i], xi = xi4[i];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int j = 0; j < GN; ++j) {
                const float a_r = (&xr.x)[u], a_i = (&xi.x)[u], b_r = (&yr[j].x)[u], b_i = (&yi[j].x)[u];
                br[i][j] = fmaf(a_r, b_r, br[i][j]);
                br[i][j] = fmaf(-a_i, b_i, br[i][j]);
                bi[i][j] = fmaf(a_r, b_i, bi[i][j]);
                bi[i][j] = fmaf(a_i, b_r, bi[i][j]);
              }
          }
        } else {
          double2 yr[GN], yi[GN];
#pragma unroll
          for (int j = 0; j < GN; ++j) {
            yr[j] = *reinterpret_cast<const double2*>(st + (int64_t)(2 * Mh + gn0 + j) * ks + kk);
            yi[j] = *reinterpret_cast<const double2*>(st + (int64_t)(2 * Mh + N + gn0 + j) * ks + kk);
          }
#pragma unroll
          for (int i = 0; i < GM; ++i) {
            const double2 xr = *reinterpret_cast<const double2*>(st + (int64_t)(gm0 + i) * ks + kk);
            const double2 xi = *reinterpret_cast<const double2*>(st + (int64_t)(Mh + gm0 + i) * ks + kk);
#pragma unroll
            for (int j = 0; j < GN; ++j)
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const double a_r = (&xr.x)[u], a_i = (&xi.x)[u], b_r = (&yr[j].x)[u], b_i = (&yi[j].x)[u];
                ar[i][j] = fma(a_r, b_r, ar[i][j]);
                ar[i][j] = fma(-a_i, b_i, ar[i][j]);
                ai[i][j] = fma(a_r, b_i, ai[i][j]);
                ai[i][j] = fma(a_i, b_r, ai[i][j]);
              }
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[cur]);
      if constexpr (sizeof(R) == 4) {
        // fold the stage's fp32 sums (iters x 4 terms per lane: 8 for KS = 256) into fp64
        // (folding every 2 stages measured no faster)
        if (++unfolded == 1) {
          unfolded = 0;
#pragma unroll
          for (int i = 0; i < GM; ++i)
#pragma unroll
            for (int j = 0; j < GN; ++j) {
              ar[i][j] += (double)br[i][j]; ai[i][j] += (double)bi[i][j];
              br[i][j] = 0.f; bi[i][j] = 0.f;
            }
        }
      }
    }
    if constexpr (sizeof(R) == 4) {
#pragma unroll
      for (int i = 0; i < GM; ++i)
#pragma unroll
        for (int j = 0; j < GN; ++j) { ar[i][j] += (double)br[i][j]; ai[i][j] += (double)bi[i][j]; }
    }
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int j = 0; j < GN; ++j) {
        double re = ar[i][j], im = ai[i][j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          re += __shfl_xor_sync(0xffffffffu, re, off);
          im += __shfl_xor_sync(0xffffffffu, im, off);
        }
        if (lane == 0) {
          const int o = (h * Mh + gm0 + i) * N + gn0 + j;
          if (S * wpg == 1) {          // one partial per output: write C directly
            C2* C = reinterpret_cast<C2*>(ptrs[c_node]) + (int64_t)b * M * N + o;
            if (accumulate) { re += C->x; im += C->y; }
            *C = C2{(R)re, (R)im};
          } else {
            partial[(((int64_t)b * S + s) * wpg + wsub) * (M * N) + o] = make_double2(re, im);
          }
        }
      }
  }
}

// C[b][o] (+)= sum_s partial[b][s][o]: one warp per output, lane l sums s = l, l + 32, ...
// in order, then a fixed shuffle tree -- deterministic, and parallel when a long
// contraction has few outputs (a scalar: S x 8 partials)
template <typename R>
__global__ void skinny_reduce_kernel(const double2* __restrict__ partial, int32_t S, int32_t O, int64_t n_out,
                                     void* const* __restrict__ ptrs, int32_t c_node, int32_t accumulate) {
  using C2 = typename cplx_t<R>::type;
  C2* C = reinterpret_cast<C2*>(ptrs[c_node]);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_out; i += warps) {
    const int64_t b = i / O, o = i % O;
    double re = 0.0, im = 0.0;
    for (int s = lane; s < S; s += 32) {
      const double2 v = partial[(b * S + s) * O + o];
      re += v.x;
      im += v.y;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, off);
      im += __shfl_xor_sync(0xffffffffu, im, off);
    }
    if (lane == 0) {
      if (accumulate) { re += C[i].x; im += C[i].y; }
      C[i] = C2{(R)re, (R)im};
    }
  }
}

// packed fp32 pair FMA (FFMA2: two fp32 lanes per instruction, half the issue slots of FFMA)
__device__ __forceinline__ void fma2_(uint64_t& d, uint64_t a, uint64_t b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

// ------------------------------------------------------------------- wide ----
// C[b][m][n] = sum_k X[b][m][k] Y[b][n][k] with K <= WD_MAXK (16): a short contraction
// onto a large output, bound by writing C.  A CTA covers rows [m0, m0 + tm) (tm <=
// WD_TM) x columns [n0, n0 + 256): the X rows go to shared memory (fp64, read as
// broadcasts), each thread keeps its column's Y row in registers (K contiguous in the
// planar operand: vector loads) and writes its column of the tile, consecutive threads on
// consecutive n (coalesced).  Tiles are visited grid-stride with the row tile fastest so
// CTAs running together share Y columns in L2.  Accumulation in the plan's type: fp32 FMA
// for complex64 (K <= 16 terms: the fp32-path bound of DESIGN.md "Tolerances"; fp64 here
// ran at the FP64 pipe's ~12 TFLOP/s, 4x slower than writing C), fp64 for complex128.
// KMAX = K (a template argument): the Y row lives in K-sized register arrays, so short-K
// steps keep the occupancy (the 16-wide arrays held 128 registers at any K).
#ifndef TN_WD_TM_C128
#define TN_WD_TM_C128 64
#endif
constexpr int WD_THREADS = 256, WD_TM = 32, WD_MAXK = 16;
// rows per tile: 32 for complex64, 64 for complex128 (fewer tiles per batch: configs[3]'s
// (11, 7, 7, 2) step re-read Y once per 32-row tile)
template <typename R>
__host__ __device__ constexpr int wd_tm() { return sizeof(R) == 8 ? TN_WD_TM_C128 : WD_TM; }

// GATHER: X and Y are the raw operands (interleaved complex, any stored index order), read
// through the step's offset tables `gm` (no planar pack pass; the tables' K offsets go to
// shared memory once per CTA); else X / Y are the planar packed operands.
// F2 (complex64, CPT = 2, gathered): packed fp32 pair FMAs (FFMA2), 4 per k and row
// instead of 8 FFMA.
template <typename R, int CPT, int KMAX, bool GATHER, bool F2 = false>
__global__ void __launch_bounds__(WD_THREADS) wide_kernel(const R* __restrict__ X, const R* __restrict__ Y,
                                                          void* const* __restrict__ ptrs, int32_t c_node,
                                                          int32_t m_bits, int32_t n_bits, int32_t k_bits,
                                                          int64_t n_tiles, const GatherMaps gm,
                                                          const int64_t* __restrict__ tab) {
  // CPT adjacent columns per thread (2 for complex64: each broadcast X load serves two
  // outputs and each thread stores 16 bytes)
  using C2 = typename cplx_t<R>::type;
  __shared__ __align__(16) R xs[2][wd_tm<R>()][WD_MAXK];  // (rows of KMAX <= WD_MAXK)
  __shared__ int64_t kofs[2][KMAX];                  // GATHER: K offsets of X and Y
  C2* __restrict__ C = reinterpret_cast<C2*>(ptrs[c_node]);
  const int64_t M = int64_t(1) << m_bits, N = int64_t(1) << n_bits;
  const int K = 1 << k_bits;
  const C2* __restrict__ Xc = GATHER ? reinterpret_cast<const C2*>(ptrs[gm.a_node]) : nullptr;
  const C2* __restrict__ Yc = GATHER ? reinterpret_cast<const C2*>(ptrs[gm.b_node]) : nullptr;
  if constexpr (GATHER) {
    if (threadIdx.x < K) {
      kofs[0][threadIdx.x] = gmap(tab, gm.Ak, threadIdx.x);
      kofs[1][threadIdx.x] = gmap(tab, gm.Bk, threadIdx.x);
    }
  }
  const int tm = (int)(M < wd_tm<R>() ? M : wd_tm<R>());
  constexpr int TN = WD_THREADS * CPT;
  const int64_t mt = M / tm, ncb = (N + TN - 1) / TN;
  // N < TN: the threads split into row groups, each covering all N columns
  const int tpr = (int)((N < TN ? N : TN) / CPT);   // threads per row group
  const int groups = WD_THREADS / tpr, rg = threadIdx.x / tpr;
  constexpr int V = 16 / sizeof(R);                  // elements per 16-byte vector load
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t b = tile / (ncb * mt), r = tile % (ncb * mt);
    const int64_t m0 = (r % mt) * tm, n = (r / mt) * TN + (threadIdx.x % tpr) * CPT;
    const R* __restrict__ xb = X + b * 2 * M * K;
    const R* __restrict__ yb = Y + b * 2 * N * K;
    __syncthreads();                                 // the previous tile's xs reads are done
    if constexpr (GATHER) {
      const int64_t xbo = gmap(tab, gm.Ab, b);
      for (int e = threadIdx.x; e < tm * K; e += WD_THREADS) {
        const int i = e / K, k = e % K;
        const C2 v = Xc[xbo + gmap(tab, gm.Am, m0 + i) + kofs[0][k]];
        xs[0][i][k] = v.x;
        xs[1][i][k] = v.y;
      }
    } else {
      for (int e = threadIdx.x; e < 2 * tm * K; e += WD_THREADS) {
        const int p = e / (tm * K), i = (e / K) % tm, k = e % K;
        xs[p][i][k] = xb[(p * M + m0 + i) * K + k];
      }
    }
    __syncthreads();
    if (n >= N || rg >= groups) continue;
    if constexpr (F2) {
      // gathered Y entries are (re, im) register pairs: per column c, P += x_r (y_re, y_im)
      // and Q += x_i (y_re, y_im) (broadcast X element), re = P.lo - Q.hi, im = P.hi + Q.lo
      static_assert(sizeof(R) == 4 && CPT == 2 && GATHER, "FFMA2 wide: complex64, two columns, gathered");
      uint64_t yp[CPT][KMAX];
      const int64_t yb0 = gmap(tab, gm.Bb, b);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int64_t yo = yb0 + gmap(tab, gm.Bn, n + c);
#pragma unroll
        for (int k = 0; k < KMAX; ++k) yp[c][k] = *reinterpret_cast<const unsigned long long*>(Yc + yo + kofs[1][k]);
      }
      C2* __restrict__ cp = C + (b * M + m0) * N + n;
      for (int i = rg; i < tm; i += groups) {
        uint64_t P[CPT] = {0, 0}, Q[CPT] = {0, 0};
#pragma unroll
        for (int q = 0; q < KMAX / 4; ++q) {
          const float4 xr = *reinterpret_cast<const float4*>(&xs[0][i][q * 4]);
          const float4 xi = *reinterpret_cast<const float4*>(&xs[1][i][q * 4]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint64_t a_r, a_i;
            asm("mov.b64 %0, {%1,%1};" : "=l"(a_r) : "f"((&xr.x)[u]));
            asm("mov.b64 %0, {%1,%1};" : "=l"(a_i) : "f"((&xi.x)[u]));
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
              fma2_(P[c], a_r, yp[c][q * 4 + u]);
              fma2_(Q[c], a_i, yp[c][q * 4 + u]);
            }
          }
        }
        float p0r, p0i, q0r, q0i, p1r, p1i, q1r, q1i;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(p0r), "=f"(p0i) : "l"(P[0]));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(q0r), "=f"(q0i) : "l"(Q[0]));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(p1r), "=f"(p1i) : "l"(P[1]));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(q1r), "=f"(q1i) : "l"(Q[1]));
        *reinterpret_cast<float4*>(cp + (int64_t)i * N) = make_float4(p0r - q0i, p0i + q0r, p1r - q1i, p1i + q1r);
      }
    } else {
      R yr[CPT][KMAX], yi[CPT][KMAX];
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if constexpr (GATHER) {
          const int64_t yo = gmap(tab, gm.Bb, b) + gmap(tab, gm.Bn, n + c);
#pragma unroll
          for (int k = 0; k < KMAX; ++k) {
            const C2 v = Yc[yo + kofs[1][k]];
            yr[c][k] = v.x;
            yi[c][k] = v.y;
          }
        } else if (K % V == 0) {
#pragma unroll
          for (int q = 0; q < KMAX / V; ++q) {
            if (q * V < K) {
              R vr[V], vi[V];
              *reinterpret_cast<float4*>(vr) = __ldg(reinterpret_cast<const float4*>(yb + (n + c) * K) + q);
              *reinterpret_cast<float4*>(vi) = __ldg(reinterpret_cast<const float4*>(yb + (N + n + c) * K) + q);
#pragma unroll
              for (int u = 0; u < V; ++u) { yr[c][q * V + u] = vr[u]; yi[c][q * V + u] = vi[u]; }
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < KMAX; ++k)
            if (k < K) { yr[c][k] = __ldg(yb + (n + c) * K + k); yi[c][k] = __ldg(yb + (N + n + c) * K + k); }
        }
      }
      C2* __restrict__ cp = C + (b * M + m0) * N + n;
      for (int i = rg; i < tm; i += groups) {
        R re[CPT], im[CPT];
#pragma unroll
        for (int c = 0; c < CPT; ++c) { re[c] = 0; im[c] = 0; }
        if (K % V == 0) {       // the row of X as 16-byte broadcast loads (the LDS count bounded this loop)
#pragma unroll
          for (int q = 0; q < KMAX / V; ++q) {
            if (q * V < K) {
              R xr[V], xi[V];
              *reinterpret_cast<float4*>(xr) = *reinterpret_cast<const float4*>(&xs[0][i][q * V]);
              *reinterpret_cast<float4*>(xi) = *reinterpret_cast<const float4*>(&xs[1][i][q * V]);
#pragma unroll
              for (int u = 0; u < V; ++u)
#pragma unroll
                for (int c = 0; c < CPT; ++c) {
                  re[c] = fma(xr[u], yr[c][q * V + u], re[c]);
                  re[c] = fma(-xi[u], yi[c][q * V + u], re[c]);
                  im[c] = fma(xr[u], yi[c][q * V + u], im[c]);
                  im[c] = fma(xi[u], yr[c][q * V + u], im[c]);
                }
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < KMAX; ++k) {
            if (k < K) {
              const R ar = xs[0][i][k], ai = xs[1][i][k];
#pragma unroll
              for (int c = 0; c < CPT; ++c) {
                re[c] = fma(ar, yr[c][k], re[c]);
                re[c] = fma(-ai, yi[c][k], re[c]);
                im[c] = fma(ar, yi[c][k], im[c]);
                im[c] = fma(ai, yr[c][k], im[c]);
              }
            }
          }
        }
        if constexpr (CPT == 2) {
          static_assert(sizeof(R) == 4, "two columns per thread: complex64 only");
          *reinterpret_cast<float4*>(cp + (int64_t)i * N) = make_float4(re[0], im[0], re[1], im[1]);
        } else {
          cp[(int64_t)i * N] = C2{re[0], im[0]};
        }
      }
    }
  }
}

// C[b][o] (+)= sum_s partial[b][s][o] for few outputs (n_out <= 4 x 148): one CTA per
// output, thread t sums s = t, t + 256, ... in order, then a fixed tree over the CTA
// (deterministic) -- the warp-per-output kernel above leaves a scalar's S partials to one
// warp (configs[3]'s K = 2^20 dot product: 29 us)
template <typename R>
__global__ void __launch_bounds__(256) skinny_reduce_cta_kernel(const double2* __restrict__ partial, int32_t S,
                                                                int32_t O, int64_t n_out, void* const* __restrict__ ptrs,
                                                                int32_t c_node, int32_t accumulate) {
  using C2 = typename cplx_t<R>::type;
  __shared__ double2 red[256];
  C2* C = reinterpret_cast<C2*>(ptrs[c_node]);
  for (int64_t i = blockIdx.x; i < n_out; i += gridDim.x) {
    const int64_t b = i / O, o = i % O;
    double re = 0.0, im = 0.0;
    for (int s = threadIdx.x; s < S; s += 256) {
      const double2 v = partial[(b * S + s) * O + o];
      re += v.x;
      im += v.y;
    }
    red[threadIdx.x] = double2{re, im};
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
      if (threadIdx.x < h) {
        red[threadIdx.x].x += red[threadIdx.x + h].x;
        red[threadIdx.x].y += red[threadIdx.x + h].y;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      double r = red[0].x, m = red[0].y;
      if (accumulate) { r += C[i].x; m += C[i].y; }
      C[i] = C2{(R)r, (R)m};
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- batched skinny, gathered ----
// Skinny steps without K-slabs (Eq. (3): C[b][m][n] =
// sum_k X[b][m][k] Y[b][n][k], M N <= 256): one CTA per batch (grid-stride) stages chunks of
// KC of K of X[b] and Y[b] in shared memory, gathering the raw interleaved operands
// through the step's offset tables (GatherMaps: no planar pack pass, no K split, no
// reduction launch), k-major ([k][row]) so the output threads read conflict-free.  The 256
// threads are M N outputs x G = 256 / (M N) lanes of K (lane j takes k = j, j + G, ...); the
// lanes' fp64 sums are added in lane order (deterministic).  Products and sums in fp64
// for both dtypes.
constexpr int BS_THREADS = 256;
template <typename C2>
__device__ __forceinline__ void bs_cp_async(C2* smem, const C2* gmem) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(C2) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem) : "memory");
}
template <typename R>
__global__ void __launch_bounds__(BS_THREADS) bskinny_kernel(const GatherMaps gm, const int64_t* __restrict__ tab,
                                                              void* const* __restrict__ ptrs, int32_t c_node,
                                                              int32_t m_bits, int32_t n_bits, int32_t k_bits,
                                                              int32_t kc_bits, int64_t n_batches, int32_t s_bits,
                                                              double2* __restrict__ partial) {
  using C2 = typename cplx_t<R>::type;
  extern __shared__ __align__(16) unsigned char bs_smem[];
  const int M = 1 << m_bits, N = 1 << n_bits, KC = 1 << kc_bits;
  const int64_t K = int64_t(1) << k_bits;
  const int MP = M + 1, NP = N + 1;                           // padded rows: conflict-free staging
  C2* xs = reinterpret_cast<C2*>(bs_smem);                    // [KC][M + 1]
  C2* ys = xs + KC * MP;                                      // [KC][N + 1]
  int64_t* rowX = reinterpret_cast<int64_t*>(ys + KC * NP);   // [M]
  int64_t* rowY = rowX + M;                                   // [N]
  int64_t* kX = rowY + N;                                     // [KC]
  int64_t* kY = kX + KC;                                      // [KC]
  double2* red = reinterpret_cast<double2*>(kY + KC);         // [BS_THREADS]
  const C2* __restrict__ A = reinterpret_cast<const C2*>(ptrs[gm.a_node]);
  const C2* __restrict__ B = reinterpret_cast<const C2*>(ptrs[gm.b_node]);
  C2* __restrict__ C = reinterpret_cast<C2*>(ptrs[c_node]);
  const int O = M * N, G = BS_THREADS / O;                    // O <= 256: G >= 1
  const int o = threadIdx.x / G, j = threadIdx.x % G;
  const int om = o / N, on = o % N;
  // items (batch, K range): 2^s_bits contiguous K ranges per batch (few batches, long K);
  // with more than one range the CTA writes partial[b][range][o] (summed in order by
  // skinny_reduce_*_kernel) instead of C
  const int64_t KR = K >> s_bits;
  // per CTA: the row offsets inside a batch and -- when one chunk is a whole K range of
  // every item -- the K offsets; per item only the two batch offsets are looked up
  for (int r = threadIdx.x; r < M + N; r += BS_THREADS) {
    if (r < M) rowX[r] = gmap(tab, gm.Am, r);
    else rowY[r - M] = gmap(tab, gm.Bn, r - M);
  }
  const bool kfixed = s_bits == 0 && KC == K;
  if (kfixed)
    for (int k = threadIdx.x; k < KC; k += BS_THREADS) {
      kX[k] = gmap(tab, gm.Ak, k);
      kY[k] = gmap(tab, gm.Bk, k);
    }
  for (int64_t item = blockIdx.x; item < (n_batches << s_bits); item += gridDim.x) {
    const int64_t b = item >> s_bits, kr = item & ((int64_t(1) << s_bits) - 1);
    const int64_t xb = gmap(tab, gm.Ab, b), yb = gmap(tab, gm.Bb, b);
    double re = 0.0, im = 0.0;
    for (int64_t k0 = kr * KR; k0 < (kr + 1) * KR; k0 += KC) {
      __syncthreads();                      // offsets ready; the previous chunk / item consumed
      if (!kfixed) {
        for (int k = threadIdx.x; k < KC; k += BS_THREADS) {
          kX[k] = gmap(tab, gm.Ak, k0 + k);
          kY[k] = gmap(tab, gm.Bk, k0 + k);
        }
        __syncthreads();
      }
      // gather along the operand's stride-1 direction (K or rows) so a warp's loads
      // coalesce; cp.async straight to shared memory (every element's load in flight at once)
      for (int e = threadIdx.x; e < M * KC; e += BS_THREADS) {
        const int r = gm.a_kfast ? e >> kc_bits : e & (M - 1);
        const int k = gm.a_kfast ? e & (KC - 1) : e >> m_bits;
        bs_cp_async(&xs[k * MP + r], &A[xb + rowX[r] + kX[k]]);
      }
      for (int e = threadIdx.x; e < N * KC; e += BS_THREADS) {
        const int r = gm.b_kfast ? e >> kc_bits : e & (N - 1);
        const int k = gm.b_kfast ? e & (KC - 1) : e >> n_bits;
        bs_cp_async(&ys[k * NP + r], &B[yb + rowY[r] + kY[k]]);
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      // four independent accumulator pairs (k = j + G (4 i + u)) hide the FMA latency
      // (all 8 shared loads of a group issued before its FMAs: the loop was bound by the
      // shared-load latency, ncu stall_short_sb)
      double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
      int k = j;
      for (; k + 3 * G < KC; k += 4 * G) {
        C2 x[4], y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[u] = xs[(k + u * G) * MP + om];
          y[u] = ys[(k + u * G) * NP + on];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double xr = x[u].x, xi = x[u].y, yr = y[u].x, yi = y[u].y;
          ar[u] = fma(xr, yr, fma(-xi, yi, ar[u]));
          ai[u] = fma(xr, yi, fma(xi, yr, ai[u]));
        }
      }
      for (; k < KC; k += G) {
        const C2 x = xs[k * MP + om], y = ys[k * NP + on];
        const double xr = x.x, xi = x.y, yr = y.x, yi = y.y;
        ar[0] = fma(xr, yr, fma(-xi, yi, ar[0]));
        ai[0] = fma(xr, yi, fma(xi, yr, ai[0]));
      }
      re += (ar[0] + ar[1]) + (ar[2] + ar[3]);
      im += (ai[0] + ai[1]) + (ai[2] + ai[3]);
    }
    red[threadIdx.x] = double2{re, im};
    __syncthreads();
    if (threadIdx.x < O) {
      double sr = 0.0, si = 0.0;
      for (int q = 0; q < G; ++q) {
        sr += red[threadIdx.x * G + q].x;
        si += red[threadIdx.x * G + q].y;
      }
      const int mm = threadIdx.x / N, nn = threadIdx.x % N;
      if (s_bits > 0) partial[(item << (m_bits + n_bits)) + threadIdx.x] = double2{sr, si};
      else C[(b * M + mm) * (int64_t)N + nn] = C2{(R)sr, (R)si};
    }
  }
}
__host__ __device__ constexpr int bskinny_smem(int m_bits, int n_bits, int kc_bits, int esz) {
  return (((1 << m_bits) + (1 << n_bits) + 2) << kc_bits) * esz + ((1 << m_bits) + (1 << n_bits)) * 8 +
         2 * (1 << kc_bits) * 8 + BS_THREADS * 16;
}

}  // namespace tnd
