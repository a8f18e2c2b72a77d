// Small-tensor path: many independent early-stage pairwise contractions (bond
// dimensions 2-16, a few to a few thousand entries) batched into ONE launch per
// wave of the contraction tree.  HBM/latency bound, so it runs on the CUDA cores:
// each thread owns output elements, the permutation to matricised form is folded
// into the loads through the GroupMap offset tables (no transpose pass).
// PAPER.md Fig. 1b (l.54): C = sum over shared indices of A * B.
#include "common.cuh"

namespace tnd {

// Accumulation is in fp64 for both complex64 and complex128 (the small path is
// latency/HBM bound, so the wider FMA is free; it removes the K-length fp32
// random-walk error of long reductions).  Long reductions with few outputs split K
// over a warp (g_log2 = 5) or the whole CTA (g_log2 = 7), reduced by shuffles and
// shared memory in fp64.
template <typename R>
__global__ void __launch_bounds__(128) small_contract_kernel(
    const SmallStep* __restrict__ steps, const int64_t* __restrict__ cta_prefix, int32_t n_steps,
    const int64_t* __restrict__ tab, void* const* __restrict__ ptrs, const int32_t* __restrict__ cta_step) {
  using C2 = typename cplx_t<R>::type;
  __shared__ double red[2][4];
  // step of this CTA: last s with cta_prefix[s] <= blockIdx.x -- one load from the wave's
  // CTA -> step table (a binary search is ~log2(steps) dependent L2 round trips: 4 us of a
  // 15 us wave of 412 steps), or the search without a table
  int lo = 0;
  if (cta_step) {
    lo = __ldg(cta_step + blockIdx.x);
  } else {
    int hi = n_steps - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(cta_prefix + mid) <= (int64_t)blockIdx.x) lo = mid; else hi = mid - 1;
    }
  }
  const SmallStep& d = steps[lo];
  const C2* __restrict__ A = reinterpret_cast<const C2*>(ptrs[d.a]);
  const C2* __restrict__ B = reinterpret_cast<const C2*>(ptrs[d.b]);
  C2* __restrict__ C = reinterpret_cast<C2*>(ptrs[d.c]);
  const int64_t start = ((int64_t)blockIdx.x - cta_prefix[lo]) * d.opc;
  const int64_t total = int64_t(1) << (d.nb_bits + d.m_bits + d.n_bits);
  const int64_t end = min(total, start + d.opc);
  const int64_t K = int64_t(1) << d.k_bits;
  const int64_t nmask = (int64_t(1) << d.n_bits) - 1, mmask = (int64_t(1) << d.m_bits) - 1;
  const int G = 1 << d.g_log2;
  const int gl = threadIdx.x & (G - 1);
  const int per = blockDim.x >> d.g_log2;       // outputs in flight per CTA
  for (int64_t o0 = start; o0 < end; o0 += per) {
    const int64_t o = o0 + (threadIdx.x >> d.g_log2);
    double re = 0.0, im = 0.0;
    if (o < end) {
      const int64_t n = o & nmask;
      const int64_t m = (o >> d.n_bits) & mmask;
      const int64_t bb = o >> (d.n_bits + d.m_bits);
      const int64_t ao = gmap(tab, d.Ab, bb) + gmap(tab, d.Am, m);
      const int64_t bo = gmap(tab, d.Bb, bb) + gmap(tab, d.Bn, n);
      for (int64_t k = gl; k < K; k += G) {
        const C2 a = A[ao + gmap(tab, d.Ak, k)];
        const C2 b = B[bo + gmap(tab, d.Bk, k)];
        re = fma((double)a.x, (double)b.x, re);
        re = fma(-(double)a.y, (double)b.y, re);
        im = fma((double)a.x, (double)b.y, im);
        im = fma((double)a.y, (double)b.x, im);
      }
    }
    if (G >= 32) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
      }
    }
    if (G == 128) {
      if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = re; red[1][threadIdx.x >> 5] = im; }
      __syncthreads();
      re = (red[0][0] + red[0][1]) + (red[0][2] + red[0][3]);
      im = (red[1][0] + red[1][1]) + (red[1][2] + red[1][3]);
      __syncthreads();
    }
    if (o < end && gl == 0) C[o] = C2{(R)re, (R)im};
  }
}

// Leaf pointers of one (bitstring, slice) pass: a leaf whose output legs / sliced
// indices are bound to values v_j lives at base + sum_j v_j * stride_j.
// var_kind >= 0: qubit id (value = bits[q]); var_kind < 0: sliced index number
// (-1 - j), value = digit j of the slice id (last sliced index fastest).
__global__ void set_leaf_ptrs_kernel(void** __restrict__ ptrs, const int64_t* __restrict__ leaf_base,
                                     const int32_t* __restrict__ var_begin, const int32_t* __restrict__ var_kind,
                                     const int64_t* __restrict__ var_stride, int32_t n_leaves,
                                     const uint8_t* __restrict__ bits, const int64_t* __restrict__ slice_id,
                                     const int32_t* __restrict__ slice_dim_log2, const int32_t* __restrict__ slice_shift,
                                     int32_t elem_bytes, char* arena_leaves) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_leaves) return;
  int64_t off = leaf_base[t];
  const int64_t s = *slice_id;
  for (int v = var_begin[t]; v < var_begin[t + 1]; ++v) {
    int k = var_kind[v];
    int64_t val;
    if (k >= 0) val = bits[k];
    else {
      int j = -1 - k;
      // slice ids are int64: sliced bits at positions >= 63 are 0 (tn.h, tn_plan_info)
      val = slice_shift[j] >= 63 ? 0 : (s >> slice_shift[j]) & ((int64_t(1) << slice_dim_log2[j]) - 1);
    }
    off += val * var_stride[v];
  }
  ptrs[t] = arena_leaves + off * elem_bytes;
}

// amp (complex128) += root scalar * 2^root_exp (undoes the plan's leaf scaling, in
// fp64); advance the slice counter (one thread)
template <typename R>
__global__ void accumulate_root_kernel(const void* const* __restrict__ ptrs, int32_t root, int32_t root_exp,
                                       double2* __restrict__ amp, int64_t* __restrict__ slice_id) {
  using C2 = typename cplx_t<R>::type;
  const C2 v = *reinterpret_cast<const C2*>(ptrs[root]);
  amp->x += ldexp((double)v.x, root_exp);
  amp->y += ldexp((double)v.y, root_exp);
  *slice_id += 1;
}

}  // namespace tnd
