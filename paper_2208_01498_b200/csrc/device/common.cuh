// Shared device-side definitions of the contraction engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace tnd {

// A group of tensor indices (batch / row / contracted) of one operand: the offset of
// group coordinate x (row-major over the group's indices) is the sum of two table
// lookups, because every dimension is a power of two and offsets are additive over
// the bits of x:  off(x) = tab[hi + (x >> lo_bits)] + tab[lo + (x & (2^lo_bits - 1))].
struct GroupMap {
  int32_t bits;      // log2 of the group size
  int32_t lo_bits;
  int64_t lo_off;    // offsets into the int64 table pool
  int64_t hi_off;
};

__device__ __forceinline__ int64_t gmap(const int64_t* __restrict__ tab, const GroupMap& g, int64_t x) {
  return __ldg(tab + g.hi_off + (x >> g.lo_bits)) + __ldg(tab + g.lo_off + (x & ((int64_t(1) << g.lo_bits) - 1)));
}

// One pairwise step C[b][m][n] = sum_k A[b][m][k] * B[b][k][n] on the small path.
struct SmallStep {
  int32_t a, b, c;                 // node ids in the device pointer table
  int32_t nb_bits, m_bits, n_bits, k_bits;
  int32_t g_log2;                  // log2 threads cooperating on one output (0, 5 or 7)
  int32_t opc;                     // outputs per CTA
  int32_t pad;
  GroupMap Ab, Am, Ak, Bb, Bk, Bn;
};

// Offset tables of a step whose kernel reads its raw operands (no pack pass): batch /
// free / contracted groups of A (rows M) and B (rows N) in their stored layouts, the
// operands' node ids, and whether each operand's stride-1 index is a contracted one.
struct GatherMaps {
  GroupMap Ab, Am, Ak, Bb, Bn, Bk;
  int32_t a_node, b_node;
  int32_t a_kfast, b_kfast;
};

template <typename T> struct cplx_t;
template <> struct cplx_t<float> { using type = float2; };
template <> struct cplx_t<double> { using type = double2; };

}  // namespace tnd
