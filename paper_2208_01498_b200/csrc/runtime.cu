// Runtime of the B200 contraction engine: C-ABI (include/tn.h), execution plans,
// device arena, launch schedule and CUDA-graph replay.
//
// A plan turns (network, order) into:
//   * leaf tensors resident in HBM, output legs and sliced indices moved to the
//     front so that binding a bitstring / slice is a pointer offset (no copies);
//   * for every pairwise step of the order (Eq. (3)), its index classes
//     (batch / left / right / contracted) and a kernel path: the warp-batched small
//     kernel (one launch per wave of independent steps) or the tcgen05 GEMM
//     (pack + GEMM) for GEMM-shaped complex64 steps;
//   * one device arena: every intermediate and every pack buffer gets an offset by
//     first-fit over its live interval in the launch sequence (memory planner);
//   * one CUDA graph per slice, replayed for every slice and bitstring.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "device/common.cuh"
#include "device/gemm_tc.cu"
#include "device/small.cu"
#include "device/skinny.cu"
#include "device/zgemm.cu"
#include "host/tn_host.hpp"
#include "tn.h"

using tnd::GroupMap;
using tnd::PackDesc;
using tnd::SmallStep;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define CK(x)                                                                                         \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) throw Err(TN_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)

template <class F>
int guard(F&& f) {
  try {
    f();
    return TN_OK;
  } catch (const Err& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TN_EINTERNAL;
  }
}

constexpr int OUTS_PER_CTA = 512;
constexpr int64_t ALIGN = 1024;

// ------------------------------------------------------------- table pool ---
struct TabPool {
  std::vector<int64_t> v;
  // dims: (log2 dim, element stride) of the group's indices in group order (last fastest)
  GroupMap add(const std::vector<std::pair<int, int64_t>>& g) {
    int bits = 0;
    for (auto& p : g) bits += p.first;
    GroupMap m;
    m.bits = bits;
    m.lo_bits = bits - bits / 2;
    auto off = [&](int64_t x) {
      int64_t o = 0;
      int sh = 0;
      for (int i = (int)g.size() - 1; i >= 0; --i) {
        o += ((x >> sh) & ((int64_t(1) << g[i].first) - 1)) * g[i].second;
        sh += g[i].first;
      }
      return o;
    };
    m.lo_off = (int64_t)v.size();
    for (int64_t x = 0; x < (int64_t(1) << m.lo_bits); ++x) v.push_back(off(x));
    m.hi_off = (int64_t)v.size();
    for (int64_t y = 0; y < (int64_t(1) << (bits - m.lo_bits)); ++y) v.push_back(off(y << m.lo_bits));
    return m;
  }
};

struct NodeLayout {
  std::vector<int> inds;  // stored order (row-major)
  int bits = 0;
};

std::vector<std::pair<int, int64_t>> group_of(const std::vector<int>& group, const NodeLayout& L,
                                              const std::vector<int>& l2) {
  // element strides of L's stored layout
  std::vector<int64_t> st(L.inds.size());
  int64_t acc = 1;
  for (int k = (int)L.inds.size() - 1; k >= 0; --k) {
    st[k] = acc;
    acc <<= l2[L.inds[k]];
  }
  std::vector<std::pair<int, int64_t>> g;
  for (int i : group) {
    auto it = std::find(L.inds.begin(), L.inds.end(), i);
    if (it == L.inds.end()) throw Err(TN_EINTERNAL, "index not in operand");
    g.push_back({l2[i], st[it - L.inds.begin()]});
  }
  return g;
}

// index classes of a pairwise step
struct Classes {
  std::vector<int> batch, lfree, rfree, contr;
};
Classes classify(const NodeLayout& A, const NodeLayout& B, const std::set<int>& kept) {
  Classes c;
  std::set<int> sb(B.inds.begin(), B.inds.end()), sa(A.inds.begin(), A.inds.end());
  for (int i : A.inds) {
    if (sb.count(i)) (kept.count(i) ? c.batch : c.contr).push_back(i);
    else {
      if (!kept.count(i)) throw Err(TN_EUNSUPPORTED, "index private to one operand must be kept");
      c.lfree.push_back(i);
    }
  }
  for (int i : B.inds)
    if (!sa.count(i)) {
      if (!kept.count(i)) throw Err(TN_EUNSUPPORTED, "index private to one operand must be kept");
      c.rfree.push_back(i);
    }
  return c;
}
int sum_bits(const std::vector<int>& g, const std::vector<int>& l2) {
  int b = 0;
  for (int i : g) b += l2[i];
  return b;
}

// ---------------------------------------------------------- tensor maps -----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Err(TN_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}
// packed operand planes [b][plane][rows][K] fp16; a box = BK x box_rows x all planes
CUtensorMap make_plane_map(void* base, int k_bits, int r_bits, int nb_bits, int box_rows, int planes) {
  CUtensorMap m;
  cuuint64_t dims[3] = {cuuint64_t(1) << k_bits, cuuint64_t(1) << r_bits, cuuint64_t(planes) << nb_bits};
  cuuint64_t strides[2] = {(cuuint64_t(1) << k_bits) * 2, (cuuint64_t(1) << (k_bits + r_bits)) * 2};
  cuuint32_t box[3] = {(cuuint32_t)tnd::tc::BK, (cuuint32_t)box_rows, (cuuint32_t)planes};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Err(TN_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// planar operand [b][2][rows][K] (fp32 or fp64) of the staged skinny kernel: 3-D map
// (K, rows, 2 << nb_bits), boxes {box_k, box_rows, 2 planes}, no swizzle
CUtensorMap make_planar_map(void* base, int k_bits, int r_bits, int nb_bits, int box_k, int box_rows, int esz_real) {
  CUtensorMap m;
  cuuint64_t dims[3] = {cuuint64_t(1) << k_bits, cuuint64_t(1) << r_bits, cuuint64_t(2) << nb_bits};
  cuuint64_t strides[2] = {(cuuint64_t(1) << k_bits) * esz_real, (cuuint64_t(1) << (k_bits + r_bits)) * esz_real};
  cuuint32_t box[3] = {(cuuint32_t)box_k, (cuuint32_t)box_rows, 2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, esz_real == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base,
                           dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Err(TN_ECUDA, "cuTensorMapEncodeTiled (planar) failed: " + std::to_string((int)r));
  return m;
}

// C of a tensor-core step, [rows][N] complex64 as [rows][2N] fp32, for TMA stores of 32 x
// 16-complex boxes (SWIZZLE_128B)
CUtensorMap make_c_map(void* base, int n_bits, int64_t rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cuuint64_t(2) << n_bits, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t(2) << n_bits) * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Err(TN_ECUDA, "cuTensorMapEncodeTiled (C) failed: " + std::to_string((int)r));
  return m;
}

// The dynamic shared memory limit is a per-device function attribute: set it once per
// (kernel, current device), under a lock (plans may live on several devices / threads).
void ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done.count({fn, dev})) return;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({fn, dev});
}

template <int BN>
void ensure_gemm_attr() {
  ensure_smem_attr((const void*)tnd::tc::cgemm_f16x2s_kernel<BN>, tnd::tc::Cfg<BN>::SMEM);
}

// one tensor-core step: pack X, pack Y, GEMM
// split-K only to fill the GPU: a step with few output tiles splits K over CTAs (each
// split >= 16 stages), summed in fp64 by splitk_reduce_kernel
constexpr int MIN_SPLIT_STAGES = 16;

enum { K_TC = 0, K_DMMA = 1, K_SKINNY = 2, K_WIDE = 3 };
struct TcStep {
  int kind = K_TC;                // K_TC: complex64 block-scaled fp16x2 tcgen05; K_DMMA: complex128
                                  // DMMA; K_SKINNY / K_WIDE: CUDA-core split-K / wide (skinny.cu)
  int esz = 8;                    // bytes per complex element of the plan
  PackDesc px, py;
  int64_t x_off = 0, y_off = 0;   // pack buffers (arena offsets)
  int64_t p_off = 0;              // split-K partials (arena offset), S > 1 only
  int S = 1;                      // K splits per slab
  int k_lo = 0;                   // log2 K of one slab
  int n_slabs = 1;                // K-slabs packed and multiplied in turn (bounded pack buffers)
  std::vector<int64_t> slab_x, slab_y;   // source offsets of each slab
  int32_t c_node;
  int nb_bits, m_bits, n_bits, k_bits, BN;
  bool pair = false;              // K_TC on CTA pairs (cta_group::2, 256 x 128 tiles)
  int kc_split = 1 << 30;         // K stages per split (K_TC)
  int m_lo = 0;                   // log2 rows of X per row slab (= m_bits without row slabs)
  int n_mslabs = 1;               // row slabs of X (bounded pack buffer when C is large)
  int n_kchunks = 1;              // pair kernel launches over consecutive K ranges of kc_split stages
  CUtensorMap ta, tb;
  CUtensorMap tc;                 // C [b * M_c + row][N] complex64 for TMA stores (pair kernels)
  double flops;
  bool gather = false;            // K_DMMA: operands gathered by the GEMM (no pack pass)
  tnd::zg::GatherMaps gmaps{};
};

// TN_DMMA_GATHER=0 / TN_WIDE_GATHER=0: complex128 tensor-core steps / wide steps pack
// their operands first (A/B switches)
bool dmma_gather_enabled() {
  static bool v = [] {
    const char* e = std::getenv("TN_DMMA_GATHER");
    return !(e && e[0] == '0');
  }();
  return v;
}
bool wide_gather_enabled() {
  static bool v = [] {
    const char* e = std::getenv("TN_WIDE_GATHER");
    return !(e && e[0] == '0');
  }();
  return v;
}

// profiling marks: an event recorded before each kernel class (0 small, 1 pack, 2 gemm,
// 3 reduce, 4 other) and its kernel (TN_K_*, tn_profile.k_*); time between consecutive
// marks is attributed to the earlier one
struct Marks {
  std::vector<std::pair<cudaEvent_t, int>> v;
  std::vector<int> fine;
  std::vector<std::string> tags;
  void mark(cudaStream_t st, int cat, int k, std::string tag = "") {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    // under stream capture (a profiled graph) the record must become an external event
    // record node: a plain record is only an intra-graph dependency marker, not timed
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else CK(cudaEventRecord(e, st));
    v.push_back({e, cat});
    fine.push_back(k);
    tags.push_back(std::move(tag));
  }
};
// TN_PROFILE_DUMP=<ms>: tn_contract_profiled prints every interval longer than <ms>
double profile_dump_ms() {
  static double v = [] {
    const char* e = std::getenv("TN_PROFILE_DUMP");
    return e ? std::atof(e) : -1.0;
  }();
  return v;
}
std::string shape_tag(const char* kind, int nb, int m, int n, int k) {
  return std::string(kind) + " nb=" + std::to_string(nb) + " m=" + std::to_string(m) + " n=" + std::to_string(n) +
         " k=" + std::to_string(k);
}

// TN_GEMM_PERSIST=0 launches one CTA pair per output tile instead of the persistent kernel
bool gemm_persist_enabled() {
  static bool v = [] {
    const char* e = std::getenv("TN_GEMM_PERSIST");
    return !(e && e[0] == '0');
  }();
  return v;
}

// the persistent pair kernel serves steps with <= 32 K stages per tile
bool uses_persist(const TcStep& t) {
  static const int64_t max_stages = [] {       // TN_PERSIST_MAX_STAGES: experiments
    const char* e = std::getenv("TN_PERSIST_MAX_STAGES");
    return e ? (int64_t)std::atoll(e) : int64_t(32);
  }();
  const int64_t stages_per_tile = std::min<int64_t>(t.kc_split, ((int64_t(1) << t.k_lo) + tnd::tc::BK - 1) / tnd::tc::BK);
  return t.kind == K_TC && t.pair && gemm_persist_enabled() && stages_per_tile <= max_stages;
}

// kernel class (TN_K_*) of a complex64 tensor-core step's GEMM launches
int gemm_class(const TcStep& t) {
  return uses_persist(t) ? TN_K_GEMM_PERSIST : t.pair ? TN_K_GEMM_PAIR : TN_K_GEMM_SINGLE;
}

// bytes of the 4 fp16 planes of a packed complex64 operand (its chunk scales follow)
int64_t plane_bytes(const PackDesc& d) { return int64_t(8) << (d.nb_bits + d.r_bits + d.k_bits); }

// 64 x 32 tiles for a gathered DMMA step (TN_DMMA_BN=32, an experiment switch): meant to
// fill the partial last wave of 64 x 64 tiles (configs[3]'s dominant step: 1024 tiles =
// 3.46 waves of 296 slots), but the halved warp tile (one 16-row fragment per warp) costs
// more than the tail: configs[3] 1.92 -> 1.96 ms per amplitude (measured), so 64 wide
// (also measured per step: 64 x 32 tiles only for steps under one wave of 64 x 64 tiles,
// configs[3]'s K = 256 steps, 0.096 -> 0.107 ms each: the tile count is not what limits them)
bool dmma_bn32(const TcStep&) {
  static const bool v = [] {
    const char* e = std::getenv("TN_DMMA_BN");
    return e && std::atoi(e) == 32;
  }();
  return v;
}

// Tail split of a gathered DMMA step (2 CTAs of 64 x 64 tiles per SM: 296 slots): T tiles
// are F full waves plus r tiles.  The F waves run as one launch; the r tail tiles run as a
// second launch with K split over clusters of ks in {2, 4} CTAs (the leader adds the
// partial accumulators over DSMEM, zgemm.cu), so the tail takes ceil(ks r / 296) / ks of a
// wave instead of one (configs[3]'s dominant step: 1024 tiles = 3 waves + 136 -> 3.5 wave
// times).  ks is the choice with the least estimated time (+ 0.05 wave per split for the
// reduction), each CTA keeping >= 128 of K.  An experiment switch (TN_DMMA_TAIL=1), off by
// default: measured slower on configs[3] (its dominant step 0.577 -> 0.60 ms, DMMA 1.02 ->
// 1.05 ms per amplitude): a partial wave of single CTAs per SM already runs near the SM's
// DMMA rate (2 CTAs per SM share one pipe), and the second launch adds a drain bubble.
struct DmmaSplit {
  int64_t tiles = 0, n_main = 0;   // linear tiles (batch-major); the first n_main in the main launch
  int ks = 1;                      // K split of the tail tiles (1: no tail launch)
};
DmmaSplit dmma_split(const TcStep& t) {
  static const bool on = [] {
    const char* e = std::getenv("TN_DMMA_TAIL");
    return e && e[0] == '1';
  }();
  DmmaSplit d;
  const int bn = dmma_bn32(t) ? 32 : tnd::zg::BN;
  d.tiles = ((((int64_t(1) << t.n_bits) + bn - 1) / bn) * (((int64_t(1) << t.m_bits) + tnd::zg::BM - 1) / tnd::zg::BM))
            << t.nb_bits;
  d.n_main = d.tiles;
  if (!on || !t.gather || dmma_bn32(t)) return d;
  const int64_t S = 296, F = d.tiles / S, r = d.tiles % S;
  if (r == 0) return d;
  double best = (double)F + 1.0;
  for (int ks : {2, 4}) {
    if (t.k_bits - (ks == 2 ? 1 : 2) < 7) continue;
    const double est = (double)F + (double)((ks * r + S - 1) / S) / ks + 0.05;
    if (est < best) { best = est; d.ks = ks; }
  }
  if (d.ks > 1) d.n_main = F * S;
  return d;
}

// kernel launches of a gathered DMMA step
int dmma_launches(const TcStep& t) {
  const DmmaSplit d = dmma_split(t);
  return (d.n_main > 0 ? 1 : 0) + (d.ks > 1 ? 1 : 0);
}

void launch_dmma(const TcStep& t, char* arena, void* const* ptrs_d, const int64_t* tab_d, cudaStream_t st,
                 Marks* mk) {
  const int64_t tiles = (((int64_t(1) << t.n_bits) + tnd::zg::BN - 1) / tnd::zg::BN) *
                        (((int64_t(1) << t.m_bits) + tnd::zg::BM - 1) / tnd::zg::BM);
  dim3 grid((unsigned)tiles, 1, 1u << t.nb_bits);
  if (t.gather) {
    if (mk) mk->mark(st, 2, TN_K_DMMA, profile_dump_ms() >= 0 ? shape_tag("dmma gather", t.nb_bits, t.m_bits, t.n_bits, t.k_bits) : "");
    const DmmaSplit d = dmma_split(t);
    const int32_t M = 1 << t.m_bits, N = 1 << t.n_bits, K = 1 << t.k_bits;
    if (dmma_bn32(t)) {
      ensure_smem_attr((const void*)tnd::zg::zgemm_dmma_gather_kernel<32>, tnd::zg::g_smem<32>());
      tnd::zg::zgemm_dmma_gather_kernel<32><<<dim3((unsigned)d.tiles, 1, 1), tnd::zg::THREADS, tnd::zg::g_smem<32>(), st>>>(
          t.gmaps, tab_d, ptrs_d, t.c_node, M, N, K, 1, int64_t(0));
      g_launches++;
      CK(cudaGetLastError());
      return;
    }
    ensure_smem_attr((const void*)tnd::zg::zgemm_dmma_gather_kernel<64>, tnd::zg::g_smem<64>());
    if (d.n_main > 0) {
      tnd::zg::zgemm_dmma_gather_kernel<64><<<dim3((unsigned)d.n_main, 1, 1), tnd::zg::THREADS, tnd::zg::g_smem<64>(), st>>>(
          t.gmaps, tab_d, ptrs_d, t.c_node, M, N, K, 1, int64_t(0));
      g_launches++;
    }
    if (d.ks > 1) {              // the tail tiles, K split over clusters of d.ks CTAs
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(d.tiles - d.n_main), (unsigned)d.ks, 1);
      cfg.blockDim = dim3(tnd::zg::THREADS, 1, 1);
      cfg.dynamicSmemBytes = tnd::zg::g_smem<64>();
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 1;
      at[0].val.clusterDim.y = (unsigned)d.ks;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, tnd::zg::zgemm_dmma_gather_kernel<64>, t.gmaps, tab_d, ptrs_d, t.c_node, M, N, K,
                            (int32_t)d.ks, d.n_main));
      g_launches++;
    }
    CK(cudaGetLastError());
    return;
  }
  ensure_smem_attr((const void*)tnd::zg::zgemm_dmma_kernel, tnd::zg::SMEM);
  if (mk) mk->mark(st, 1, TN_K_PACK_PLANAR, profile_dump_ms() >= 0 ? shape_tag("f64 pack", t.nb_bits, t.m_bits, t.n_bits, t.k_bits) : "");
  for (const PackDesc* d : {&t.px, &t.py}) {
    const int64_t blocks = std::min<int64_t>(int64_t(1) << d->tile_bits, 148 * 8);
    tnd::pack_planar_kernel<double><<<(unsigned)blocks, tnd::PACK_THREADS, 0, st>>>(
        ptrs_d, *d, tab_d, reinterpret_cast<double*>(arena + (d == &t.px ? t.x_off : t.y_off)), 0);
    g_launches++;
  }
  if (mk) mk->mark(st, 2, TN_K_DMMA, profile_dump_ms() >= 0 ? shape_tag("dmma", t.nb_bits, t.m_bits, t.n_bits, t.k_bits) : "");
  tnd::zg::zgemm_dmma_kernel<<<grid, tnd::zg::THREADS, tnd::zg::SMEM, st>>>(
      reinterpret_cast<const double*>(arena + t.x_off), reinterpret_cast<const double*>(arena + t.y_off), ptrs_d,
      t.c_node, 1 << t.m_bits, 1 << t.n_bits, 1 << t.k_bits);
  g_launches++;
  CK(cudaGetLastError());
}

// Launch shape of the staged skinny kernel (skinny2_kernel), a function of the step's bits:
// 4 x 2 output groups (at most 16 per item; 32 groups -> two items per (batch, K range),
// one per half of X's rows), WPG = 16 / groups warps per group taking its stages in turn,
// stages of KS <= 256 elements of K (the TMA box limit; <= 48 KB), 2-8 stages in <= 200 KB,
// and K split into S ranges per batch so that >= 2 waves of items cover the 148 SMs.
struct Sk2Shape {
  bool use = false;
  int gm_bits = 0, gn_bits = 0, m_split = 1, wpg = 1, ks = 0, stages = 0, S = 1;
  int64_t kc = 0;
  size_t smem = 0;
};
Sk2Shape skinny2_shape(const TcStep& t) {
  Sk2Shape h;
  static const bool on = [] {
    const char* e = std::getenv("TN_SKINNY_V2");
    return !(e && e[0] == '0');
  }();
  if (!on) return h;
  const int esz = t.esz / 2;                     // bytes per real element of a plane
  h.gm_bits = std::min(t.m_bits, 2);
  h.gn_bits = std::min(t.n_bits, 1);
  int ng_bits = (t.m_bits - h.gm_bits) + (t.n_bits - h.gn_bits);
  if (ng_bits > 4) {
    if (ng_bits > 5 || t.m_bits - h.gm_bits < 1) return h;
    h.m_split = 2;
    ng_bits = 4;
  }
  h.wpg = 16 >> ng_bits;
  const int64_t K = int64_t(1) << t.k_lo;
  const int64_t ks_min = int64_t(32) * (16 / esz);       // one 16-byte vector per lane
  if (K < ks_min) return h;
  const int rows = 2 * ((1 << t.m_bits) / h.m_split + (1 << t.n_bits));
  int64_t ks = ks_min;
  while (ks * 2 <= std::min<int64_t>(K, 256) && rows * ks * 2 * esz <= 48 * 1024) ks *= 2;
  const size_t stage = (size_t)rows * ks * esz;
  if (stage > 100 * 1024) return h;
  h.ks = (int)ks;
  h.stages = (int)std::min<size_t>(8, (200 * 1024) / stage);
  h.smem = h.stages * stage + 2 * 8 * h.stages;
  const int64_t per_batch = (int64_t)h.m_split << t.nb_bits;
  const int64_t want = std::max<int64_t>(1, (2 * 148 + per_batch - 1) / per_batch);
  h.S = (int)std::max<int64_t>(1, std::min<int64_t>(want, K / ks));
  h.kc = (K + h.S - 1) / h.S;
  h.kc = (h.kc + ks - 1) / ks * ks;
  h.S = (int)((K + h.kc - 1) / h.kc);
  h.use = true;
  return h;
}

// one CTA per wide tile (the block scheduler balances the SMs as CTAs retire) instead of a
// grid-stride loop over 8 CTAs per SM, whose last round leaves slots idle: configs[3]'s
// wide steps 0.221 -> 0.211 ms per amplitude, the c64 (5, 26, 3) step 3.81 -> 3.74 ms;
// TN_WIDE_FULLGRID=0 restores the grid-stride launch
bool wide_full_grid() {
  static const bool on = [] {
    const char* e = std::getenv("TN_WIDE_FULLGRID");
    return !(e && e[0] == '0');
  }();
  return on;
}

// complex64 wide steps (gathered, K = 16) with packed fp32 pairs (FFMA2); TN_WIDE_FFMA2=0: scalar FFMA
bool wide_ffma2() {
  static const bool on = [] {
    const char* e = std::getenv("TN_WIDE_FFMA2");
    return !(e && e[0] == '0');
  }();
  return on;
}

// skinny steps without K-slabs (K <= 2^22) read their raw operands (bskinny_kernel,
// skinny.cu): one CTA per (batch, K range), no planar packs; a reduction launch only when
// few batches split K.  configs[3]'s (10, 4, 4, 7) step: packs + staged kernel 101 us ->
// 45 us; TN_SKINNY_GATHER=0 packs instead
bool bskinny_ok(const TcStep& t) {
  static const bool on = [] {
    const char* e = std::getenv("TN_SKINNY_GATHER");
    return !(e && e[0] == '0');
  }();
  return on && t.kind == K_SKINNY && t.n_slabs == 1 && t.k_bits <= 22 && t.m_bits + t.n_bits <= 8;
}
// K ranges per batch of a gathered skinny step: enough items for 4 CTAs per SM, each range
// >= 256 of K
int bskinny_s_bits(const TcStep& t) {
  int s = 0;
  while ((int64_t(1) << (t.nb_bits + s)) < 4 * 148 && t.k_bits - s > 8) ++s;
  return s;
}
// K chunk staged per item: the largest with <= 48 KB of shared memory (4 CTAs per SM)
int bskinny_s_bits(const TcStep& t);
int bskinny_kc_bits(const TcStep& t) {
  int kc = t.k_bits - bskinny_s_bits(t);             // a chunk never crosses a K range
  while (kc > 0 && tnd::bskinny_smem(t.m_bits, t.n_bits, kc, t.esz) > 48 * 1024) --kc;
  return kc;
}

// tensor maps of a staged skinny step's planar operands (in the arena at x_off / y_off)
void set_skinny_maps(TcStep& t, char* base) {
  if (t.kind != K_SKINNY || t.gather) return;
  const Sk2Shape h = skinny2_shape(t);
  if (!h.use) return;
  t.ta = make_planar_map(base + t.x_off, t.k_lo, t.m_bits, t.nb_bits, h.ks, (1 << t.m_bits) / h.m_split, t.esz / 2);
  t.tb = make_planar_map(base + t.y_off, t.k_lo, t.n_bits, t.nb_bits, h.ks, 1 << t.n_bits, t.esz / 2);
}

// partial sums per batch of a skinny step: K ranges x warps sharing an output group
int skinny_ws(const TcStep& t) {
  const Sk2Shape h = skinny2_shape(t);
  if (h.use) return h.wpg;
  int gm, gn, ng, ws;
  tnd::skinny_groups(t.m_bits, t.n_bits, gm, gn, ng, ws);
  return ws;
}

// skinny / wide steps: planar packs + CUDA-core kernel (+ ordered split-K reduction)
template <typename R>
void launch_cuda_core(const TcStep& t, char* arena, void* const* ptrs_d, const int64_t* tab_d, cudaStream_t st,
                      Marks* mk) {
  auto pack = [&](const PackDesc& d, int64_t off, int64_t base) {
    const int64_t blocks = std::min<int64_t>(int64_t(1) << d.tile_bits, 148 * 8);
    tnd::pack_planar_kernel<R><<<(unsigned)blocks, tnd::PACK_THREADS, 0, st>>>(
        ptrs_d, d, tab_d, reinterpret_cast<R*>(arena + off), base);
    g_launches++;
  };
  const R* X = reinterpret_cast<const R*>(arena + t.x_off);
  const R* Y = reinterpret_cast<const R*>(arena + t.y_off);
  const bool dump = profile_dump_ms() >= 0;
  for (int s = 0; s < t.n_slabs; ++s) {
    if (!t.gather) {   // (gathered wide steps read their raw operands)
      if (mk) mk->mark(st, 1, TN_K_PACK_PLANAR, dump ? shape_tag("planar pack", t.nb_bits, t.m_bits, t.n_bits, t.k_bits) : "");
      pack(t.px, t.x_off, t.slab_x.empty() ? 0 : t.slab_x[s]);
      pack(t.py, t.y_off, t.slab_y.empty() ? 0 : t.slab_y[s]);
    }
    if (mk) mk->mark(st, 0, t.kind == K_SKINNY ? TN_K_SKINNY : TN_K_WIDE,
                     dump ? shape_tag(t.kind == K_SKINNY ? "skinny" : "wide", t.nb_bits, t.m_bits, t.n_bits,
                                             t.k_bits) : "");
    if (t.kind == K_SKINNY && t.gather) {     // batched skinny, gathered: one CTA per batch
      const int kcb = bskinny_kc_bits(t);
      const int smem = tnd::bskinny_smem(t.m_bits, t.n_bits, kcb, t.esz);
      ensure_smem_attr((const void*)tnd::bskinny_kernel<R>, 48 * 1024 + 4096);
      const int64_t nbat = int64_t(1) << t.nb_bits;
      const int sb = bskinny_s_bits(t);
      double2* partial = reinterpret_cast<double2*>(arena + t.p_off);
      tnd::bskinny_kernel<R><<<(unsigned)std::min<int64_t>(nbat << sb, wide_full_grid() ? (int64_t(1) << 24) : 148 * 4), tnd::BS_THREADS, smem, st>>>(
          t.gmaps, tab_d, ptrs_d, t.c_node, t.m_bits, t.n_bits, t.k_bits, kcb, nbat, sb, partial);
      g_launches++;
      if (sb > 0) {
        if (mk) mk->mark(st, 3, TN_K_REDUCE);
        const int64_t n_out = int64_t(1) << (t.nb_bits + t.m_bits + t.n_bits);
        if (n_out <= 4 * 148)
          tnd::skinny_reduce_cta_kernel<R><<<(unsigned)n_out, 256, 0, st>>>(
              partial, 1 << sb, 1 << (t.m_bits + t.n_bits), n_out, ptrs_d, t.c_node, 0);
        else
          tnd::skinny_reduce_kernel<R><<<(unsigned)std::min<int64_t>((n_out + 7) / 8, 148 * 16), 256, 0, st>>>(
              partial, 1 << sb, 1 << (t.m_bits + t.n_bits), n_out, ptrs_d, t.c_node, 0);
        g_launches++;
      }
      continue;
    }
    const Sk2Shape h2 = t.kind == K_SKINNY ? skinny2_shape(t) : Sk2Shape{};
    if (t.kind == K_SKINNY && h2.use) {
      const int64_t K = int64_t(1) << t.k_lo;
      double2* partial = reinterpret_cast<double2*>(arena + t.p_off);
      const int64_t items = ((int64_t)h2.m_split << t.nb_bits) * t.S;
      const unsigned grid = (unsigned)std::min<int64_t>(items, 148);
#define TN_SKINNY2(GMB, GNB)                                                                                          \
  if (h2.gm_bits == GMB && h2.gn_bits == GNB) {                                                                       \
    ensure_smem_attr((const void*)tnd::skinny2_kernel<R, 1 << GMB, 1 << GNB>, 210 * 1024); /* >= any h2.smem */  \
    tnd::skinny2_kernel<R, 1 << GMB, 1 << GNB><<<grid, tnd::SK2_THREADS, h2.smem, st>>>(                             \
        t.ta, t.tb, partial, t.m_bits, t.n_bits, K, h2.kc, t.S, 1 << t.nb_bits, h2.m_split, h2.ks, h2.stages, ptrs_d, \
        t.c_node, s > 0);                                                                                             \
  }
      TN_SKINNY2(0, 0) TN_SKINNY2(0, 1) TN_SKINNY2(1, 0) TN_SKINNY2(1, 1) TN_SKINNY2(2, 0) TN_SKINNY2(2, 1)
#undef TN_SKINNY2
      g_launches++;
      if (t.S * h2.wpg == 1) continue;   // the kernel wrote C
      if (mk) mk->mark(st, 3, TN_K_REDUCE);
      const int64_t n_out = int64_t(1) << (t.nb_bits + t.m_bits + t.n_bits);
      if (n_out <= 4 * 148)
        tnd::skinny_reduce_cta_kernel<R><<<(unsigned)n_out, 256, 0, st>>>(
            partial, t.S * h2.wpg, 1 << (t.m_bits + t.n_bits), n_out, ptrs_d, t.c_node, s > 0);
      else
        tnd::skinny_reduce_kernel<R><<<(unsigned)std::min<int64_t>((n_out + 7) / 8, 148 * 16), 256, 0, st>>>(
            partial, t.S * h2.wpg, 1 << (t.m_bits + t.n_bits), n_out, ptrs_d, t.c_node, s > 0);
      g_launches++;
    } else if (t.kind == K_SKINNY) {
      const int64_t K = int64_t(1) << t.k_lo;
      const int64_t kc = ((K + t.S - 1) / t.S + 127) / 128 * 128;   // 16-byte aligned K ranges
      double2* partial = reinterpret_cast<double2*>(arena + t.p_off);
      int gm, gn, ng, ws;
      tnd::skinny_groups(t.m_bits, t.n_bits, gm, gn, ng, ws);
      const dim3 grid((unsigned)t.S, 1u << t.nb_bits);
#define TN_SKINNY(GMB, GNB)                                                                                   \
  if (gm == GMB && gn == GNB)                                                                                 \
    tnd::skinny_kernel<R, 1 << GMB, 1 << GNB><<<grid, tnd::SK_THREADS, 0, st>>>(X, Y, partial, t.m_bits, t.n_bits, \
                                                                                 K, kc, t.S, ptrs_d, t.c_node, s > 0);
      TN_SKINNY(0, 0) TN_SKINNY(0, 1) TN_SKINNY(0, 2) TN_SKINNY(0, 3) TN_SKINNY(0, 4)
      TN_SKINNY(1, 0) TN_SKINNY(1, 1) TN_SKINNY(1, 2) TN_SKINNY(1, 3)
      TN_SKINNY(2, 0) TN_SKINNY(2, 1) TN_SKINNY(2, 2)
#undef TN_SKINNY
      g_launches++;
      if (t.S * ws == 1) continue;      // the kernel wrote C
      if (mk) mk->mark(st, 3, TN_K_REDUCE);
      const int64_t n_out = int64_t(1) << (t.nb_bits + t.m_bits + t.n_bits);
      if (n_out <= 4 * 148)
        tnd::skinny_reduce_cta_kernel<R><<<(unsigned)n_out, 256, 0, st>>>(
            partial, t.S * skinny_ws(t), 1 << (t.m_bits + t.n_bits), n_out, ptrs_d, t.c_node, s > 0);
      else
        tnd::skinny_reduce_kernel<R><<<(unsigned)std::min<int64_t>((n_out + 7) / 8, 148 * 16), 256, 0, st>>>(
            partial, t.S * skinny_ws(t), 1 << (t.m_bits + t.n_bits), n_out, ptrs_d, t.c_node, s > 0);
      g_launches++;
    } else {
      // complex64 with N >= 2: two adjacent columns per thread
      const bool two = sizeof(R) == 4 && t.n_bits >= 1;
      const int64_t tm = std::min(tnd::wd_tm<R>(), 1 << t.m_bits), tn = int64_t(tnd::WD_THREADS) * (two ? 2 : 1);
      const int64_t tiles = (int64_t(1) << (t.nb_bits + t.m_bits)) / tm * (((int64_t(1) << t.n_bits) + tn - 1) / tn);
      const unsigned grid = (unsigned)std::min<int64_t>(tiles, wide_full_grid() ? (int64_t(1) << 30) : 148 * 8);
#define TN_WIDE(CPT, KB)                                                                                    \
  if (t.k_bits == KB) {                                                                                     \
    if (t.gather)                                                                                           \
      tnd::wide_kernel<R, CPT, 1 << KB, true><<<grid, tnd::WD_THREADS, 0, st>>>(                           \
          X, Y, ptrs_d, t.c_node, t.m_bits, t.n_bits, t.k_bits, tiles, t.gmaps, tab_d);                     \
    else                                                                                                    \
      tnd::wide_kernel<R, CPT, 1 << KB, false><<<grid, tnd::WD_THREADS, 0, st>>>(                          \
          X, Y, ptrs_d, t.c_node, t.m_bits, t.n_bits, t.k_bits, tiles, t.gmaps, tab_d);                     \
  }
      if constexpr (sizeof(R) == 4) {
        // gathered, K = 16: the FFMA2 variant (8% faster there; no gain at K = 4, 8 -- bound
        // by writing C; TN_WIDE_FFMA2=0: scalar FFMA)
        if (two && t.gather && t.k_bits == 4 && wide_ffma2()) {
          tnd::wide_kernel<R, 2, 16, true, true><<<grid, tnd::WD_THREADS, 0, st>>>(
              X, Y, ptrs_d, t.c_node, t.m_bits, t.n_bits, t.k_bits, tiles, t.gmaps, tab_d);
        } else if (two) {
          TN_WIDE(2, 0) TN_WIDE(2, 1) TN_WIDE(2, 2) TN_WIDE(2, 3) TN_WIDE(2, 4)
        }
      }
      if (!two) { TN_WIDE(1, 0) TN_WIDE(1, 1) TN_WIDE(1, 2) TN_WIDE(1, 3) TN_WIDE(1, 4) }
#undef TN_WIDE
      g_launches++;
    }
  }
  CK(cudaGetLastError());
}

void launch_tc(const TcStep& t, char* arena, void* const* ptrs_d, const int64_t* tab_d, cudaStream_t st,
               Marks* mk = nullptr) {
  static bool group_set = [] {      // TN_GEMM_GROUP_M: M tiles per raster group (experiments)
    const char* e = std::getenv("TN_GEMM_GROUP_M");
    if (e && std::atoi(e) > 0) {
      const int g = std::atoi(e);
      CK(cudaMemcpyToSymbol(tnd::tc::d_group_m, &g, sizeof(int)));
    }
    const char* sp = std::getenv("TN_GEMM_SERP");
    if (sp) {
      const int v = std::atoi(sp);
      CK(cudaMemcpyToSymbol(tnd::tc::d_serp, &v, sizeof(int)));
    }
    return true;
  }();
  (void)group_set;
  if (t.kind == K_DMMA) return launch_dmma(t, arena, ptrs_d, tab_d, st, mk);
  if (t.kind == K_SKINNY || t.kind == K_WIDE) {
    if (t.esz == 8) return launch_cuda_core<float>(t, arena, ptrs_d, tab_d, st, mk);
    return launch_cuda_core<double>(t, arena, ptrs_d, tab_d, st, mk);
  }
  auto pack = [&](const PackDesc& d, int64_t off, int64_t base) {
    const int64_t blocks = std::min<int64_t>(int64_t(1) << d.tile_bits, 148 * 8);
    tnd::pack_f16x2s_kernel<<<(unsigned)blocks, tnd::PACK_THREADS, 0, st>>>(
        ptrs_d, d, tab_d, reinterpret_cast<__half*>(arena + off),
        reinterpret_cast<float*>(arena + off + plane_bytes(d)), base);
    g_launches++;
  };
  const float* sca = reinterpret_cast<const float*>(arena + t.x_off + plane_bytes(t.px));
  const float* scb = reinterpret_cast<const float*>(arena + t.y_off + plane_bytes(t.py));
  const int64_t tiles = (((int64_t(1) << t.n_bits) + t.BN - 1) / t.BN) * (((int64_t(1) << t.m_lo) + 127) / 128);
  dim3 grid((unsigned)tiles, 1, (unsigned)((1u << t.nb_bits) * t.S));
  float2* partial = t.S > 1 ? reinterpret_cast<float2*>(arena + t.p_off) : nullptr;
  // row slabs (outer) or K-slabs (inner); at most one of them has more than one slab
  for (int ms = 0; ms < t.n_mslabs; ++ms)
  for (int s = 0; s < t.n_slabs; ++s) {
    if (mk) mk->mark(st, 1, TN_K_PACK_TC, profile_dump_ms() >= 0 ? shape_tag("pack", t.nb_bits, t.m_bits, t.n_bits, t.k_bits) : "");
    pack(t.px, t.x_off, t.slab_x.empty() ? 0 : t.slab_x[t.n_mslabs > 1 ? ms : s]);
    if (ms == 0) pack(t.py, t.y_off, t.slab_y.empty() ? 0 : t.slab_y[s]);
    if (mk) mk->mark(st, 2, gemm_class(t), profile_dump_ms() >= 0 ? shape_tag("gemm", t.nb_bits, t.m_bits, t.n_bits, t.k_bits) : "");
    const int acc = s > 0;
    const int m_off = ms << t.m_lo;
    // persistent tile loop only for short K per tile (<= 32 stages): there the per-CTA
    // prologue / fill / drain is a large share; long tiles are faster one per CTA pair
    if (uses_persist(t)) {
      ensure_smem_attr((const void*)tnd::tc::cgemm2p_f16x2s_kernel, tnd::tc::Cfg2P::SMEM);
      const int64_t tiles = (int64_t(1) << (t.m_lo - 8)) * (int64_t(1) << (t.n_bits - 7)) * (int64_t(1) << t.nb_bits) * t.S;
      const int64_t n_pairs = std::min<int64_t>(tiles, 74);
      tnd::tc::cgemm2p_f16x2s_kernel<<<(unsigned)(2 * n_pairs), tnd::tc::Cfg2::THREADS, tnd::tc::Cfg2P::SMEM, st>>>(
          t.ta, t.tb, sca, scb, ptrs_d, t.c_node, 1 << t.m_lo, 1 << t.n_bits, 1 << t.k_lo, 1 << t.nb_bits, t.S,
          t.kc_split, partial, acc, m_off, 1 << t.m_bits, t.tc);
    } else if (t.pair) {
      ensure_smem_attr((const void*)tnd::tc::cgemm2_f16x2s_kernel, tnd::tc::Cfg2::SMEM);
      const int64_t pairs = (int64_t(1) << (t.m_lo - 8)) * (int64_t(1) << (t.n_bits - 7));
      dim3 grid2((unsigned)(2 * pairs), 1, (unsigned)((1u << t.nb_bits) * t.S));
      for (int ch = 0; ch < t.n_kchunks; ++ch) {
        tnd::tc::cgemm2_f16x2s_kernel<<<grid2, tnd::tc::Cfg2::THREADS, tnd::tc::Cfg2::SMEM, st>>>(
            t.ta, t.tb, sca, scb, ptrs_d, t.c_node, 1 << t.m_lo, 1 << t.n_bits, 1 << t.k_lo, 1 << t.nb_bits,
            t.kc_split, partial, acc || ch > 0, m_off, 1 << t.m_bits, t.tc, ch * t.kc_split);
        if (ch > 0) g_launches++;
      }
    } else if (t.BN == 128) {
      ensure_gemm_attr<128>();
      tnd::tc::cgemm_f16x2s_kernel<128><<<grid, tnd::tc::Cfg<128>::THREADS, tnd::tc::Cfg<128>::SMEM, st>>>(
          t.ta, t.tb, sca, scb, ptrs_d, t.c_node, 1 << t.m_lo, 1 << t.n_bits, 1 << t.k_lo, 1 << t.nb_bits, t.kc_split,
          partial, acc, m_off, 1 << t.m_bits);
    } else {
      ensure_gemm_attr<64>();
      tnd::tc::cgemm_f16x2s_kernel<64><<<grid, tnd::tc::Cfg<64>::THREADS, tnd::tc::Cfg<64>::SMEM, st>>>(
          t.ta, t.tb, sca, scb, ptrs_d, t.c_node, 1 << t.m_lo, 1 << t.n_bits, 1 << t.k_lo, 1 << t.nb_bits, t.kc_split,
          partial, acc, m_off, 1 << t.m_bits);
    }
    g_launches++;
    if (t.S > 1) {
      if (mk) mk->mark(st, 3, TN_K_REDUCE);
      const int64_t n = int64_t(1) << (t.nb_bits + t.m_bits + t.n_bits);
      const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 32);
      tnd::splitk_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(partial, t.S, n, ptrs_d, t.c_node, acc);
      g_launches++;
    }
  }
  CK(cudaGetLastError());
}

// entries of one packed K-slab operand: 2^30 (12 GB for complex64); TN_PACK_CAP_LOG2
// overrides it (tests force K-slabs on small shapes)
int pack_cap_log2() {
  static int v = [] {
    const char* e = std::getenv("TN_PACK_CAP_LOG2");
    return e ? std::atoi(e) : 30;
  }();
  return v;
}

// TN_GEMM_PAIR=0 disables the cta_group::2 GEMM (A/B comparisons)
bool gemm_pair_enabled() {
  static bool v = [] {
    const char* e = std::getenv("TN_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}

void finish_tc_shape(TcStep& t) {
  t.BN = (t.n_bits >= 7) ? 128 : 64;
  // Bounded pack buffers.  X (the larger operand) over the cap: row slabs of X when Y fits
  // whole (each slab writes its own rows of C, no extra traffic), else K-slabs (C += per
  // slab: 2|C| extra bytes per slab, cheap only when C is small).
  const int cap = pack_cap_log2();
  const int over_x = t.nb_bits + t.m_bits + t.k_bits - cap, over_y = t.nb_bits + t.n_bits + t.k_bits - cap;
  t.m_lo = t.m_bits;
  t.n_mslabs = 1;
  t.k_lo = t.k_bits;
  t.n_slabs = 1;
  static const bool row_slabs = [] {
    const char* e = std::getenv("TN_ROW_SLABS");
    return !(e && e[0] == '0');
  }();
  // row slabs pay off only for a large C (K-slabs re-read and re-write it per slab) and
  // keep >= 2 waves of CTAs per slab (no split-K inside row slabs)
  const int m_slab = t.m_bits - std::max(over_x, 0);
  const bool big_c = t.nb_bits + t.m_bits + t.n_bits >= 26;
  const bool enough_tiles = t.nb_bits + m_slab + t.n_bits >= 14 + 9;   // >= 2^9 tiles of 128 x 128
  if (row_slabs && over_x > 0 && over_y <= 0 && m_slab >= 8 && big_c && enough_tiles) {
    t.m_lo = t.m_bits - over_x;
    t.n_mslabs = 1 << over_x;
  } else {
    const int over = std::max(over_x, over_y);
    t.k_lo = std::max(std::min(t.k_bits, 5), t.k_bits - std::max(0, over));
    t.n_slabs = 1 << (t.k_bits - t.k_lo);
  }
  t.pair = gemm_pair_enabled() && t.m_lo >= 8 && t.n_bits >= 7;
  const int64_t nk_all = ((int64_t(1) << t.k_lo) + tnd::tc::BK - 1) / tnd::tc::BK;
  // CTAs without split-K: 128 x BN tiles, or 256 x 128 tiles on CTA pairs (2 CTAs each)
  const int64_t ctas = (int64_t(1) << t.nb_bits) *
                       (t.pair ? 2 * (int64_t(1) << (t.m_lo - 8)) * (int64_t(1) << (t.n_bits - 7))
                               : ((int64_t(1) << t.m_lo) + 127) / 128 * (((int64_t(1) << t.n_bits) + t.BN - 1) / t.BN));
  // split-K only below 2 waves; among the admissible splits take the best wave fill
  // (units of residency: SMs, or SM pairs for the pair kernel)
  const int64_t smax = std::max<int64_t>(1, nk_all / MIN_SPLIT_STAGES);
  const int64_t unit = t.pair ? 2 : 1, slots = t.pair ? 74 : 148;
  int64_t best = 1;
  if (t.n_mslabs == 1 && ctas < 2 * 148) {
    double best_eff = -1;
    for (int64_t S = (2 * 148 + ctas - 1) / ctas; S <= std::min<int64_t>(smax, 8 * ((2 * 148 + ctas - 1) / ctas)); ++S) {
      const double w = double(ctas / unit * S) / slots;
      const double eff = w / std::ceil(w);
      if (eff > best_eff + 0.02) { best_eff = eff; best = S; }
    }
    best = std::min<int64_t>(best, smax);
  }
  int64_t kc = (nk_all + best - 1) / best;
  kc = (kc + tnd::tc::PROMO - 1) / tnd::tc::PROMO * tnd::tc::PROMO;   // splits start on a scale chunk
  t.kc_split = (int)kc;
  t.S = (int)((nk_all + kc - 1) / kc);
  // K-chunks: a long-K pair GEMM runs as consecutive launches over K ranges of 16384
  // (8192 when K = 16384), C += by TMA reduce-add -- the waves of a launch then share the
  // operand panels of one K range in L2: DRAM reads 101 -> 71 GB and 1.31 -> 1.36 GHz under
  // the power cap on a (2^14, 2^12, 2^16) step (scripts/kslab_probe.sh); TN_GEMM_KCHUNK=0
  // turns it off
  static const bool kchunk = [] {
    const char* e = std::getenv("TN_GEMM_KCHUNK");
    return !(e && e[0] == '0');
  }();
  t.n_kchunks = 1;
  if (kchunk && t.pair && t.S == 1 && nk_all >= 512) {
    const int64_t cs = nk_all >= 1024 ? 512 : 256;
    t.kc_split = (int)cs;
    t.n_kchunks = (int)((nk_all + cs - 1) / cs);
  }
}
int64_t tc_partial_bytes(const TcStep& t) {
  if (t.kind == K_SKINNY)
    return t.gather ? (bskinny_s_bits(t) > 0 ? int64_t(16) << (t.nb_bits + bskinny_s_bits(t) + t.m_bits + t.n_bits) : 0)
                    : (int64_t(16) * t.S * skinny_ws(t)) << (t.nb_bits + t.m_bits + t.n_bits);
  if (t.kind != K_TC) return 0;
  return t.S > 1 ? (int64_t(8) * t.S) << (t.nb_bits + t.m_bits + t.n_bits) : 0;
}

// threads per output and outputs per CTA of a small step (long reductions split K)
void set_small_mode(SmallStep& d) {
  const int ob = d.nb_bits + d.m_bits + d.n_bits;
  d.g_log2 = (d.k_bits >= 10 && ob <= 12) ? 7 : (d.k_bits >= 6 && ob <= 16) ? 5 : 0;
  d.opc = (128 >> d.g_log2) * 4;
}

struct Wave {
  double flops = 0, bytes = 0;
  std::vector<SmallStep> steps;
  std::vector<int64_t> prefix;
  SmallStep* steps_d = nullptr;
  int64_t* prefix_d = nullptr;
  int32_t* cta_step_d = nullptr;    // CTA -> step (plans; nullptr: the kernel searches prefix)
  int64_t n_cta = 0;
};

template <typename R>
void launch_wave(const Wave& w, void* const* ptrs_d, const int64_t* tab_d, cudaStream_t st) {
  tnd::small_contract_kernel<R><<<(unsigned)w.n_cta, 128, 0, st>>>(w.steps_d, w.prefix_d, (int)w.steps.size(), tab_d,
                                                                     ptrs_d, w.cta_step_d);
  g_launches++;
  CK(cudaGetLastError());
}

// Pack descriptor: bit permutation from the operand's stored layout to [b][rows][k]
// (destination planes [b][planes][rows][k]); see pack_f16x2s_kernel / pack_planar_kernel.
// k_lo < k bits: only the lowest k_lo bits of the k group are packed (a K-slab); the
// source offsets of the remaining high k bits, one per slab, are appended to `slabs`.
PackDesc make_pack(TabPool& pool, int src_node, const NodeLayout& L, const std::vector<int>& batch,
                   const std::vector<int>& rows, const std::vector<int>& kg, const std::vector<int>& l2,
                   int planes = 6, int k_lo = -1, std::vector<int64_t>* slabs = nullptr, int r_lo = -1) {
  PackDesc d{};
  d.src = src_node;
  d.nb_bits = sum_bits(batch, l2);
  const int r_all = sum_bits(rows, l2);
  const int k_all = sum_bits(kg, l2);
  if (k_lo < 0 || k_lo > k_all) k_lo = k_all;
  if (r_lo < 0 || r_lo > r_all) r_lo = r_all;
  if (k_lo < k_all && r_lo < r_all) throw Err(TN_EINTERNAL, "pack: K-slabs and row slabs together");
  d.k_bits = k_lo;
  d.r_bits = r_lo;
  const int D_all = d.nb_bits + r_all + k_all;
  const int D = d.nb_bits + d.r_bits + d.k_bits, RK = d.r_bits + d.k_bits;
  d.plane = int64_t(1) << RK;
  // source bit of every destination bit
  std::map<int, int> src_shift;
  {
    int sh = 0;
    for (int k = (int)L.inds.size() - 1; k >= 0; --k) { src_shift[L.inds[k]] = sh; sh += l2[L.inds[k]]; }
  }
  std::vector<int> order = batch;
  order.insert(order.end(), rows.begin(), rows.end());
  order.insert(order.end(), kg.begin(), kg.end());
  std::vector<int> pi_all(D_all), pi(D);
  {
    int sh = 0;
    for (int k = (int)order.size() - 1; k >= 0; --k) {
      int i = order[k];
      for (int u = 0; u < l2[i]; ++u) pi_all[sh + u] = src_shift.at(i) + u;
      sh += l2[i];
    }
  }
  // destination bits of the full order: [0, k_all) K, [k_all, k_all + r_all) rows, then
  // batch.  A slab fixes either the top K bits [k_lo, k_all) (K-slab) or the top row bits
  // [k_all + r_lo, k_all + r_all) (row slab); the remaining bits shift down.
  const int f0 = k_lo < k_all ? k_lo : k_all + r_lo;                 // first fixed bit
  const int nf = (k_all - k_lo) + (r_all - r_lo);                   // fixed bits
  for (int j = 0; j < D; ++j) pi[j] = j < f0 ? pi_all[j] : pi_all[j + nf];
  if (slabs) {
    slabs->clear();
    for (int64_t s = 0; s < (int64_t(1) << nf); ++s) {
      int64_t o = 0;
      for (int u = 0; u < nf; ++u) if ((s >> u) & 1) o += int64_t(1) << pi_all[f0 + u];
      slabs->push_back(o);
    }
  }
  auto dst_contrib = [&](int dbit) -> int64_t {
    return dbit < RK ? (int64_t(1) << dbit) : ((int64_t(1) << (dbit - RK)) * planes * d.plane);
  };
  std::vector<char> inT(D, 0);
  int t = 0;
  for (int j = 0; j < std::min(tnd::SCALE_LOG2, D); ++j) if (!inT[j]) { inT[j] = 1; ++t; }
  for (int j = 0; j < D; ++j) if (pi[j] < 4 && !inT[j]) { inT[j] = 1; ++t; }
  for (int j = 0; j < D && t < std::min(tnd::PACK_MAX_T, D); ++j) if (!inT[j]) { inT[j] = 1; ++t; }
  if (t < 3 || (planes == 4 && (t < 8 || k_lo < 4)))
    throw Err(TN_EUNSUPPORTED, "tensor-core pack needs >= 256 elements and K >= 16 per operand");
  d.t_bits = t;
  int ld = 0;
  while (ld < D && inT[ld]) ++ld;
  d.ld = std::min(ld, RK);
  // the pack kernels write 8 consecutive destination elements per thread: a (batch, row)
  // block of the destination must hold >= 8 contiguous entries (rows + K bits >= 3)
  if (d.ld < 3) throw Err(TN_EUNSUPPORTED, "pack: an operand needs rows + K >= 8 entries per batch");
  std::vector<int> Tsrc, Tdst, nonT;
  for (int j = 0; j < D; ++j) (inT[j] ? Tdst : nonT).push_back(j);
  Tsrc = Tdst;
  std::sort(Tsrc.begin(), Tsrc.end(), [&](int a, int b) { return pi[a] < pi[b]; });
  std::map<int, int> rank;
  for (size_t k = 0; k < Tdst.size(); ++k) rank[Tdst[k]] = (int)k;
  d.e_src = (int64_t)pool.v.size();
  for (int64_t e = 0; e < (int64_t(1) << t); ++e) {
    int64_t o = 0;
    for (int i = 0; i < t; ++i) if ((e >> i) & 1) o += int64_t(1) << pi[Tsrc[i]];
    pool.v.push_back(o);
  }
  d.e_q = (int64_t)pool.v.size();
  for (int64_t e = 0; e < (int64_t(1) << t); ++e) {
    int64_t q = 0;
    for (int i = 0; i < t; ++i) if ((e >> i) & 1) q |= int64_t(1) << rank[Tsrc[i]];
    pool.v.push_back(q);
  }
  d.tile_bits = (int)nonT.size();
  std::vector<std::pair<int, int64_t>> gs, gd, gq;
  for (int k = (int)nonT.size() - 1; k >= 0; --k) {
    gs.push_back({1, int64_t(1) << pi[nonT[k]]});
    gd.push_back({1, dst_contrib(nonT[k])});
  }
  for (int k = (int)Tdst.size() - 1; k >= d.ld; --k) gq.push_back({1, dst_contrib(Tdst[k])});
  d.tile_src = pool.add(gs);
  d.tile_dst = pool.add(gd);
  d.q_hi = pool.add(gq);
  return d;
}

// Order of an index group (contracted K, or X's rows) in the packed operand.  With slabs
// the slab bits are the HIGHEST bits of the group (its first indices): take them from
// the indices with the largest strides in `big`, so every slab reads contiguous runs of
// it (slab bits among its fast bits would read 1 element per 2^bits, re-fetching each
// sector once per slab).
std::vector<int> slab_k_order(const std::vector<int>& contr, const NodeLayout& big, const std::vector<int>& l2,
                              int n_slabs) {
  std::vector<int> k = contr;
  if (n_slabs <= 1) return k;
  std::map<int, int> shift;   // bit position of each index in `big`
  int sh = 0;
  for (int j = (int)big.inds.size() - 1; j >= 0; --j) { shift[big.inds[j]] = sh; sh += l2[big.inds[j]]; }
  std::stable_sort(k.begin(), k.end(), [&](int a, int b) { return shift.at(a) > shift.at(b); });
  return k;
}

// complex128 tensor-core step reading its raw operands (zgemm_dmma_gather_kernel): offset
// tables of the batch / free / contracted groups of X and Y in their stored layouts, and
// which group holds each operand's stride-1 index (the gather's fast direction)
void set_gather_maps(TcStep& t, TabPool& pool, int X, const NodeLayout& LX, int Y, const NodeLayout& LY,
                     const std::vector<int>& batch, const std::vector<int>& fx, const std::vector<int>& fy,
                     const std::vector<int>& kord, const std::vector<int>& l2) {
  if (t.kind == K_DMMA ? !dmma_gather_enabled() : t.kind == K_WIDE ? !wide_gather_enabled() : !bskinny_ok(t)) return;
  t.gather = true;
  auto& g = t.gmaps;
  g.Ab = pool.add(group_of(batch, LX, l2));
  g.Am = pool.add(group_of(fx, LX, l2));
  g.Ak = pool.add(group_of(kord, LX, l2));
  g.Bb = pool.add(group_of(batch, LY, l2));
  g.Bn = pool.add(group_of(fy, LY, l2));
  g.Bk = pool.add(group_of(kord, LY, l2));
  g.a_node = X;
  g.b_node = Y;
  auto kfast = [&](const NodeLayout& L) {
    return !L.inds.empty() && std::count(kord.begin(), kord.end(), L.inds.back()) > 0;
  };
  g.a_kfast = kfast(LX);
  g.b_kfast = kfast(LY);
}

// decide the path of a step (TC only for complex64 GEMM-shaped steps)
bool want_tc(int dtype, int nb, int m, int n, int k) {
  if (dtype == TN_C128)   // DMMA tiles of 64 x 64 complex, K staged 16 at a time
    return k >= 3 && std::max(m, n) >= 6 && std::min(m, n) >= 5 && (nb + m + n + k) >= 20;
  // N down to 8 (a 64-wide tile, 1/8 used): for such skinny-N steps with a long K the GEMM
  // is bound by reading the big operand once, which the tensor-core path does at HBM speed
  return k >= 4 && std::max(m, n) >= 6 && std::min(m, n) >= 3 && (nb + m + n + k) >= 22;
}
// CUDA-core paths for large non-GEMM-shaped steps (skinny.cu): long contraction with
// few outputs, or short contraction with a large output
bool want_skinny(int nb, int m, int n, int k) {
  // (K >= 64 with many batches: staging each batch's rows through L1 beats the small
  // kernel's per-output re-reads of A and B)
  return (k >= 10 || (k >= 6 && nb >= 6)) && m <= 6 && n <= 6 && m + n <= 8 && nb <= 15 && (nb + m + n + k) >= 20;
}
bool want_wide(int nb, int m, int n, int k) {
  // each planar operand needs >= 8 entries per batch (rows + K bits >= 3, see make_pack)
  return k <= 4 && (nb + m + n) >= 18 && nb <= 24 && (m + k) >= 3 && (n + k) >= 3;
}
void finish_tc_kind(TcStep& t, int dtype) {
  t.kind = dtype == TN_C128 ? K_DMMA : K_TC;
  t.esz = dtype == TN_C128 ? 16 : 8;
  if (t.kind == K_DMMA) {
    t.S = 1; t.BN = tnd::zg::BN; t.k_lo = t.k_bits; t.n_slabs = 1; t.pair = false;
    t.m_lo = t.m_bits; t.n_mslabs = 1;
  }
}
// skinny / wide: K-slabs bound the planar pack buffers; skinny splits each slab's K
// over S CTAs per batch (>= 4 waves of CTAs, >= 4096 K per CTA)
void finish_cuda_core(TcStep& t, int dtype, int kind) {
  t.kind = kind;
  t.m_lo = t.m_bits;
  t.n_mslabs = 1;
  t.esz = dtype == TN_C128 ? 16 : 8;
  t.BN = 0;
  const int over = std::max(t.nb_bits + t.m_bits, t.nb_bits + t.n_bits) + t.k_bits - pack_cap_log2();
  t.k_lo = kind == K_SKINNY ? std::max(std::min(t.k_bits, 6), t.k_bits - std::max(0, over)) : t.k_bits;
  t.n_slabs = 1 << (t.k_bits - t.k_lo);
  if (kind == K_SKINNY) {
    const Sk2Shape h = skinny2_shape(t);
    const int64_t K = int64_t(1) << t.k_lo, want = std::max<int64_t>(1, (148 * 4) >> std::min(t.nb_bits, 20));
    t.S = h.use ? h.S : (int)std::max<int64_t>(1, std::min<int64_t>(want, K / 4096));
  } else {
    t.S = 1;
  }
}
int64_t pack_bytes(const TcStep& t, int rows_bits) {
  if (t.gather) return 16;                       // no pack buffer
  if (t.kind != K_TC) return int64_t(t.esz) << (t.nb_bits + rows_bits + t.k_lo);
  // 4 fp16 planes + one fp32 scale per row and 128-wide K chunk (+ slack: the GEMM's
  // scale copies read whole 128-row / BN-column tiles)
  return (int64_t(8) << (t.nb_bits + rows_bits + t.k_lo)) +
         (int64_t(4) << (t.nb_bits + rows_bits + std::max(t.k_lo - tnd::SCALE_LOG2, 0))) + 1024;
}

// first-fit offsets for (size, [lo, hi]) items
std::vector<int64_t> first_fit(const std::vector<int64_t>& size, const std::vector<std::pair<int, int>>& iv,
                               int64_t& total) {
  size_t n = size.size();
  std::vector<size_t> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return size[a] > size[b]; });
  std::vector<int64_t> off(n, -1);
  std::vector<size_t> placed;
  total = 0;
  for (size_t it : ord) {
    int64_t sz = (size[it] + ALIGN - 1) / ALIGN * ALIGN;
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (size_t p : placed)
      if (!(iv[p].second < iv[it].first || iv[it].second < iv[p].first))
        busy.push_back({off[p], off[p] + (size[p] + ALIGN - 1) / ALIGN * ALIGN});
    std::sort(busy.begin(), busy.end());
    int64_t o = 0;
    for (auto& b : busy) {
      if (o + sz <= b.first) break;
      o = std::max(o, b.second);
    }
    off[it] = o;
    placed.push_back(it);
    total = std::max(total, o + sz);
  }
  return off;
}

}  // namespace

// =============================================================== handles ======
struct tn_network_s {
  tn::Network net;
};
struct tn_order_s {
  tn::Order ord;
  const tn::Network* net;
};

struct tn_plan_s {
  const tn::Network* net = nullptr;
  int dtype = TN_C64, device = 0, esz = 8;
  int n_leaves = 0, n_nodes = 0, root = 0;
  std::vector<int> l2;
  std::vector<Wave> waves;
  std::vector<TcStep> tcs;
  std::vector<std::pair<int, int>> launches;  // (0, wave) | (1, tc)
  // Slice-invariant prologue: launches [0, n_pro) contract the
  // subtrees that hold no sliced index -- the same in every slice of one bitstring -- and
  // run once per bitstring; their outputs that feed per-slice steps (the frontier) stay
  // in the arena while launches [n_pro, end) run once per slice.
  int n_pro = 0;
  double flops_pro = 0;             // Eq. (3) flops of the prologue (part of `flops`)
  int64_t frontier_bytes = 0;
  int64_t kernels_pro = 0;
  cudaGraphExec_t graph_pro = nullptr;
  // profiled graphs of the prologue / a slice (profile_phase), captured on first use
  struct ProfGraph {
    cudaGraphExec_t exec = nullptr;
    Marks mk;
    tn_profile stat{};
    int64_t kernels = 0;
    bool failed = false;
    bool pending = false;           // deferred mode: replayed, its times not read yet
    void reset() {
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
      for (auto& e : mk.v) cudaEventDestroy(e.first);
      mk = Marks();
      stat = tn_profile{};
    }
  };
  ProfGraph prof_graph[2][2];       // [phase][buffer]: two per phase for deferred replays
  bool prof_defer = false;          // tn_profile_defer: profiled calls do not wait
  int prof_buf[2] = {0, 0};         // next buffer per phase (deferred mode)
  tn_profile prof_acc{};            // device times of deferred replays read so far
  bool prepared = false;            // tn_prepare ran and no other contraction call since
  int64_t n_slices = 1;
  int slice_bits = 0;
  double flops = 0, tc_flops = 0;
  int n_small = 0;
  // device
  char* arena = nullptr;
  int64_t arena_bytes = 0;
  char* leaves = nullptr;
  int64_t* tab_d = nullptr;
  void** ptrs_d = nullptr;
  int64_t* leaf_base_d = nullptr;
  int32_t* var_begin_d = nullptr;
  int32_t* var_kind_d = nullptr;
  int64_t* var_stride_d = nullptr;
  int32_t* sl_log2_d = nullptr;
  int32_t* sl_shift_d = nullptr;
  uint8_t* bits_d = nullptr;
  int64_t* slice_d = nullptr;
  double2* amp_d = nullptr;      // complex128 accumulator of one contraction
  int root_exp = 0;              // the root carries 2^-root_exp of leaf scaling
  cudaStream_t cap = nullptr;
  cudaGraphExec_t graph = nullptr;
  int64_t kernels_per_slice = 0;
  std::vector<int32_t> step_table;   // 6 per step: path, nb, m, n, k, launch position
  std::vector<int64_t> node_off;     // arena offset of every intermediate (-1: leaf)
  // Provably zero slices: a leaf whose only sliced index is j and whose other indices are
  // output legs (or open bonds) can vanish entirely for some value v of j given the
  // output bits (e.g. the delta of a CZ bond next to a bound output leg): slices with
  // that digit contribute exactly 0 and are skipped when the bitstring is on the host.
  struct Forced {
    int pos = 0, dim_log2 = 0;
    std::vector<int> qubits;        // output legs of the leaf (their bits select the row)
    std::vector<uint8_t> zero;      // zero[(combo << dim_log2) | v]
  };
  std::vector<Forced> forced;
  std::vector<int32_t> sl_shift_h, sl_log2_h;

  // Extra lanes (tn_plan_set_lanes): independent copies of the per-contraction state --
  // arena, pointer table, bitstring / slice / amplitude slots, tensor maps, stream and
  // graph -- so tn_amplitudes runs several bitstrings concurrently.  Lane 0 is the
  // plan's own state above.
  struct Lane {
    char* arena = nullptr;
    void** ptrs_d = nullptr;
    uint8_t* bits_d = nullptr;
    int64_t* slice_d = nullptr;
    double2* amp_d = nullptr;
    std::vector<TcStep> tcs;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph = nullptr, graph_pro = nullptr;
  };
  std::vector<Lane> extra;

  // record one pass of a phase: 0 = the slice-invariant prologue (launches [0, n_pro)),
  // 1 = one slice (launches [n_pro, end) + the fp64 root accumulation)
  void record_lane(cudaStream_t st, char* arena_l, void** ptrs_l, uint8_t* bits_l, int64_t* slice_l, double2* amp_l,
                   const std::vector<TcStep>& tcs_l, int phase) {
    tnd::set_leaf_ptrs_kernel<<<(n_leaves + 127) / 128, 128, 0, st>>>(
        ptrs_l, leaf_base_d, var_begin_d, var_kind_d, var_stride_d, n_leaves, bits_l, slice_l, sl_log2_d, sl_shift_d,
        esz, leaves);
    int64_t k = 1;
    const size_t l0 = phase == 0 ? 0 : (size_t)n_pro, l1 = phase == 0 ? (size_t)n_pro : launches.size();
    for (size_t li = l0; li < l1; ++li) {
      const auto& L = launches[li];
      if (L.first == 0) {
        if (dtype == TN_C64) launch_wave<float>(waves[L.second], ptrs_l, tab_d, st);
        else launch_wave<double>(waves[L.second], ptrs_l, tab_d, st);
        k += 1;
      } else {
        launch_tc(tcs_l[L.second], arena_l, ptrs_l, tab_d, st);
        const auto& t = tcs_l[L.second];
        k += t.kind == K_DMMA ? (t.gather ? dmma_launches(t) : 3) : t.kind == K_SKINNY ? (t.gather ? (bskinny_s_bits(t) > 0 ? 2 : 1) : (t.S * skinny_ws(t) == 1 ? 3 : 4) * t.n_slabs) : t.kind == K_WIDE ? (t.gather ? 1 : 3) * t.n_slabs
             : t.n_mslabs * t.n_slabs * (t.S > 1 ? 3 : 2) + (t.n_mslabs > 1 ? 1 : t.n_slabs);
      }
    }
    if (phase == 0) {
      CK(cudaGetLastError());
      kernels_pro = k;
      return;
    }
    if (dtype == TN_C64) tnd::accumulate_root_kernel<float><<<1, 1, 0, st>>>(ptrs_l, root, root_exp, amp_l, slice_l);
    else tnd::accumulate_root_kernel<double><<<1, 1, 0, st>>>(ptrs_l, root, root_exp, amp_l, slice_l);
    CK(cudaGetLastError());
    kernels_per_slice = k + 1;
  }
  // capture a phase as a CUDA graph on stream st
  cudaGraphExec_t capture(cudaStream_t st, char* arena_l, void** ptrs_l, uint8_t* bits_l, int64_t* slice_l,
                          double2* amp_l, const std::vector<TcStep>& tcs_l, int phase) {
    cudaGraph_t g;
    cudaGraphExec_t e;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const int64_t before = g_launches.load();
    record_lane(st, arena_l, ptrs_l, bits_l, slice_l, amp_l, tcs_l, phase);
    g_launches = before;  // captured launches are counted when replayed
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&e, g, 0));
    CK(cudaGraphDestroy(g));
    return e;
  }

  ~tn_plan_s() {
    for (auto& l : extra) {
      if (l.graph) cudaGraphExecDestroy(l.graph);
      if (l.graph_pro) cudaGraphExecDestroy(l.graph_pro);
      if (l.stream) cudaStreamDestroy(l.stream);
      for (void* p : {(void*)l.arena, (void*)l.ptrs_d, (void*)l.bits_d, (void*)l.slice_d, (void*)l.amp_d})
        if (p) cudaFree(p);
    }
    if (graph) cudaGraphExecDestroy(graph);
    if (graph_pro) cudaGraphExecDestroy(graph_pro);
    for (auto& ph : prof_graph)
      for (auto& g : ph) g.reset();
    if (cap) cudaStreamDestroy(cap);
    for (auto& w : waves) { cudaFree(w.steps_d); cudaFree(w.prefix_d); if (w.cta_step_d) cudaFree(w.cta_step_d); }
    for (void* p : {(void*)arena, (void*)leaves, (void*)tab_d, (void*)ptrs_d, (void*)leaf_base_d, (void*)var_begin_d,
                    (void*)var_kind_d, (void*)var_stride_d, (void*)sl_log2_d, (void*)sl_shift_d, (void*)bits_d,
                    (void*)slice_d, (void*)amp_d})
      if (p) cudaFree(p);
  }
};

namespace {

__global__ void set_i64_kernel(int64_t* p, int64_t v) { *p = v; }
__global__ void add_amp_kernel(double2* dst, const double2* src) {
  dst->x += src->x;
  dst->y += src->y;
}

template <typename T>
T* upload(const std::vector<T>& v) {
  T* p = nullptr;
  size_t n = std::max<size_t>(v.size(), 1);
  CK(cudaMalloc(&p, n * sizeof(T)));
  if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

void check_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0)
    throw Err(TN_ECUDA, "no CUDA device " + std::to_string(device));
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, device));
  if (p.major != 10) throw Err(TN_ECUDA, std::string("sm_100 device required, found ") + p.name);
  CK(cudaSetDevice(device));
}

void build_plan(tn_plan_s& P, const tn::Network& net, const tn::Order& ord, bool allow_reuse) {
  P.net = &net;
  P.esz = P.dtype == TN_C64 ? 8 : 16;
  const int n = (int)net.tensors.size();
  P.n_leaves = n;
  P.n_nodes = n + (int)ord.steps.size();
  P.root = P.n_nodes - 1;
  P.l2.resize(net.dims.size());
  for (size_t i = 0; i < net.dims.size(); ++i) P.l2[i] = net.log2dim((int)i);
  const auto& l2 = P.l2;
  std::set<int> sliced(ord.slices.begin(), ord.slices.end());
  std::map<int, int> slice_pos;
  for (size_t j = 0; j < ord.slices.size(); ++j) slice_pos[ord.slices[j]] = (int)j;
  std::map<int, int> out_q;
  for (int q = 0; q < net.n_qubits; ++q) out_q[net.out_leg[q]] = q;

  // ---- leaves: vars (output legs, sliced indices) first ----
  std::vector<NodeLayout> L(P.n_nodes);
  std::vector<int64_t> leaf_base(n), var_stride;
  std::vector<int32_t> var_begin(n + 1, 0), var_kind;
  std::vector<char> leaf_host;
  int64_t leaf_elems = 0;
  // Leaf scaling: binding an output leg or fixing a sliced index
  // bit shrinks the contraction by ~2^-1/2, so a sliced amplitude of many qubits
  // leaves the complex64 exponent range (config 4 slices reach 2^-165).  Leaf t is
  // scaled by 2^c_t, c_t the integer steps of a running sum of half a bit per bound
  // leg / sliced bit it holds; the root is multiplied by 2^-sum c_t in fp64.
  int half_bits = 0, scale_exp = 0;
  for (int t = 0; t < n; ++t) {
    const auto& T = net.tensors[t];
    std::vector<int> vars, rest;
    for (int i : T.inds) (out_q.count(i) || sliced.count(i) ? vars : rest).push_back(i);
    int bound = 0;
    for (int i : vars) bound += out_q.count(i) ? 1 : l2[i];
    const int c_t = (half_bits + bound) / 2 - half_bits / 2;
    half_bits += bound;
    scale_exp += c_t;
    const double leaf_scale = std::ldexp(1.0, c_t);
    L[t].inds = rest;
    L[t].bits = sum_bits(rest, l2);
    std::vector<int> ninds = vars;
    ninds.insert(ninds.end(), rest.begin(), rest.end());
    // strides of the original (canonical) layout
    std::vector<int64_t> st(T.inds.size());
    int64_t acc = 1;
    for (int k = (int)T.inds.size() - 1; k >= 0; --k) { st[k] = acc; acc *= net.dims[T.inds[k]]; }
    leaf_base[t] = leaf_elems;
    var_begin[t] = (int32_t)var_kind.size();
    int64_t vs = int64_t(1) << L[t].bits;
    std::vector<int64_t> vstr(vars.size());
    for (int k = (int)vars.size() - 1; k >= 0; --k) { vstr[k] = vs; vs <<= l2[vars[k]]; }
    for (size_t k = 0; k < vars.size(); ++k) {
      var_kind.push_back(out_q.count(vars[k]) ? out_q[vars[k]] : -1 - slice_pos[vars[k]]);
      var_stride.push_back(vstr[k]);
    }
    var_begin[t + 1] = (int32_t)var_kind.size();
    // permuted data
    size_t off = leaf_host.size();
    leaf_host.resize(off + (size_t)acc * P.esz);
    std::vector<int> dig(ninds.size());
    for (int64_t it = 0; it < acc; ++it) {
      int64_t r = it;
      for (int k = (int)ninds.size() - 1; k >= 0; --k) { dig[k] = (int)(r % net.dims[ninds[k]]); r /= net.dims[ninds[k]]; }
      int64_t src = 0;
      for (size_t k = 0; k < ninds.size(); ++k) {
        size_t pos = std::find(T.inds.begin(), T.inds.end(), ninds[k]) - T.inds.begin();
        src += st[pos] * dig[k];
      }
      const tn::cplx z = T.data[src] * leaf_scale;
      if (P.dtype == TN_C64) {
        float v[2] = {(float)z.real(), (float)z.imag()};
        std::memcpy(&leaf_host[off + it * 8], v, 8);
      } else {
        double v[2] = {z.real(), z.imag()};
        std::memcpy(&leaf_host[off + it * 16], v, 16);
      }
    }
    leaf_elems += acc;
    // keep leaf bases 128-byte aligned
    int64_t pad = (16 - (leaf_elems % 16)) % 16;
    leaf_elems += pad;
    leaf_host.resize((size_t)leaf_elems * P.esz, 0);
  }

  P.root_exp = -scale_exp;

  // ---- steps ----
  auto kept_all = tn::kept_per_step(net, ord.steps);
  std::vector<int> parent(P.n_nodes, -1);
  std::vector<int> kind(ord.steps.size(), 0), big_index(ord.steps.size(), -1);
  TabPool pool;
  std::vector<SmallStep> small_desc(ord.steps.size());
  for (size_t k = 0; k < ord.steps.size(); ++k) {
    int a = ord.steps[k].first, b = ord.steps[k].second, c = n + (int)k;
    parent[a] = parent[b] = (int)k;
    std::set<int> kept;
    for (int i : kept_all[k]) if (!sliced.count(i)) kept.insert(i);
    Classes cl = classify(L[a], L[b], kept);
    int nb = sum_bits(cl.batch, l2), ml = sum_bits(cl.lfree, l2), mr = sum_bits(cl.rfree, l2), kk = sum_bits(cl.contr, l2);
    P.flops += 8.0 * std::ldexp(1.0, nb + ml + mr + kk);
    const int big = want_tc(P.dtype, nb, ml, mr, kk) ? (P.dtype == TN_C128 ? K_DMMA : K_TC)
                    : want_skinny(nb, ml, mr, kk)  ? K_SKINNY
                    : want_wide(nb, ml, mr, kk)    ? K_WIDE
                                                   : -1;
    if (big >= 0) {
      // tensor cores: X = operand with the larger free group becomes the MMA's M side;
      // wide: the larger free group becomes C's contiguous (column) side
      bool swap = big == K_WIDE ? ml > mr : mr > ml;
      int X = swap ? b : a, Y = swap ? a : b;
      std::vector<int> fx = swap ? cl.rfree : cl.lfree;
      const auto& fy = swap ? cl.lfree : cl.rfree;
      TcStep t;
      t.nb_bits = nb; t.m_bits = sum_bits(fx, l2); t.n_bits = sum_bits(fy, l2); t.k_bits = kk;
      t.c_node = c;
      if (big == K_TC || big == K_DMMA) {
        finish_tc_shape(t);
        finish_tc_kind(t, P.dtype);
      } else {
        finish_cuda_core(t, P.dtype, big);
      }
      const int planes = t.kind == K_TC ? 4 : 2;
      const std::vector<int> kord = slab_k_order(cl.contr, L[X].bits >= L[Y].bits ? L[X] : L[Y], l2, t.n_slabs);
      // row slabs: X's largest-stride free indices first (the slab bits), in C's layout too
      fx = slab_k_order(fx, L[X], l2, t.n_mslabs);
      t.px = make_pack(pool, X, L[X], cl.batch, fx, kord, l2, planes, t.k_lo, &t.slab_x, t.m_lo);
      t.py = make_pack(pool, Y, L[Y], cl.batch, fy, kord, l2, planes, t.k_lo, &t.slab_y);
      set_gather_maps(t, pool, X, L[X], Y, L[Y], cl.batch, fx, fy, kord, l2);   // DMMA / wide
      t.flops = 8.0 * std::ldexp(1.0, nb + ml + mr + kk);
      if (t.kind == K_TC || t.kind == K_DMMA) P.tc_flops += t.flops;
      L[c].inds = cl.batch;
      L[c].inds.insert(L[c].inds.end(), fx.begin(), fx.end());
      L[c].inds.insert(L[c].inds.end(), fy.begin(), fy.end());
      kind[k] = 1;
      big_index[k] = (int)P.tcs.size();
      P.tcs.push_back(t);
    } else {
      SmallStep d{};
      d.a = a; d.b = b; d.c = c;
      d.nb_bits = nb; d.m_bits = ml; d.n_bits = mr; d.k_bits = kk;
      d.Ab = pool.add(group_of(cl.batch, L[a], l2));
      d.Am = pool.add(group_of(cl.lfree, L[a], l2));
      d.Ak = pool.add(group_of(cl.contr, L[a], l2));
      d.Bb = pool.add(group_of(cl.batch, L[b], l2));
      d.Bk = pool.add(group_of(cl.contr, L[b], l2));
      d.Bn = pool.add(group_of(cl.rfree, L[b], l2));
      set_small_mode(d);
      small_desc[k] = d;
      L[c].inds = cl.batch;
      L[c].inds.insert(L[c].inds.end(), cl.lfree.begin(), cl.lfree.end());
      L[c].inds.insert(L[c].inds.end(), cl.rfree.begin(), cl.rfree.end());
      P.n_small++;
    }
    L[c].bits = sum_bits(L[c].inds, l2);
  }

  P.step_table.assign(6 * ord.steps.size(), 0);
  for (size_t k = 0; k < ord.steps.size(); ++k) {
    int32_t* e = &P.step_table[6 * k];
    if (kind[k]) {
      const auto& t = P.tcs[big_index[k]];
      e[0] = t.kind == K_SKINNY ? TN_PATH_SKINNY : t.kind == K_WIDE ? TN_PATH_WIDE : TN_PATH_TC; e[1] = t.nb_bits; e[2] = t.m_bits; e[3] = t.n_bits; e[4] = t.k_bits;
    } else {
      const auto& d = small_desc[k];
      e[0] = TN_PATH_SMALL; e[1] = d.nb_bits; e[2] = d.m_bits; e[3] = d.n_bits; e[4] = d.k_bits;
    }
  }
  // ---- slice-invariant prologue ----
  // A node is slice-invariant when no leaf below it holds a sliced index: it is the same
  // in every slice of a bitstring.  Phase 0 = those steps (once per bitstring), phase 1 =
  // the rest (once per slice).  TN_SLICE_REUSE=0 puts every step in phase 1.
  static const bool reuse_on = [] {
    const char* e = std::getenv("TN_SLICE_REUSE");
    return !(e && e[0] == '0');
  }();
  std::vector<char> inv(P.n_nodes, 0);
  for (int t = 0; t < n; ++t) {
    inv[t] = 1;
    for (int i : net.tensors[t].inds) if (sliced.count(i)) inv[t] = 0;
  }
  std::vector<int> phase(ord.steps.size(), 1);
  double inv_flops = 0;
  for (size_t k = 0; k < ord.steps.size(); ++k) {
    inv[n + k] = inv[ord.steps[k].first] && inv[ord.steps[k].second];
    if (inv[n + k])
      inv_flops += kind[k] ? P.tcs[big_index[k]].flops
                           : 8.0 * std::ldexp(1.0, small_desc[k].nb_bits + small_desc[k].m_bits +
                                                       small_desc[k].n_bits + small_desc[k].k_bits);
  }
  // the frontier costs arena memory: reuse only when it saves >= 2% of a slice's work
  const bool reuse = reuse_on && allow_reuse && !sliced.empty() && inv_flops >= 0.02 * P.flops;
  for (size_t k = 0; k < ord.steps.size(); ++k)
    if (reuse && inv[n + k]) phase[k] = 0;
  // big steps in launch order: phase 0 first, each phase in step order (topological)
  {
    std::vector<int> order_k;
    for (int ph = 0; ph < 2; ++ph)
      for (size_t k = 0; k < ord.steps.size(); ++k)
        if (kind[k] && phase[k] == ph) order_k.push_back((int)k);
    std::vector<TcStep> tcs2;
    for (int k : order_k) {
      tcs2.push_back(P.tcs[big_index[k]]);
      big_index[k] = (int)tcs2.size() - 1;
    }
    P.tcs = std::move(tcs2);
  }
  int n_big0 = 0;
  for (size_t k = 0; k < ord.steps.size(); ++k) if (kind[k] && phase[k] == 0) ++n_big0;
  // ---- schedule: small steps in waves between tensor-core steps ----
  // slot s of a small step: it runs after big step s - 1 (launch order); per phase, the
  // small steps of one slot go in waves by dependency depth
  std::vector<int> slot(ord.steps.size(), 0), depth(ord.steps.size(), 0);
  int n_big = (int)P.tcs.size();
  std::vector<std::map<int, std::vector<int>>> slot_waves[2];
  slot_waves[0].resize(n_big + 1);
  slot_waves[1].resize(n_big + 1);
  for (size_t k = 0; k < ord.steps.size(); ++k) {
    if (kind[k]) continue;
    int s = phase[k] == 1 ? n_big0 : 0;
    for (int ch : {ord.steps[k].first, ord.steps[k].second}) {
      if (ch < n) continue;
      int ck = ch - n;
      s = std::max(s, kind[ck] ? big_index[ck] + 1 : slot[ck]);
    }
    int d = 1;
    for (int ch : {ord.steps[k].first, ord.steps[k].second}) {
      if (ch < n) continue;
      int ck = ch - n;
      if (!kind[ck] && slot[ck] == s && phase[ck] == phase[k]) d = std::max(d, depth[ck] + 1);
    }
    slot[k] = s;
    depth[k] = d;
    slot_waves[phase[k]][s][d].push_back((int)k);
  }
  std::vector<int> step_pos(ord.steps.size(), 0);
  for (int ph = 0; ph < 2; ++ph) {
    if (ph == 1) P.n_pro = (int)P.launches.size();
    const int s_lo = ph == 0 ? 0 : n_big0, s_hi = ph == 0 ? n_big0 : n_big;
    for (int s = s_lo; s <= s_hi; ++s) {
      for (auto& kv : slot_waves[ph][s]) {
        Wave w;
        int64_t acc = 0;
        for (int k : kv.second) {
          w.prefix.push_back(acc);
          const auto& d = small_desc[k];
          int64_t outs = int64_t(1) << (d.nb_bits + d.m_bits + d.n_bits);
          acc += (outs + d.opc - 1) / d.opc;
          w.steps.push_back(d);
          w.flops += 8.0 * std::ldexp(1.0, d.nb_bits + d.m_bits + d.n_bits + d.k_bits);
          w.bytes += P.esz * (std::ldexp(1.0, L[d.a].bits) + std::ldexp(1.0, L[d.b].bits) + std::ldexp(1.0, L[d.c].bits));
          step_pos[k] = (int)P.launches.size();
        }
        w.prefix.push_back(acc);
        w.n_cta = acc;
        P.launches.push_back({0, (int)P.waves.size()});
        P.waves.push_back(std::move(w));
      }
      if (s < s_hi) {
        for (size_t k = 0; k < ord.steps.size(); ++k)
          if (kind[k] && big_index[k] == s) step_pos[k] = (int)P.launches.size();
        P.launches.push_back({1, s});
      }
    }
  }
  for (size_t k = 0; k < ord.steps.size(); ++k) {
    if (phase[k] != 0) continue;
    P.flops_pro += kind[k] ? P.tcs[big_index[k]].flops
                           : 8.0 * std::ldexp(1.0, small_desc[k].nb_bits + small_desc[k].m_bits +
                                                       small_desc[k].n_bits + small_desc[k].k_bits);
  }

  for (size_t k = 0; k < ord.steps.size(); ++k) P.step_table[6 * k + 5] = step_pos[k];
  // ---- arena: intermediates + pack buffers, first fit over live intervals ----
  // Every launch position L has two phases: 2L (tensor-core packs read the raw operands)
  // and 2L+1 (GEMM / small wave).  A tensor-core step's raw operands die after its pack
  // phase, its pack buffers live through both phases, its output is born at 2L+1.
  std::vector<int64_t> sizes;
  std::vector<std::pair<int, int>> ivs;
  std::vector<int> owner;  // >=0: node id; -1 - 2*tc: pack X; -2 - 2*tc: pack Y; <= -1000000: partials
  const int last = 2 * (int)P.launches.size() + 2;
  for (size_t k = 0; k < ord.steps.size(); ++k) {
    int c = n + (int)k;
    int born = 2 * step_pos[k] + 1;
    int hi = last;
    if (parent[c] >= 0) {
      // a big step's operands die after its pack phase -- unless it packs in slabs: then
      // slab s + 1 is packed after the GEMM of slab s wrote C, so they live through it
      const int pk = parent[c];
      bool slabbed = false;
      if (kind[pk]) {
        const auto& pt = P.tcs[big_index[pk]];
        // (a gathering DMMA step reads its raw operands in its GEMM phase too)
        slabbed = pt.n_slabs > 1 || pt.n_mslabs > 1 || pt.gather;
      }
      hi = 2 * step_pos[pk] + ((kind[pk] && !slabbed) ? 0 : 1);
      // the frontier of the prologue stays while the slices run
      if (phase[k] == 0 && phase[pk] == 1) {
        hi = last;
        P.frontier_bytes += (int64_t(1) << L[c].bits) * P.esz;
      }
    }
    sizes.push_back((int64_t(1) << L[c].bits) * P.esz);
    ivs.push_back({born, hi});
    owner.push_back(c);
  }
  for (size_t k = 0; k < ord.steps.size(); ++k) {
    if (!kind[k]) continue;
    const auto& t = P.tcs[big_index[k]];
    const int p0 = 2 * step_pos[k];
    sizes.push_back(pack_bytes(t, t.m_lo));
    ivs.push_back({p0, p0 + 1});
    owner.push_back(-1 - 2 * big_index[k]);
    sizes.push_back(pack_bytes(t, t.n_bits));
    ivs.push_back({p0, p0 + 1});
    owner.push_back(-2 - 2 * big_index[k]);
    if (tc_partial_bytes(t) > 0) {
      sizes.push_back(tc_partial_bytes(t));
      ivs.push_back({p0 + 1, p0 + 1});
      owner.push_back(-1000000 - big_index[k]);
    }
  }
  int64_t total = 0;
  auto offs = first_fit(sizes, ivs, total);
  P.arena_bytes = std::max<int64_t>(total, ALIGN);
  size_t free_b = 0, tot_b = 0;
  CK(cudaMemGetInfo(&free_b, &tot_b));
  if ((size_t)P.arena_bytes + (size_t)(leaf_host.size() + pool.v.size() * 8) + (size_t(1) << 30) > free_b)
    throw Err(TN_ENOMEM, "arena of " + std::to_string(P.arena_bytes) + " bytes does not fit free device memory " +
                             std::to_string(free_b));
  CK(cudaMalloc(&P.arena, P.arena_bytes));
  std::vector<void*> ptrs(P.n_nodes, nullptr);
  P.node_off.assign(P.n_nodes, -1);
  for (size_t j = 0; j < owner.size(); ++j) {
    if (owner[j] >= 0) { ptrs[owner[j]] = P.arena + offs[j]; P.node_off[owner[j]] = offs[j]; }
    else if (owner[j] <= -1000000) P.tcs[-1000000 - owner[j]].p_off = offs[j];
    else {
      int o = -1 - owner[j];
      if (o % 2 == 0) P.tcs[o / 2].x_off = offs[j];
      else P.tcs[o / 2].y_off = offs[j];
    }
  }
  for (auto& t : P.tcs) {
    set_skinny_maps(t, P.arena);
    if (t.kind != K_TC) continue;
    t.ta = make_plane_map(P.arena + t.x_off, t.k_lo, t.m_lo, t.nb_bits, 128, 4);
    t.tb = make_plane_map(P.arena + t.y_off, t.k_lo, t.n_bits, t.nb_bits, t.pair ? tnd::tc::Cfg2::BNH : t.BN, 4);
    if (t.pair)
      t.tc = make_c_map(P.arena + P.node_off[t.c_node], t.n_bits, int64_t(1) << (t.nb_bits + t.m_bits));
  }

  // ---- uploads ----
  P.leaves = upload(leaf_host);
  P.tab_d = upload(pool.v);
  P.ptrs_d = upload(ptrs);
  P.leaf_base_d = upload(leaf_base);
  P.var_begin_d = upload(var_begin);
  P.var_kind_d = upload(var_kind);
  P.var_stride_d = upload(var_stride);
  std::vector<int32_t> sl_log2, sl_shift(ord.slices.size());
  int sh = 0;
  for (int j = (int)ord.slices.size() - 1; j >= 0; --j) { sl_shift[j] = sh; sh += l2[ord.slices[j]]; }
  for (int i : ord.slices) sl_log2.push_back(l2[i]);
  P.slice_bits = sh;
  P.n_slices = sh >= 63 ? INT64_MAX : int64_t(1) << sh;
  P.sl_shift_h = sl_shift;
  P.sl_log2_h = sl_log2;
  for (int t = 0; t < n; ++t) {
    const auto& T = net.tensors[t];
    int only = -1, cnt = 0;
    for (int i : T.inds) if (sliced.count(i)) { only = i; ++cnt; }
    if (cnt != 1) continue;
    tn_plan_s::Forced f;
    f.pos = slice_pos[only];
    f.dim_log2 = l2[only];
    std::vector<int> oax;                 // axes of the output legs
    for (size_t a = 0; a < T.inds.size(); ++a)
      if (out_q.count(T.inds[a])) { oax.push_back((int)a); f.qubits.push_back(out_q[T.inds[a]]); }
    const int sax = (int)(std::find(T.inds.begin(), T.inds.end(), only) - T.inds.begin());
    f.zero.assign(size_t(1) << (f.qubits.size() + f.dim_log2), 1);
    std::vector<int64_t> st(T.inds.size());
    int64_t acc = 1;
    for (int k = (int)T.inds.size() - 1; k >= 0; --k) { st[k] = acc; acc *= net.dims[T.inds[k]]; }
    for (int64_t e = 0; e < acc; ++e) {
      if (T.data[e] == tn::cplx(0, 0)) continue;
      size_t combo = 0;
      for (size_t q = 0; q < oax.size(); ++q) combo = (combo << 1) | size_t((e / st[oax[q]]) % net.dims[T.inds[oax[q]]] & 1);
      const int v = (int)((e / st[sax]) % net.dims[only]);
      f.zero[(combo << f.dim_log2) | v] = 0;
    }
    bool any = false;
    for (uint8_t z : f.zero) any |= z != 0;
    if (any) P.forced.push_back(std::move(f));
  }
  P.sl_log2_d = upload(sl_log2);
  P.sl_shift_d = upload(sl_shift);
  CK(cudaMalloc(&P.bits_d, std::max(1, net.n_qubits)));
  CK(cudaMemset(P.bits_d, 0, std::max(1, net.n_qubits)));
  CK(cudaMalloc(&P.slice_d, sizeof(int64_t)));
  CK(cudaMemset(P.slice_d, 0, sizeof(int64_t)));
  CK(cudaMalloc(&P.amp_d, 16));
  CK(cudaMemset(P.amp_d, 0, 16));
  for (auto& w : P.waves) {
    w.steps_d = upload(w.steps);
    w.prefix_d = upload(w.prefix);
    if (w.n_cta <= (int64_t(1) << 22)) {
      std::vector<int32_t> cs((size_t)w.n_cta);
      for (size_t q = 0; q < w.steps.size(); ++q)
        for (int64_t b = w.prefix[q]; b < w.prefix[q + 1]; ++b) cs[(size_t)b] = (int32_t)q;
      w.cta_step_d = upload(cs);
    }
  }
  if (n == 1 && ord.steps.empty()) P.root = 0;
  // ---- capture the prologue and one slice as CUDA graphs ----
  ensure_gemm_attr<128>();
  ensure_gemm_attr<64>();
  CK(cudaStreamCreateWithFlags(&P.cap, cudaStreamNonBlocking));
  if (P.n_pro > 0) P.graph_pro = P.capture(P.cap, P.arena, P.ptrs_d, P.bits_d, P.slice_d, P.amp_d, P.tcs, 0);
  P.graph = P.capture(P.cap, P.arena, P.ptrs_d, P.bits_d, P.slice_d, P.amp_d, P.tcs, 1);
}

// one more lane of per-contraction state (see tn_plan_s::Lane)
void add_lane(tn_plan_s& P) {
  size_t free_b = 0, tot_b = 0;
  CK(cudaMemGetInfo(&free_b, &tot_b));
  if ((size_t)P.arena_bytes + (size_t(1) << 30) > free_b)
    throw Err(TN_ENOMEM, "lane arena of " + std::to_string(P.arena_bytes) + " bytes does not fit free device memory");
  tn_plan_s::Lane l;
  CK(cudaMalloc(&l.arena, P.arena_bytes));
  std::vector<void*> ptrs(P.n_nodes, nullptr);
  for (int i = 0; i < P.n_nodes; ++i)
    if (P.node_off[i] >= 0) ptrs[i] = l.arena + P.node_off[i];
  l.ptrs_d = upload(ptrs);
  CK(cudaMalloc(&l.bits_d, std::max(1, P.net->n_qubits)));
  CK(cudaMemset(l.bits_d, 0, std::max(1, P.net->n_qubits)));
  CK(cudaMalloc(&l.slice_d, sizeof(int64_t)));
  CK(cudaMemset(l.slice_d, 0, sizeof(int64_t)));
  CK(cudaMalloc(&l.amp_d, 16));
  CK(cudaMemset(l.amp_d, 0, 16));
  l.tcs = P.tcs;
  for (auto& t : l.tcs) {
    set_skinny_maps(t, l.arena);
    if (t.kind != K_TC) continue;
    t.ta = make_plane_map(l.arena + t.x_off, t.k_lo, t.m_lo, t.nb_bits, 128, 4);
    t.tb = make_plane_map(l.arena + t.y_off, t.k_lo, t.n_bits, t.nb_bits, t.pair ? tnd::tc::Cfg2::BNH : t.BN, 4);
    if (t.pair)
      t.tc = make_c_map(l.arena + P.node_off[t.c_node], t.n_bits, int64_t(1) << (t.nb_bits + t.m_bits));
  }
  CK(cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking));
  if (P.n_pro > 0) l.graph_pro = P.capture(l.stream, l.arena, l.ptrs_d, l.bits_d, l.slice_d, l.amp_d, l.tcs, 0);
  l.graph = P.capture(l.stream, l.arena, l.ptrs_d, l.bits_d, l.slice_d, l.amp_d, l.tcs, 1);
  P.extra.push_back(std::move(l));
}

// one phase (0: prologue, 1: the slice at *slice_d) issued on `st` with CUDA event marks
// around every kernel class; its algorithmic flops / bytes and counts are ADDED to stat
void record_profiled(tn_plan_s& P, int phase, cudaStream_t st, Marks& mk, tn_profile& stat) {
  mk.mark(st, 4, TN_K_OTHER);
  tnd::set_leaf_ptrs_kernel<<<(P.n_leaves + 127) / 128, 128, 0, st>>>(
      P.ptrs_d, P.leaf_base_d, P.var_begin_d, P.var_kind_d, P.var_stride_d, P.n_leaves, P.bits_d, P.slice_d,
      P.sl_log2_d, P.sl_shift_d, P.esz, P.leaves);
  g_launches++;
  stat.n_other++;
  const size_t l0 = phase == 0 ? 0 : (size_t)P.n_pro, l1 = phase == 0 ? (size_t)P.n_pro : P.launches.size();
  for (size_t li = l0; li < l1; ++li) {
    const auto& L = P.launches[li];
    if (L.first == 0) {
      {
        const auto& w = P.waves[L.second];
        size_t big = 0;
        for (size_t q = 1; q < w.steps.size(); ++q) {
          const auto &x = w.steps[q], &y = w.steps[big];
          if (x.nb_bits + x.m_bits + x.n_bits + x.k_bits > y.nb_bits + y.m_bits + y.n_bits + y.k_bits) big = q;
        }
        const auto& d = w.steps[big];
        mk.mark(st, 0, TN_K_SMALL, profile_dump_ms() >= 0 ? shape_tag(("wave of " + std::to_string(w.steps.size()) + ", largest").c_str(),
                                                         d.nb_bits, d.m_bits, d.n_bits, d.k_bits) : "");
      }
      if (P.dtype == TN_C64) launch_wave<float>(P.waves[L.second], P.ptrs_d, P.tab_d, st);
      else launch_wave<double>(P.waves[L.second], P.ptrs_d, P.tab_d, st);
      stat.n_small++;
      stat.flops_small += P.waves[L.second].flops;
      stat.bytes_small += P.waves[L.second].bytes;
      stat.k_flops[TN_K_SMALL] += P.waves[L.second].flops;
      stat.k_bytes[TN_K_SMALL] += P.waves[L.second].bytes;
    } else {
      const auto& t = P.tcs[L.second];
      launch_tc(t, P.arena, P.ptrs_d, P.tab_d, st, &mk);
      const double ex = std::ldexp(1.0, t.nb_bits + t.m_bits + t.k_bits), ey = std::ldexp(1.0, t.nb_bits + t.n_bits + t.k_bits);
      stat.n_pack += 2 * t.n_slabs;
      // algorithmic bytes: a planar pack reads and writes every entry once (2 esz per
      // entry); the fp16x2 pack reads 8 and writes 8 bytes per entry plus one fp32
      // scale per 128-entry K chunk; skinny / wide read both planar operands and write C
      if (t.kind == K_SKINNY || t.kind == K_WIDE) {   // CUDA-core: accounted with the small path
        const double b = t.esz * (ex + ey + std::ldexp(1.0, t.nb_bits + t.m_bits + t.n_bits));
        stat.n_small += t.n_slabs;
        stat.flops_small += t.flops;
        stat.bytes_small += b;
        if (!t.gather) stat.bytes_pack += 2.0 * t.esz * (ex + ey);
        const int kc = t.kind == K_SKINNY ? TN_K_SKINNY : TN_K_WIDE;
        stat.k_flops[kc] += t.flops;
        stat.k_bytes[kc] += b;
        if (!t.gather) stat.k_bytes[TN_K_PACK_PLANAR] += 2.0 * t.esz * (ex + ey);
      } else {
        const double pb = t.gather ? 0.0 : (t.kind == K_DMMA ? 32.0 : 16.0 + 4.0 / 128.0) * (ex + ey);
        stat.n_gemm += t.n_slabs * t.n_mslabs;
        stat.n_pack += t.n_mslabs - 1;
        stat.flops_gemm += t.flops;
        stat.bytes_pack += pb;
        stat.k_flops[t.kind == K_DMMA ? TN_K_DMMA : gemm_class(t)] += t.flops;
        stat.k_bytes[t.kind == K_DMMA ? TN_K_PACK_PLANAR : TN_K_PACK_TC] += pb;
      }
    }
  }
  if (phase == 1) {
    mk.mark(st, 4, TN_K_OTHER);
    if (P.dtype == TN_C64) tnd::accumulate_root_kernel<float><<<1, 1, 0, st>>>(P.ptrs_d, P.root, P.root_exp, P.amp_d, P.slice_d);
    else tnd::accumulate_root_kernel<double><<<1, 1, 0, st>>>(P.ptrs_d, P.root, P.root_exp, P.amp_d, P.slice_d);
    g_launches++;
    stat.n_other++;
  }
  mk.mark(st, -1, TN_K_OTHER);
}

// device times between consecutive marks (all recorded), ADDED to pr
void read_marks(const Marks& mk, tn_profile& pr) {
  for (size_t j = 0; j + 1 < mk.v.size(); ++j) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, mk.v[j].first, mk.v[j + 1].first));
    if (profile_dump_ms() >= 0 && ms > profile_dump_ms())
      fprintf(stderr, "[tn profile] %8.3f ms  cat %d  %s\n", ms, mk.v[j].second, mk.tags[j].c_str());
    if (mk.fine[j] >= 0 && mk.fine[j] < TN_K_COUNT) {
      pr.k_ms[mk.fine[j]] += ms;
      pr.k_intervals[mk.fine[j]]++;
    }
    switch (mk.v[j].second) {
      case 0: pr.ms_small += ms; break;
      case 1: pr.ms_pack += ms; break;
      case 2: pr.ms_gemm += ms; break;
      case 3: pr.ms_other += ms; break;     // split-K reduction
      default: pr.ms_other += ms; break;
    }
  }
}

void add_profile(tn_profile& a, const tn_profile& b) {
  a.ms_small += b.ms_small; a.ms_pack += b.ms_pack; a.ms_gemm += b.ms_gemm; a.ms_other += b.ms_other;
  a.flops_gemm += b.flops_gemm; a.flops_small += b.flops_small;
  a.bytes_small += b.bytes_small; a.bytes_pack += b.bytes_pack;
  a.n_gemm += b.n_gemm; a.n_pack += b.n_pack; a.n_small += b.n_small; a.n_other += b.n_other;
  for (int k = 0; k < 16; ++k) {
    a.k_ms[k] += b.k_ms[k]; a.k_flops[k] += b.k_flops[k]; a.k_bytes[k] += b.k_bytes[k];
    a.k_intervals[k] += b.k_intervals[k];
  }
}

// TN_PROFILE_GRAPH=0: profiled calls launch eagerly instead of replaying the profiled graphs
bool profile_graph_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TN_PROFILE_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

// one profiled phase, timings ADDED to pr: by default a replay of the phase's profiled CUDA
// graph -- the same launches as the plan's graph with event records between the kernel
// classes, captured once per plan -- so the timed launches have the production path's
// (graph) launch gaps; eagerly (launch by launch) with TN_PROFILE_GRAPH=0 or if the capture
// failed
void profile_phase(tn_plan_s& P, int phase, cudaStream_t st, tn_profile& pr) {
  // deferred mode (tn_profile_defer): alternate two profiled graphs per phase, read the
  // times of a buffer's previous replay (two calls back) before replaying it again, return
  // only the algorithmic counters now -- the host never waits on the call in flight
  const int buf = P.prof_defer ? P.prof_buf[phase] : 0;
  if (P.prof_defer) P.prof_buf[phase] ^= 1;
  auto& G = P.prof_graph[phase][buf];
  if (profile_graph_enabled() && !G.failed) {
    if (!G.exec) {
      cudaGraph_t g = nullptr;
      const int64_t before = g_launches.load();
      try {
        CK(cudaStreamBeginCapture(P.cap, cudaStreamCaptureModeThreadLocal));
        record_profiled(P, phase, P.cap, G.mk, G.stat);
        CK(cudaStreamEndCapture(P.cap, &g));
        CK(cudaGraphInstantiate(&G.exec, g, 0));
        CK(cudaGraphDestroy(g));
        G.kernels = g_launches.load() - before;
      } catch (const Err&) {
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(P.cap, &dead);
        if (dead) cudaGraphDestroy(dead);
        cudaGetLastError();
        G.failed = true;
        G.reset();
      }
      g_launches = before;   // captured launches are counted when replayed
    }
    if (!G.failed) {
      if (G.pending) {          // deferred: this buffer's previous replay
        CK(cudaEventSynchronize(G.mk.v.back().first));
        read_marks(G.mk, P.prof_acc);
        G.pending = false;
      }
      CK(cudaGraphLaunch(G.exec, st));
      g_launches += G.kernels;
      if (P.prof_defer) {
        G.pending = true;
      } else {
        CK(cudaStreamSynchronize(st));
        read_marks(G.mk, pr);
      }
      add_profile(pr, G.stat);
      return;
    }
  }
  Marks mk;
  tn_profile stat;
  std::memset(&stat, 0, sizeof(stat));
  record_profiled(P, phase, st, mk, stat);
  CK(cudaEventSynchronize(mk.v.back().first));
  read_marks(mk, pr);
  add_profile(pr, stat);
  for (auto& e : mk.v) cudaEventDestroy(e.first);
}

// eager, profiled: the prologue (if asked and the plan has one), then slices [s0, s1)
void profile_slices(tn_plan_s& P, int64_t s0, int64_t s1, cudaStream_t st, tn_profile& pr, bool prologue) {
  std::memset(&pr, 0, sizeof(pr));
  if (prologue && P.n_pro > 0 && s1 > s0) profile_phase(P, 0, st, pr);
  for (int64_t s = s0; s < s1; ++s) profile_phase(P, 1, st, pr);
}

// allowed values of every sliced index for a host bitstring (bit v of mask[j]); a slice
// with a digit outside its mask contracts to exactly 0 (tn_plan_s::Forced)
std::vector<uint32_t> slice_masks(const tn_plan_s& P, const uint8_t* bits) {
  std::vector<uint32_t> m(P.sl_log2_h.size());
  for (size_t j = 0; j < m.size(); ++j) m[j] = (P.sl_log2_h[j] >= 5) ? 0xffffffffu : (1u << (1 << P.sl_log2_h[j])) - 1;
  for (const auto& f : P.forced) {
    size_t combo = 0;
    for (int q : f.qubits) combo = (combo << 1) | (bits[q] & 1);
    for (int v = 0; v < (1 << f.dim_log2); ++v)
      if (f.zero[(combo << f.dim_log2) | v]) m[f.pos] &= ~(1u << v);
  }
  return m;
}
bool slice_allowed(const tn_plan_s& P, const std::vector<uint32_t>& m, int64_t s) {
  for (size_t j = 0; j < m.size(); ++j) {
    const int v = P.sl_shift_h[j] >= 63 ? 0 : (int)((s >> P.sl_shift_h[j]) & ((int64_t(1) << P.sl_log2_h[j]) - 1));
    if (!((m[j] >> v) & 1)) return false;
  }
  return true;
}
bool masks_full(const tn_plan_s& P, const std::vector<uint32_t>& m) {
  for (size_t j = 0; j < m.size(); ++j)
    if (P.sl_log2_h[j] < 5 && m[j] != (1u << (1 << P.sl_log2_h[j])) - 1) return false;
  return true;
}

// graph replays of slices [s0, s1) on `st`; with a host bitstring, provably zero slices
// are skipped (the slice counter is set before each replay)
// the slice-invariant prologue of the bitstring in P.bits_d (graph)
void run_prologue(tn_plan_s& P, cudaStream_t st) {
  if (P.n_pro == 0) return;
  CK(cudaGraphLaunch(P.graph_pro, st));
  g_launches += P.kernels_pro;
}

// bits == nullptr: the bitstring already in P.bits_d and its prologue already run
// (tn_contract_prepared); otherwise copy it in and run the prologue first
void run_slices(tn_plan_s& P, const uint8_t* bits, bool bits_on_device, int64_t s0, int64_t s1, cudaStream_t st) {
  if (s0 < 0 || s1 > P.n_slices || s0 > s1) throw Err(TN_EINVAL, "slice range out of bounds");
  if (!bits && P.n_pro > 0 && !P.prepared) throw Err(TN_EINVAL, "tn_contract_prepared without tn_prepare");
  if (bits) P.prepared = false;     // this call's prologue replaces the prepared bitstring
  CK(cudaSetDevice(P.device));
  if (bits && P.net->n_qubits > 0)
    CK(cudaMemcpyAsync(P.bits_d, bits, P.net->n_qubits, bits_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(P.amp_d, 0, 16, st));
  std::vector<uint32_t> m;
  if (bits && !bits_on_device && !P.forced.empty()) m = slice_masks(P, bits);
  if (bits && s1 > s0) {
    bool any = m.empty();
    for (int64_t s = s0; s < s1 && !any; ++s) any = slice_allowed(P, m, s);
    if (any) run_prologue(P, st);
  }
  if (m.empty() || masks_full(P, m)) {
    set_i64_kernel<<<1, 1, 0, st>>>(P.slice_d, s0);
    for (int64_t s = s0; s < s1; ++s) {
      CK(cudaGraphLaunch(P.graph, st));
      g_launches += P.kernels_per_slice;
    }
    return;
  }
  for (int64_t s = s0; s < s1; ++s) {
    if (!slice_allowed(P, m, s)) continue;
    set_i64_kernel<<<1, 1, 0, st>>>(P.slice_d, s);
    CK(cudaGraphLaunch(P.graph, st));
    g_launches += P.kernels_per_slice + 1;
  }
}

}  // namespace

// ================================================================== C ABI =====
extern "C" {

const char* tn_last_error(void) { return g_err.c_str(); }
const char* tn_version(void) { return "paper_2208_01498_b200 0.1 (sm_100a)"; }
int64_t tn_kernel_launches(void) { return g_launches.load(); }

int tn_build_network(int32_t n_qubits, const double* qubit_xy, int32_t n_gates, const int32_t* gate_qubits,
                     const double* gate_mats, int32_t diag_hyper, tn_network* out) {
  return guard([&] {
    if (!out || n_qubits < 1 || !qubit_xy || n_gates < 0 || (n_gates > 0 && (!gate_qubits || !gate_mats)))
      throw Err(TN_EINVAL, "tn_build_network: bad arguments");
    for (int g = 0; g < n_gates; ++g) {
      int a = gate_qubits[2 * g], b = gate_qubits[2 * g + 1];
      if (a < 0 || a >= n_qubits || b >= n_qubits || b == a || b < -1)
        throw Err(TN_EINVAL, "tn_build_network: bad qubit ids in gate " + std::to_string(g));
    }
    auto h = std::make_unique<tn_network_s>();
    h->net = tn::build_network(n_qubits, qubit_xy, n_gates, gate_qubits, gate_mats, diag_hyper != 0);
    *out = h.release();
  });
}
void tn_network_free(tn_network net) { delete net; }

int tn_network_get_info(tn_network h, tn_network_info* info) {
  return guard([&] {
    if (!h || !info) throw Err(TN_EINVAL, "null");
    info->n_tensors = (int32_t)h->net.tensors.size();
    info->n_indices = (int32_t)h->net.dims.size();
    info->n_qubits = h->net.n_qubits;
    int mr = 0;
    for (auto& t : h->net.tensors) mr = std::max(mr, (int)t.inds.size());
    info->max_rank = mr;
    info->radius = h->net.radius;
    info->k_bound = h->net.k_bound;
  });
}
int tn_network_dims(tn_network h, int32_t* dims, int32_t* out_legs) {
  return guard([&] {
    if (!h) throw Err(TN_EINVAL, "null");
    if (dims) for (size_t i = 0; i < h->net.dims.size(); ++i) dims[i] = h->net.dims[i];
    if (out_legs) for (int q = 0; q < h->net.n_qubits; ++q) out_legs[q] = h->net.out_leg[q];
  });
}
int tn_network_tensor(tn_network h, int32_t t, int32_t* rank, int32_t* inds, double* pos, double* data,
                      int64_t data_cap) {
  return guard([&] {
    if (!h || t < 0 || t >= (int)h->net.tensors.size()) throw Err(TN_EINVAL, "bad tensor id");
    const auto& T = h->net.tensors[t];
    if (rank) *rank = (int32_t)T.inds.size();
    if (inds) for (size_t k = 0; k < T.inds.size(); ++k) inds[k] = T.inds[k];
    if (pos) { pos[0] = T.px; pos[1] = T.py; }
    if (data) {
      if (data_cap < (int64_t)T.data.size() * 2) throw Err(TN_EINVAL, "data buffer too small");
      for (size_t k = 0; k < T.data.size(); ++k) { data[2 * k] = T.data[k].real(); data[2 * k + 1] = T.data[k].imag(); }
    }
  });
}

void tn_order_params_default(tn_order_params* p) {
  if (!p) return;
  tn::OrderParams d;
  p->leaf_size = d.leaf_size; p->a_max = d.a_max; p->n_valid = d.n_valid; p->max_tries = d.max_tries;
  p->n_seeds = d.n_seeds; p->max_log2_size = d.max_log2_size;
}

int tn_find_order(tn_network h, const tn_order_params* params, uint64_t seed, tn_order* out) {
  return guard([&] {
    if (!h || !out) throw Err(TN_EINVAL, "null");
    tn::OrderParams p;
    if (params) {
      p.leaf_size = params->leaf_size; p.a_max = params->a_max; p.n_valid = params->n_valid;
      p.max_tries = params->max_tries; p.n_seeds = params->n_seeds; p.max_log2_size = params->max_log2_size;
    }
    if (p.leaf_size < 1 || p.a_max < 1 || p.n_valid < 1 || p.max_tries < 1 || p.n_seeds < 1)
      throw Err(TN_EINVAL, "tn_find_order: bad params");
    auto o = std::make_unique<tn_order_s>();
    o->ord = tn::find_order(h->net, seed, p);
    o->net = &h->net;
    *out = o.release();
  });
}
int tn_order_import(tn_network h, const int32_t* steps, int32_t n_steps, const int32_t* slices, int32_t n_slices,
                    int32_t median_fallbacks, tn_order* out) {
  return guard([&] {
    if (!h || !out || n_steps < 0 || n_slices < 0 || (n_steps > 0 && !steps) || (n_slices > 0 && !slices))
      throw Err(TN_EINVAL, "tn_order_import: null or negative argument");
    const tn::Network& net = h->net;
    const int n = (int)net.tensors.size();
    if (n_steps != std::max(n - 1, 0))
      throw Err(TN_EINVAL, "tn_order_import: a contraction tree of " + std::to_string(n) + " tensors has " +
                               std::to_string(std::max(n - 1, 0)) + " steps, got " + std::to_string(n_steps));
    // every step takes two distinct live nodes (leaves 0..n-1 or earlier results) and
    // creates node n + k: n - 1 such steps leave exactly one node, the root
    std::vector<char> alive(n + n_steps, 0);
    std::fill(alive.begin(), alive.begin() + n, 1);
    std::vector<std::pair<int, int>> st(n_steps);
    for (int k = 0; k < n_steps; ++k) {
      const int a = steps[2 * k], b = steps[2 * k + 1];
      if (a == b || a < 0 || b < 0 || a >= n + k || b >= n + k || !alive[a] || !alive[b])
        throw Err(TN_EINVAL, "tn_order_import: step " + std::to_string(k) + " does not contract two live nodes");
      alive[a] = alive[b] = 0;
      alive[n + k] = 1;
      st[k] = {a, b};
    }
    // sliced indices: distinct closed (non-output) indices of the network, kept sorted
    std::vector<char> closed(net.dims.size(), 0);
    for (int t = 0; t < n; ++t)
      for (int i : net.closed_inds(t)) closed[i] = 1;
    std::vector<int> sl(slices, slices + n_slices);
    std::sort(sl.begin(), sl.end());
    for (size_t j = 0; j < sl.size(); ++j)
      if (sl[j] < 0 || sl[j] >= (int)closed.size() || !closed[sl[j]] || (j > 0 && sl[j] == sl[j - 1]))
        throw Err(TN_EINVAL, "tn_order_import: sliced index " + std::to_string(sl[j]) +
                                 " is not a distinct closed index of the network");
    auto o = std::make_unique<tn_order_s>();
    o->ord = tn::import_order(net, std::move(st), std::move(sl), median_fallbacks);
    o->net = &net;
    *out = o.release();
  });
}

void tn_order_free(tn_order o) { delete o; }

int tn_order_get_info(tn_order o, tn_order_info* info) {
  return guard([&] {
    if (!o || !info) throw Err(TN_EINVAL, "null");
    const auto& od = o->ord;
    info->n_steps = (int32_t)od.steps.size();
    info->n_slices = (int32_t)od.slices.size();
    info->max_step_log2 = od.step_m.empty() ? 0 : *std::max_element(od.step_m.begin(), od.step_m.end());
    info->max_size_log2 = od.step_res.empty() ? 0 : *std::max_element(od.step_res.begin(), od.step_res.end());
    info->median_fallbacks = od.median_fallbacks;
    info->log2_total_2M = od.total_2M > 0 ? std::log2(od.total_2M) : 0;
    // one slice: drop the sliced bits of every step
    auto kept = tn::kept_per_step(*o->net, od.steps);
    std::set<int> sl(od.slices.begin(), od.slices.end());
    int n = (int)o->net->tensors.size();
    std::vector<std::vector<int>> node(n + od.steps.size());
    for (int t = 0; t < n; ++t) node[t] = o->net->closed_inds(t);
    double w = 0;
    int sbits = 0;
    for (int i : od.slices) sbits += o->net->log2dim(i);
    const int64_t nsl = sbits >= 63 ? INT64_MAX : int64_t(1) << sbits;
    for (size_t k = 0; k < od.steps.size(); ++k) {
      std::set<int> u(node[od.steps[k].first].begin(), node[od.steps[k].first].end());
      u.insert(node[od.steps[k].second].begin(), node[od.steps[k].second].end());
      int m = 0;
      for (int i : u) if (!sl.count(i)) m += o->net->log2dim(i);
      w += std::ldexp(1.0, m + 1);
      node[n + k] = kept[k];
    }
    info->log2_slice_2M = w > 0 ? std::log2(w) : 0;
    info->n_slice_assignments = nsl;
    info->slice_bits = sbits;
  });
}
int tn_order_steps(tn_order o, int32_t* steps) {
  return guard([&] {
    if (!o || !steps) throw Err(TN_EINVAL, "null");
    for (size_t k = 0; k < o->ord.steps.size(); ++k) { steps[2 * k] = o->ord.steps[k].first; steps[2 * k + 1] = o->ord.steps[k].second; }
  });
}
int tn_order_slices(tn_order o, int32_t* slices) {
  return guard([&] {
    if (!o) throw Err(TN_EINVAL, "null");
    if (slices) for (size_t k = 0; k < o->ord.slices.size(); ++k) slices[k] = o->ord.slices[k];
  });
}

int tn_plan_create(tn_network h, tn_order o, int32_t dtype, int32_t device, tn_plan* out) {
  return guard([&] {
    if (!h || !o || !out || o->net != &h->net) throw Err(TN_EINVAL, "tn_plan_create: bad handles");
    if (dtype != TN_C64 && dtype != TN_C128) throw Err(TN_EINVAL, "bad dtype");
    check_device(device);
    auto p = std::make_unique<tn_plan_s>();
    p->dtype = dtype;
    p->device = device;
    try {
      build_plan(*p, h->net, o->ord, true);
    } catch (const Err& e) {
      // the slice-reuse frontier does not fit: plan without it
      if (e.code != TN_ENOMEM) throw;
      p = std::make_unique<tn_plan_s>();
      p->dtype = dtype;
      p->device = device;
      build_plan(*p, h->net, o->ord, false);
    }
    *out = p.release();
  });
}
void tn_plan_free(tn_plan p) { delete p; }

int tn_plan_get_info(tn_plan p, tn_plan_info* info) {
  return guard([&] {
    if (!p || !info) throw Err(TN_EINVAL, "null");
    info->flops_per_slice = p->flops;
    info->n_slices = p->n_slices;
    info->arena_bytes = p->arena_bytes;
    info->n_steps_small = p->n_small;
    info->n_steps_tc = (int32_t)p->tcs.size();
    info->n_launches_per_slice = (int32_t)p->kernels_per_slice;
    info->tc_flops_per_slice = p->tc_flops;
    info->slice_bits = p->slice_bits;
    info->flops_prologue = p->flops_pro;
    info->frontier_bytes = p->frontier_bytes;
    info->n_launches_prologue = (int32_t)p->kernels_pro;
  });
}

int tn_plan_steps(tn_plan p, int32_t* out) {
  return guard([&] {
    if (!p || !out) throw Err(TN_EINVAL, "null");
    std::copy(p->step_table.begin(), p->step_table.end(), out);
  });
}

int tn_contract(tn_plan p, const uint8_t* bits, int64_t slice_begin, int64_t slice_end, double* amp, void* stream) {
  return guard([&] {
    if (!p || !amp || (!bits && p->net->n_qubits > 0)) throw Err(TN_EINVAL, "null");
    cudaStream_t st = (cudaStream_t)stream;
    run_slices(*p, bits, false, slice_begin, slice_end, st);
    double h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, p->amp_d, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    amp[0] = h[0];
    amp[1] = h[1];
  });
}

int tn_contract_device(tn_plan p, const uint8_t* bits_dev, int64_t slice_begin, int64_t slice_end, void* amp_dev,
                       void* stream) {
  return guard([&] {
    if (!p || !amp_dev || (!bits_dev && p->net->n_qubits > 0)) throw Err(TN_EINVAL, "null");
    cudaStream_t st = (cudaStream_t)stream;
    run_slices(*p, bits_dev, true, slice_begin, slice_end, st);
    add_amp_kernel<<<1, 1, 0, st>>>(reinterpret_cast<double2*>(amp_dev), p->amp_d);
    g_launches++;
    CK(cudaGetLastError());
  });
}

int tn_contract_profiled(tn_plan p, const uint8_t* bits_dev, int64_t slice_begin, int64_t slice_end, void* amp_dev,
                         void* stream, tn_profile* prof) {
  return guard([&] {
    if (!p || !amp_dev || !prof || (!bits_dev && p->net->n_qubits > 0)) throw Err(TN_EINVAL, "null");
    if (slice_begin < 0 || slice_end > p->n_slices || slice_begin > slice_end) throw Err(TN_EINVAL, "slice range");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaSetDevice(p->device));
    if (p->net->n_qubits > 0) CK(cudaMemcpyAsync(p->bits_d, bits_dev, p->net->n_qubits, cudaMemcpyDeviceToDevice, st));
    p->prepared = false;
    set_i64_kernel<<<1, 1, 0, st>>>(p->slice_d, slice_begin);
    CK(cudaMemsetAsync(p->amp_d, 0, 16, st));
    profile_slices(*p, slice_begin, slice_end, st, *prof, true);
    add_amp_kernel<<<1, 1, 0, st>>>(reinterpret_cast<double2*>(amp_dev), p->amp_d);
    g_launches++;
    CK(cudaGetLastError());
  });
}

int tn_prepare(tn_plan p, const uint8_t* bits_dev, void* stream, tn_profile* prof) {
  return guard([&] {
    if (!p || (!bits_dev && p->net->n_qubits > 0)) throw Err(TN_EINVAL, "null");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaSetDevice(p->device));
    if (p->net->n_qubits > 0) CK(cudaMemcpyAsync(p->bits_d, bits_dev, p->net->n_qubits, cudaMemcpyDeviceToDevice, st));
    if (prof) {
      std::memset(prof, 0, sizeof(*prof));
      if (p->n_pro > 0) profile_phase(*p, 0, st, *prof);
    } else {
      run_prologue(*p, st);
    }
    p->prepared = true;
    CK(cudaGetLastError());
  });
}

int tn_contract_prepared(tn_plan p, int64_t slice_begin, int64_t slice_end, void* amp_dev, void* stream,
                         tn_profile* prof) {
  return guard([&] {
    if (!p || !amp_dev) throw Err(TN_EINVAL, "null");
    if (slice_begin < 0 || slice_end > p->n_slices || slice_begin > slice_end) throw Err(TN_EINVAL, "slice range");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaSetDevice(p->device));
    if (prof) {
      if (p->n_pro > 0 && !p->prepared) throw Err(TN_EINVAL, "tn_contract_prepared without tn_prepare");
      set_i64_kernel<<<1, 1, 0, st>>>(p->slice_d, slice_begin);
      CK(cudaMemsetAsync(p->amp_d, 0, 16, st));
      profile_slices(*p, slice_begin, slice_end, st, *prof, false);
    } else {
      run_slices(*p, nullptr, true, slice_begin, slice_end, st);
    }
    add_amp_kernel<<<1, 1, 0, st>>>(reinterpret_cast<double2*>(amp_dev), p->amp_d);
    g_launches++;
    CK(cudaGetLastError());
  });
}

int tn_profile_defer(tn_plan p, int32_t on) {
  return guard([&] {
    if (!p) throw Err(TN_EINVAL, "null");
    CK(cudaSetDevice(p->device));
    p->prof_defer = on != 0;
  });
}

int tn_profile_collect(tn_plan p, tn_profile* prof) {
  return guard([&] {
    if (!p || !prof) throw Err(TN_EINVAL, "null");
    CK(cudaSetDevice(p->device));
    for (auto& ph : p->prof_graph)
      for (auto& g : ph)
        if (g.pending) {
          CK(cudaEventSynchronize(g.mk.v.back().first));
          read_marks(g.mk, p->prof_acc);
          g.pending = false;
        }
    std::memset(prof, 0, sizeof(*prof));
    add_profile(*prof, p->prof_acc);
    p->prof_acc = tn_profile{};
  });
}

int tn_amplitudes(tn_plan p, const uint8_t* bits, int32_t n_bits, double* amps, void* stream) {
  return guard([&] {
    if (!p || !amps || n_bits < 0 || (!bits && n_bits > 0)) throw Err(TN_EINVAL, "null");
    cudaStream_t st = (cudaStream_t)stream;
    const int nq = p->net->n_qubits;
    CK(cudaSetDevice(p->device));
    p->prepared = false;
    if (p->extra.empty() || n_bits < 2) {
      for (int j = 0; j < n_bits; ++j) {
        run_slices(*p, bits + (size_t)j * nq, false, 0, p->n_slices, st);
        CK(cudaMemcpyAsync(amps + 2 * j, p->amp_d, 16, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
      return;
    }
    // lanes: bitstring j on lane j mod L, each lane on its own stream; bitstrings in, and
    // amplitudes out, move in one copy each
    const int L = 1 + (int)p->extra.size();
    uint8_t* bits_all = nullptr;
    double2* res = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&bits_all), std::max<size_t>(1, (size_t)n_bits * nq), st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&res), (size_t)n_bits * 16, st));
    if (nq > 0) CK(cudaMemcpyAsync(bits_all, bits, (size_t)n_bits * nq, cudaMemcpyHostToDevice, st));
    cudaEvent_t ready;
    CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(cudaEventRecord(ready, st));
    std::vector<cudaStream_t> ls(L);
    ls[0] = p->cap;
    for (int l = 1; l < L; ++l) ls[l] = p->extra[l - 1].stream;
    for (int l = 0; l < L; ++l) CK(cudaStreamWaitEvent(ls[l], ready, 0));
    for (int j = 0; j < n_bits; ++j) {
      const int l = j % L;
      cudaStream_t ss = ls[l];
      uint8_t* bd = l ? p->extra[l - 1].bits_d : p->bits_d;
      int64_t* sd = l ? p->extra[l - 1].slice_d : p->slice_d;
      double2* ad = l ? p->extra[l - 1].amp_d : p->amp_d;
      cudaGraphExec_t gr = l ? p->extra[l - 1].graph : p->graph;
      cudaGraphExec_t gp = l ? p->extra[l - 1].graph_pro : p->graph_pro;
      if (nq > 0) CK(cudaMemcpyAsync(bd, bits_all + (size_t)j * nq, nq, cudaMemcpyDeviceToDevice, ss));
      CK(cudaMemsetAsync(ad, 0, 16, ss));
      std::vector<uint32_t> m;
      if (!p->forced.empty()) m = slice_masks(*p, bits + (size_t)j * nq);
      const bool full = m.empty() || masks_full(*p, m);
      if (gp && p->n_slices > 0) {
        CK(cudaGraphLaunch(gp, ss));
        g_launches += p->kernels_pro;
      }
      if (full) set_i64_kernel<<<1, 1, 0, ss>>>(sd, 0);
      for (int64_t s = 0; s < p->n_slices; ++s) {
        if (!full) {
          if (!slice_allowed(*p, m, s)) continue;
          set_i64_kernel<<<1, 1, 0, ss>>>(sd, s);
        }
        CK(cudaGraphLaunch(gr, ss));
        g_launches += p->kernels_per_slice;
      }
      CK(cudaMemcpyAsync(res + j, ad, 16, cudaMemcpyDeviceToDevice, ss));
    }
    for (int l = 0; l < L; ++l) {
      CK(cudaEventRecord(ready, ls[l]));
      CK(cudaStreamWaitEvent(st, ready, 0));
    }
    CK(cudaMemcpyAsync(amps, res, (size_t)n_bits * 16, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(bits_all, st));
    CK(cudaFreeAsync(res, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaEventDestroy(ready));
  });
}

int tn_contributing_slices(tn_plan p, const uint8_t* bits, int64_t* count) {
  return guard([&] {
    if (!p || !count || (!bits && p->net->n_qubits > 0)) throw Err(TN_EINVAL, "null");
    const auto m = slice_masks(*p, bits);
    double c = 1.0;
    for (size_t j = 0; j < m.size(); ++j)
      c *= p->sl_log2_h[j] >= 5 ? std::ldexp(1.0, p->sl_log2_h[j]) : (double)__builtin_popcount(m[j]);
    *count = c >= 9.2e18 ? INT64_MAX : (int64_t)c;
  });
}

int tn_contributing_slice_ids(tn_plan p, const uint8_t* bits, int64_t slice_begin, int64_t cap, int64_t* ids,
                              int64_t* n) {
  return guard([&] {
    if (!p || !n || cap < 0 || (cap > 0 && !ids) || (!bits && p->net->n_qubits > 0) || slice_begin < 0)
      throw Err(TN_EINVAL, "null");
    const auto m = slice_masks(*p, bits);
    int64_t k = 0;
    for (int64_t s = slice_begin; s < p->n_slices && k < cap; ++s)
      if (slice_allowed(*p, m, s)) ids[k++] = s;
    *n = k;
  });
}

int tn_plan_set_lanes(tn_plan p, int32_t n_lanes) {
  return guard([&] {
    if (!p || n_lanes < 1) throw Err(TN_EINVAL, "tn_plan_set_lanes: bad arguments");
    CK(cudaSetDevice(p->device));
    while ((int)p->extra.size() + 1 < n_lanes) add_lane(*p);
  });
}

int tn_contract_pair(int32_t dtype, const void* A, int32_t rank_a, const int32_t* inds_a, const void* B, int32_t rank_b,
                     const int32_t* inds_b, void* C, int32_t rank_c, const int32_t* inds_c, const int32_t* dims,
                     int32_t n_dims, int32_t path, void* stream) {
  return guard([&] {
    if (!A || !B || !C || !dims || rank_a < 0 || rank_b < 0 || rank_c < 0 || (rank_a && !inds_a) ||
        (rank_b && !inds_b) || (rank_c && !inds_c))
      throw Err(TN_EINVAL, "tn_contract_pair: null argument");
    if (dtype != TN_C64 && dtype != TN_C128) throw Err(TN_EINVAL, "bad dtype");
    std::vector<int> l2(n_dims);
    for (int i = 0; i < n_dims; ++i) {
      int d = dims[i], l = 0;
      while ((1 << l) < d) ++l;
      if (d < 1 || (1 << l) != d) throw Err(TN_EINVAL, "dimensions must be powers of two");
      l2[i] = l;
    }
    auto chk = [&](const int32_t* ii, int r) {
      std::vector<int> v(ii, ii + r);
      for (int i : v) if (i < 0 || i >= n_dims) throw Err(TN_EINVAL, "index id out of range");
      if (std::set<int>(v.begin(), v.end()).size() != v.size()) throw Err(TN_EINVAL, "repeated index");
      return v;
    };
    NodeLayout LA, LB;
    LA.inds = chk(inds_a, rank_a);
    LB.inds = chk(inds_b, rank_b);
    std::vector<int> ci = chk(inds_c, rank_c);
    std::set<int> kept(ci.begin(), ci.end());
    for (int i : ci)
      if (!std::count(LA.inds.begin(), LA.inds.end(), i) && !std::count(LB.inds.begin(), LB.inds.end(), i))
        throw Err(TN_EINVAL, "output index not in an operand");
    Classes cl = classify(LA, LB, kept);
    // C must be [batch][free of one operand][free of the other] (each group in C's order)
    std::set<int> sbt(cl.batch.begin(), cl.batch.end()), sl(cl.lfree.begin(), cl.lfree.end()),
        sr(cl.rfree.begin(), cl.rfree.end());
    size_t nbt = cl.batch.size();
    for (size_t k = 0; k < nbt; ++k)
      if (!sbt.count(ci[k])) throw Err(TN_EUNSUPPORTED, "C must start with the batch indices");
    bool l_first = nbt < ci.size() ? sl.count(ci[nbt]) > 0 : true;
    std::vector<int> g1(ci.begin() + nbt, ci.begin() + nbt + (l_first ? cl.lfree.size() : cl.rfree.size()));
    std::vector<int> g2(ci.begin() + nbt + g1.size(), ci.end());
    for (int i : g1) if (!(l_first ? sl : sr).count(i)) throw Err(TN_EUNSUPPORTED, "C groups must be contiguous");
    for (int i : g2) if (!(l_first ? sr : sl).count(i)) throw Err(TN_EUNSUPPORTED, "C groups must be contiguous");
    std::vector<int> batch(ci.begin(), ci.begin() + nbt);
    int nb = sum_bits(batch, l2), kk = sum_bits(cl.contr, l2);
    const NodeLayout& LX = l_first ? LA : LB;
    const NodeLayout& LY = l_first ? LB : LA;
    int mx = sum_bits(g1, l2), my = sum_bits(g2, l2);
    const int auto_kind = want_tc(dtype, nb, mx, my, kk) ? (dtype == TN_C128 ? K_DMMA : K_TC)
                          : want_skinny(nb, mx, my, kk)   ? K_SKINNY
                          : want_wide(nb, mx, my, kk)     ? K_WIDE
                                                          : -1;
    const int big = path == TN_PATH_TC       ? (dtype == TN_C128 ? K_DMMA : K_TC)
                    : path == TN_PATH_SKINNY ? K_SKINNY
                    : path == TN_PATH_WIDE   ? K_WIDE
                    : path == TN_PATH_AUTO   ? auto_kind
                                             : -1;
    if (big == K_TC && kk < 4) throw Err(TN_EUNSUPPORTED, "tensor-core path needs K >= 16 (complex64)");
    if (big == K_DMMA && kk < 1) throw Err(TN_EUNSUPPORTED, "DMMA path needs K >= 2 (complex128)");
    if (big == K_SKINNY && (mx > 6 || my > 6 || mx + my > 8 || kk < 1 || nb > 15))
      throw Err(TN_EUNSUPPORTED, "skinny path needs M, N <= 64, M N <= 256, K >= 2");
    if (big == K_WIDE && (kk > 4 || mx + kk < 3 || my + kk < 3))
      throw Err(TN_EUNSUPPORTED, "wide path needs K <= 16 and >= 8 entries per operand and batch");
    cudaStream_t st = (cudaStream_t)stream;
    int cur = 0;
    CK(cudaGetDevice(&cur));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, cur));
    if (prop.major != 10) throw Err(TN_ECUDA, "sm_100 device required");
    TabPool pool;
    std::vector<void*> ptrs = {const_cast<void*>(l_first ? A : B), const_cast<void*>(l_first ? B : A), C};
    std::vector<void*> allocs;
    struct FreeOnExit {                 // scratch goes back to the pool on every exit path
      std::vector<void*>& v;
      cudaStream_t s;
      ~FreeOnExit() {
        for (void* p : v) cudaFreeAsync(p, s);
      }
    } free_on_exit{allocs, st};
    auto dalloc = [&](size_t bytes) {
      void* p = nullptr;
      CK(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), st));
      allocs.push_back(p);
      return p;
    };
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    };
    void** ptrs_d = (void**)dalloc(3 * sizeof(void*));
    h2d(ptrs_d, ptrs.data(), 3 * sizeof(void*));
    if (big >= 0) {
      TcStep t;
      t.nb_bits = nb; t.m_bits = mx; t.n_bits = my; t.k_bits = kk;
      if (big == K_TC || big == K_DMMA) {
        finish_tc_shape(t);
        finish_tc_kind(t, dtype);
      } else {
        finish_cuda_core(t, dtype, big);
      }
      t.c_node = 2;
      const int planes = t.kind == K_TC ? 4 : 2;
      const std::vector<int> kord = slab_k_order(cl.contr, mx >= my ? LX : LY, l2, t.n_slabs);
      t.px = make_pack(pool, 0, LX, batch, g1, kord, l2, planes, t.k_lo, &t.slab_x, t.m_lo);
      t.py = make_pack(pool, 1, LY, batch, g2, kord, l2, planes, t.k_lo, &t.slab_y);
      set_gather_maps(t, pool, 0, LX, 1, LY, batch, g1, g2, kord, l2);   // DMMA / wide
      size_t xb = (size_t)pack_bytes(t, t.kind == K_TC ? t.m_lo : mx), yb = (size_t)pack_bytes(t, my);
      size_t pb = (size_t)tc_partial_bytes(t);
      char* scratch = (char*)dalloc(xb + yb + pb + 3 * ALIGN);
      int64_t* tab_d = (int64_t*)dalloc(pool.v.size() * 8);
      h2d(tab_d, pool.v.data(), pool.v.size() * 8);
      t.x_off = 0;
      t.y_off = (int64_t)((xb + ALIGN - 1) / ALIGN * ALIGN);
      t.p_off = t.y_off + (int64_t)((yb + ALIGN - 1) / ALIGN * ALIGN);
      set_skinny_maps(t, scratch);
      if (t.kind == K_TC) {
        t.ta = make_plane_map(scratch + t.x_off, t.k_lo, t.m_lo, nb, 128, 4);
        t.tb = make_plane_map(scratch + t.y_off, t.k_lo, my, nb, t.pair ? tnd::tc::Cfg2::BNH : t.BN, 4);
        if (t.pair) t.tc = make_c_map(C, my, int64_t(1) << (nb + mx));
      }
      launch_tc(t, scratch, ptrs_d, tab_d, st);
      CK(cudaStreamSynchronize(st));  // host staging buffers must outlive the copies
    } else {
      SmallStep d{};
      d.a = 0; d.b = 1; d.c = 2;
      d.nb_bits = nb; d.m_bits = mx; d.n_bits = my; d.k_bits = kk;
      d.Ab = pool.add(group_of(batch, LX, l2)); d.Am = pool.add(group_of(g1, LX, l2));
      d.Ak = pool.add(group_of(cl.contr, LX, l2));
      d.Bb = pool.add(group_of(batch, LY, l2)); d.Bk = pool.add(group_of(cl.contr, LY, l2));
      d.Bn = pool.add(group_of(g2, LY, l2));
      set_small_mode(d);
      Wave w;
      w.steps = {d};
      int64_t outs = int64_t(1) << (nb + mx + my);
      w.prefix = {0, (outs + d.opc - 1) / d.opc};
      w.n_cta = w.prefix[1];
      w.steps_d = (SmallStep*)dalloc(sizeof(SmallStep));
      h2d(w.steps_d, w.steps.data(), sizeof(SmallStep));
      w.prefix_d = (int64_t*)dalloc(2 * sizeof(int64_t));
      h2d(w.prefix_d, w.prefix.data(), 2 * sizeof(int64_t));
      int64_t* tab_d = (int64_t*)dalloc(pool.v.size() * 8);
      h2d(tab_d, pool.v.data(), pool.v.size() * 8);
      if (dtype == TN_C64) launch_wave<float>(w, ptrs_d, tab_d, st);
      else launch_wave<double>(w, ptrs_d, tab_d, st);
      CK(cudaStreamSynchronize(st));
    }
    // (scratch freed by free_on_exit)
  });
}

}  // extern "C"
