/*
 * tn.h -- C ABI of the B200-native tensor-network contraction engine
 * (arxiv 2208.01498, Wahl & Strelchuk: separator-based contraction orders for
 * quantum-circuit amplitudes <x|C|0>).
 *
 * Four calls form the boundary named in BASELINE.json's north_star:
 *   tn_build_network  circuit -> closed tensor network
 *   tn_find_order     separator hierarchy -> pairwise order  (PAPER.md l.79-96,
 *                     SM Algorithm 1 l.195-209, SM l.217) + index slicing (l.178)
 *   tn_contract       order + bitstring -> scalar amplitude  (Eq. (3), l.82-86)
 *   tn_amplitudes     batch of bitstrings -> amplitudes
 * plus the hot operation itself, exported for step-level parity tests:
 *   tn_contract_pair  one pairwise contraction (Fig. 1b, l.54) on device buffers.
 *
 * Conventions
 *   - Every function returns TN_OK (0) or a positive error code; tn_last_error()
 *     gives a thread-local message.  Nothing aborts the process; on error no output
 *     is written and no handle is created.
 *   - Complex numbers are interleaved (re, im) pairs: complex128 = 2 doubles,
 *     complex64 = 2 floats.  Tensors are dense, row-major over their index list
 *     (last index fastest).  Index dimensions are powers of two.
 *   - Handles (tn_network, tn_order, tn_plan) are owned by the caller and released
 *     with the matching *_free; a network must outlive orders and plans made from it.
 *   - "host" pointers are ordinary CPU memory; "device" pointers are CUDA global
 *     memory on the plan's device.  Streams are cudaStream_t passed as void*
 *     (NULL = legacy default stream).
 *   - There is no CPU fallback: without a usable sm_100 device every device call
 *     returns TN_ECUDA.
 */
#ifndef TN_H_
#define TN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TN_OK = 0,
  TN_EINVAL = 1,        /* bad argument (null pointer, out-of-range id, bad layout) */
  TN_ECUDA = 2,         /* CUDA runtime / driver error or no sm_100 device */
  TN_ENOMEM = 3,        /* device arena does not fit the plan's budget */
  TN_EUNSUPPORTED = 4,  /* valid request outside what the engine implements */
  TN_EINTERNAL = 5
};

enum { TN_C64 = 0, TN_C128 = 1 };               /* arithmetic type of a plan */
/* kernel path of a step: AUTO as a plan chooses; SMALL: warp-batched CUDA-core kernel;
 * TC: tensor cores (tcgen05 fp16x2 for complex64, DMMA for complex128); SKINNY: CUDA-core
 * split-K for few outputs and a long contraction; WIDE: CUDA-core tiles for a short
 * contraction and a large output (the last two read planar packed operands). */
enum { TN_PATH_AUTO = 0, TN_PATH_SMALL = 1, TN_PATH_TC = 2, TN_PATH_SKINNY = 3, TN_PATH_WIDE = 4 };

typedef struct tn_network_s* tn_network;
typedef struct tn_order_s* tn_order;
typedef struct tn_plan_s* tn_plan;

const char* tn_last_error(void);
const char* tn_version(void);

/* ------------------------------------------------------------------ network --
 * tn_build_network: the closed tensor network of <x|C|0> for a circuit of single-
 * and two-qubit gates (PAPER.md "Classical Simulation of Quantum Circuits",
 * l.115-125).  Single-qubit gates and the |0> inputs are absorbed into the two-
 * qubit gate tensors (l.116); each two-qubit gate is split into two rank-3 tensors
 * joined by a bond of dimension <= 4 (Theorem 2 proof, l.122) placed at
 * x_i + (x_j - x_i)/4 and x_j + (x_i - x_j)/4 with radius l/4 + eps.  The output
 * projections <x_q| stay open legs (one per qubit) until a bitstring is bound.
 *   n_qubits     N >= 1
 *   qubit_xy     host, N x 2 doubles: qubit positions in R^2
 *   n_gates      G >= 0, applied in order
 *   gate_qubits  host, G x 2 int32: (a, -1) for a one-qubit gate, (a, b) a != b
 *   gate_mats    host, concatenated row-major complex128 matrices: 2x2 (8 doubles)
 *                for one-qubit gates, 4x4 (32 doubles) in basis |x_a x_b> (x_a the
 *                high bit) for two-qubit gates
 *   diag_hyper   0: paper's construction; 1: diagonal gates keep their wire index
 *                (hyperedge reading R3 of DESIGN.md, used for IQP circuits)
 *   out          receives the new handle
 */
int tn_build_network(int32_t n_qubits, const double* qubit_xy, int32_t n_gates,
                     const int32_t* gate_qubits, const double* gate_mats, int32_t diag_hyper,
                     tn_network* out);
void tn_network_free(tn_network net);

typedef struct {
  int32_t n_tensors, n_indices, n_qubits, max_rank;
  double radius, k_bound;
} tn_network_info;
int tn_network_get_info(tn_network net, tn_network_info* info);
/* dims: host int32[n_indices]; out_legs: host int32[n_qubits] (index id of qubit q's
 * open output leg) */
int tn_network_dims(tn_network net, int32_t* dims, int32_t* out_legs);
/* tensor t: rank, its index ids (host int32[max_rank]), position (2 doubles) and,
 * if data != NULL, its complex128 entries (data_cap doubles available). */
int tn_network_tensor(tn_network net, int32_t t, int32_t* rank, int32_t* inds, double* pos,
                      double* data, int64_t data_cap);

/* ------------------------------------------------------------------- order ---
 * tn_find_order: recursive sphere-separator bisection of the tensors' embedding
 * (SM Algorithm 1 steps 1-7; Theorem 1 proof boundary assignment), greedy order
 * inside leaf clusters of <= leaf_size tensors (SM l.217), the randomized hierarchy
 * built n_seeds times keeping the smallest Eq. (3) total; then, if
 * max_log2_size > 0, greedy index slicing until no tensor of the contraction has
 * more than max_log2_size index bits.  Deterministic in (network, params, seed) and
 * bit-identical to oracle/ssa.py.
 */
typedef struct {
  int32_t leaf_size;      /* default 8 */
  int32_t a_max;          /* centerpoint sample size, default 32 */
  int32_t n_valid;        /* valid circles compared per separator, default 64 */
  int32_t max_tries;      /* circles per centerpoint, default 256 */
  int32_t n_seeds;        /* hierarchies built, default 4 */
  int32_t max_log2_size;  /* slicing target in index bits, <= 0: no slicing */
} tn_order_params;
void tn_order_params_default(tn_order_params* p);
int tn_find_order(tn_network net, const tn_order_params* params, uint64_t seed, tn_order* out);
void tn_order_free(tn_order ord);

/* tn_order_import: an order given explicitly -- the steps (host int32[2 * n_steps], the
 * layout tn_order_steps returns) and sliced indices (host int32[n_slices], any order) of
 * an order tn_find_order produced, e.g. on another rank (multi-GPU: one host order
 * search per job, broadcast to the ranks; paper_2208_01498_b200/dist.py shared_order).
 * The tree is SM Algorithm 1's output as a plain contraction sequence (PAPER.md l.80,
 * Fig. 2: a binary tree over the network's tensors); the per-step Eq. (3) costs
 * (l.82-86) are recomputed.  median_fallbacks is carried into tn_order_info as given.
 * Errors: TN_EINVAL unless n_steps = n_tensors - 1 and every step contracts two distinct
 * live nodes (leaves 0..n-1, step k creating node n + k), and the sliced indices are
 * distinct closed (non-output) indices of `net`.  The caller keeps ownership of the
 * arrays (copied); `net` must outlive the order. */
int tn_order_import(tn_network net, const int32_t* steps, int32_t n_steps, const int32_t* slices,
                    int32_t n_slices, int32_t median_fallbacks, tn_order* out);

typedef struct {
  int32_t n_steps, n_slices;           /* n_slices = number of sliced indices */
  int32_t max_step_log2, max_size_log2; /* unsliced: max log2 M, max log2 result size */
  int32_t median_fallbacks;
  double log2_total_2M;                 /* log2 sum_k 2 M_k, unsliced (Eq. (3)) */
  double log2_slice_2M;                 /* log2 sum_k 2 M_k of one slice */
  int64_t n_slice_assignments;          /* prod of sliced dimensions, saturated at INT64_MAX */
  int32_t slice_bits;                   /* log2 n_slice_assignments (exact) */
} tn_order_info;
int tn_order_get_info(tn_order ord, tn_order_info* info);
/* steps: host int32[2 * n_steps] (a, b) pairs; leaves are tensor ids 0..n-1 and
 * step k creates node n + k.  slices: host int32[n_slices]. */
int tn_order_steps(tn_order ord, int32_t* steps);
int tn_order_slices(tn_order ord, int32_t* slices);

/* -------------------------------------------------------------------- plan ---
 * tn_plan_create: device execution plan for (network, order) in complex64 or
 * complex128 on CUDA device `device`: uploads the leaf tensors, assigns every
 * intermediate an offset in one device arena (reused across the tree, slices and
 * bitstrings), chooses the kernel path of every step (warp-level batched small
 * kernel vs tensor-core GEMM) and captures the launch sequence of one slice.
 */
int tn_plan_create(tn_network net, tn_order ord, int32_t dtype, int32_t device, tn_plan* out);
void tn_plan_free(tn_plan plan);

typedef struct {
  double flops_per_slice;        /* 8 * sum_k M_k (real flops of complex MACs) */
  int64_t n_slices;              /* slice assignments, saturated at INT64_MAX: with more than
                                    63 sliced bits only slice ids < 2^63 are addressable (their
                                    higher sliced bits are 0) */
  int64_t arena_bytes;           /* device arena size */
  int32_t n_steps_small, n_steps_tc, n_launches_per_slice;
  double tc_flops_per_slice;     /* part of flops_per_slice on the tensor-core path */
  int32_t slice_bits;            /* log2 of the number of slice assignments */
  /* Slice reuse: the steps whose subtree holds no sliced index
   * are the same in every slice of a bitstring; they form a prologue run once per
   * bitstring (flops_prologue, part of flops_per_slice), their outputs that feed
   * per-slice steps (frontier_bytes) stay in the arena, and each slice runs the rest.
   * 0 / 0 / 0 without slicing or with TN_SLICE_REUSE=0. */
  double flops_prologue;
  int64_t frontier_bytes;
  int32_t n_launches_prologue;
} tn_plan_info;
int tn_plan_get_info(tn_plan plan, tn_plan_info* info);

/* tn_plan_steps: per step k (order of tn_order_steps), 6 int32 in out[6k..6k+5]:
 * path (TN_PATH_SMALL / TC / SKINNY / WIDE), log2 batch, log2 M, log2 N, log2 K (the GEMM
 * shape C[b][m][n] = sum_k A[b][m][k] B[b][k][n] as executed), launch position. */
int tn_plan_steps(tn_plan plan, int32_t* out);

/* tn_contract: amplitude contribution of slices [slice_begin, slice_end) for one
 * bitstring (bits: host uint8[n_qubits], 0/1).  amp: host double[2] receives the
 * sum (complex128 regardless of the plan's dtype).  Synchronizes `stream`. */
int tn_contract(tn_plan plan, const uint8_t* bits, int64_t slice_begin, int64_t slice_end,
                double* amp, void* stream);
/* tn_contract_device: same, asynchronous; bits_dev: device uint8[n_qubits];
 * amp_dev: device complex128 accumulator (2 doubles, any plan dtype), the sum is ADDED
 * to it.  Slices are summed in fp64; the plan's power-of-two leaf scaling (DESIGN.md
 * "Range") is undone in fp64 at that sum, so slices far below the complex64 range of
 * the intermediates still contribute exactly as computed. */
int tn_contract_device(tn_plan plan, const uint8_t* bits_dev, int64_t slice_begin,
                       int64_t slice_end, void* amp_dev, void* stream);
/* tn_contract_profiled: as tn_contract_device, but with CUDA events around every kernel
 * class on `stream`: it replays a profiled CUDA graph of the prologue / a slice (the
 * plan's launches with event records between them, captured on first use; eager
 * launches with TN_PROFILE_GRAPH=0) and synchronizes `stream`; prof (host) receives the
 * summed device time per kernel class and the algorithmic flops / bytes.  The same holds
 * for tn_prepare / tn_contract_prepared with a profile. */
/* kernel classes of tn_profile.k_*: small-path waves, fp16x2 tensor-core pack, the
 * complex64 tcgen05 GEMMs (single-CTA cgemm_f16x2s_kernel, one-tile-per-pair
 * cgemm2_f16x2s_kernel, persistent pair cgemm2p_f16x2s_kernel), planar pack (skinny /
 * wide / DMMA operands), complex128 DMMA GEMM, skinny, wide, split-K reductions, other */
enum {
  TN_K_SMALL = 0, TN_K_PACK_TC, TN_K_GEMM_SINGLE, TN_K_GEMM_PAIR, TN_K_GEMM_PERSIST, TN_K_PACK_PLANAR,
  TN_K_DMMA, TN_K_SKINNY, TN_K_WIDE, TN_K_REDUCE, TN_K_OTHER, TN_K_COUNT
};
typedef struct {
  double ms_small, ms_pack, ms_gemm, ms_other;
  double flops_gemm, flops_small;          /* 8 * M (real flops of the complex MACs) */
  double bytes_small, bytes_pack;          /* algorithmic bytes read + written */
  int64_t n_gemm, n_pack, n_small, n_other;
  /* per kernel class (TN_K_*): device ms between its events, algorithmic flops and
   * bytes, number of timed intervals */
  double k_ms[16], k_flops[16], k_bytes[16];
  int64_t k_intervals[16];
} tn_profile;
int tn_contract_profiled(tn_plan plan, const uint8_t* bits_dev, int64_t slice_begin, int64_t slice_end,
                         void* amp_dev, void* stream, tn_profile* prof);
/* tn_profile_defer: with on != 0 the profiled calls on `plan` (tn_contract_profiled,
 * tn_prepare / tn_contract_prepared with a profile) do not wait for their kernels: each
 * replays one of two profiled graphs per phase (reading the device times of that graph's
 * previous replay first) and returns only the algorithmic flops / bytes and counts; the
 * device times of all deferred replays are summed in the plan until tn_profile_collect
 * waits for the outstanding ones and returns them (times only: ms_*, k_ms, k_intervals),
 * clearing the sum.  So a loop of profiled calls keeps the GPU busy (bench.py's timed
 * region).  Eager profiling (TN_PROFILE_GRAPH=0) stays synchronous. */
int tn_profile_defer(tn_plan plan, int32_t on);
int tn_profile_collect(tn_plan plan, tn_profile* prof);
/* Slice reuse across calls (PAPER.md l.178 index slicing):
 * tn_contract / tn_contract_device / tn_contract_profiled / tn_amplitudes run the
 * bitstring's slice-invariant prologue once per call, then the slices.  To spread the
 * slices of one bitstring over several calls without repeating the prologue:
 * tn_prepare copies the device bitstring bits_dev (uint8[n_qubits]) into the plan and
 * runs its prologue; tn_contract_prepared then ADDS the slices [slice_begin, slice_end)
 * of that bitstring to amp_dev (device complex128).  prof == NULL: CUDA-graph replay;
 * otherwise eager launches with CUDA events, prof (host) receives the pass's profile as
 * in tn_contract_profiled.  Any other contraction call on the plan (tn_contract*,
 * tn_amplitudes) in between invalidates the prepared state: tn_contract_prepared then
 * fails with TN_EINVAL (as it does before any tn_prepare) on plans that have a prologue.
 * The caller orders the calls on one stream. */
int tn_prepare(tn_plan plan, const uint8_t* bits_dev, void* stream, tn_profile* prof);
int tn_contract_prepared(tn_plan plan, int64_t slice_begin, int64_t slice_end, void* amp_dev, void* stream,
                         tn_profile* prof);
/* tn_amplitudes: full amplitudes (all slices) of n_bits bitstrings
 * (host uint8[n_bits * n_qubits]) into host double[2 * n_bits]; host<->device
 * copies included.  With lanes (tn_plan_set_lanes) bitstring j runs on lane j mod L,
 * the lanes concurrently on their own streams (ordered after `stream`).  Synchronizes
 * `stream`. */
int tn_amplitudes(tn_plan plan, const uint8_t* bits, int32_t n_bits, double* amps, void* stream);
/* tn_contributing_slices: number of slices of the plan that are not provably zero for the
 * bitstring (host uint8[n_qubits]): a leaf whose only sliced index is j vanishes for some
 * values of j given its output bits (e.g. the delta of a CZ bond next to a bound output
 * leg), and every slice with such a digit contracts to exactly 0.  tn_contract and
 * tn_amplitudes (host bitstrings) skip those slices; the device-bitstring calls run them.
 * count saturates at INT64_MAX. */
int tn_contributing_slices(tn_plan plan, const uint8_t* bits, int64_t* count);
/* tn_contributing_slice_ids: the first (at most cap) contributing slice ids >= slice_begin,
 * ascending, into host ids[]; *n receives how many were written. */
int tn_contributing_slice_ids(tn_plan plan, const uint8_t* bits, int64_t slice_begin, int64_t cap, int64_t* ids,
                              int64_t* n);
/* tn_plan_set_lanes: give the plan n_lanes (>= 1) independent copies of its per-
 * contraction device state (arena, pointer table, bitstring / slice / amplitude slots,
 * tensor maps, stream, CUDA graph) so tn_amplitudes contracts n_lanes bitstrings at
 * once; each lane costs one more arena (tn_plan_info.arena_bytes).  TN_ENOMEM (and the
 * lanes made so far kept) when the next arena does not fit.  Lanes are never removed. */
int tn_plan_set_lanes(tn_plan plan, int32_t n_lanes);

/* ---------------------------------------------------------------- hot op ----
 * tn_contract_pair: C = sum over shared non-output indices of A * B (PAPER.md
 * Fig. 1b, l.54; cost M of Eq. (3)).  An index present in A, B and C is a batch
 * (hyperedge) index; every index of A and of B must appear in the other operand or
 * in C, and every index of C in A or B.  A, B, C: device buffers of `dtype`,
 * row-major over their index lists; dims[i] is the dimension of index id i
 * (0 <= i < n_dims, powers of two).  path: TN_PATH_AUTO picks the kernel like a
 * plan does; TN_PATH_SMALL / TC / SKINNY / WIDE force one (TN_EUNSUPPORTED if the
 * shape is outside what that kernel handles).  C must be 16-byte aligned (the
 * tensor-core pair kernels store it by TMA, the wide kernel by 16-byte vectors).
 * Runs on `stream` and synchronizes it before returning (its scratch buffers, taken
 * from the stream-ordered pool, are freed).
 */
int tn_contract_pair(int32_t dtype, const void* A, int32_t rank_a, const int32_t* inds_a,
                     const void* B, int32_t rank_b, const int32_t* inds_b, void* C,
                     int32_t rank_c, const int32_t* inds_c, const int32_t* dims, int32_t n_dims,
                     int32_t path, void* stream);

/* number of kernel launches this library issued since load (evidence counter) */
int64_t tn_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* TN_H_ */
