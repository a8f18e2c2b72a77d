// Host-side structures of the B200 tensor-network engine (network, order, plan).
// Independent of oracle/: the algorithms are re-implemented from PAPER.md
// (arxiv 2208.01498) to the recipe written in DESIGN.md; every decision that shapes
// the order uses plain IEEE-754 double arithmetic (compiled with
// -ffp-contract=off) so that tests can require bit-identical orders.
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace tn {

using cplx = std::complex<double>;

struct Tensor {
  std::vector<int> inds;     // index ids in data-axis order (row-major, last fastest)
  std::vector<cplx> data;    // complex128 entries
  double px = 0, py = 0;     // embedding position (Theorem 2 proof)
  bool core = false;
  int created = 0;
};

struct Network {
  std::vector<int> dims;            // index id -> dimension (powers of two)
  std::vector<Tensor> tensors;      // final tensors, id order
  std::vector<int> out_leg;         // qubit -> open output index
  std::vector<int> out_owner;       // qubit -> tensor holding it
  double radius = 0, k_bound = 1, l = 0, r = 1;
  int F = 0, n_qubits = 0;
  bool diag_hyper = false;
  int log2dim(int i) const;
  bool is_out(int i) const;
  std::vector<int> closed_inds(int t) const;
};

// PAPER.md l.115-125 (Theorem 2 proof) + DESIGN.md readings R1-R4.
Network build_network(int n, const double* xy, int n_gates, const int32_t* gq,
                      const double* mats, bool diag_hyper, double eps_frac = 0.01);

struct OrderParams {
  int leaf_size = 8, a_max = 32, n_valid = 64, max_tries = 256, n_seeds = 4;
  int max_log2_size = 0;  // slicing target (index bits of the largest tensor), <= 0: none
};

struct Order {
  std::vector<std::pair<int, int>> steps;   // leaves 0..n-1, step k creates n+k
  std::vector<int> slices;                  // sliced index ids (sorted)
  std::vector<int> step_m;                  // log2 M of Eq. (3) per step (unsliced)
  std::vector<int> step_res;                // log2 result size per step (unsliced)
  double total_2M = 0;                      // sum_k 2 M_k (unsliced)
  int median_fallbacks = 0;
};

// SM Algorithm 1 + Theorem 1 proof hierarchy + greedy leaves (R5-R10), slicing R11.
Order find_order(const Network& net, uint64_t seed, const OrderParams& p);
// explicit steps / sliced indices (already validated) with their Eq. (3) costs
Order import_order(const Network& net, std::vector<std::pair<int, int>> steps, std::vector<int> slices,
                   int median_fallbacks);
std::vector<int> choose_slices(const Network& net, const std::vector<std::pair<int, int>>& steps,
                               int max_log2_size);

// per-step kept-index sets (sorted), as in the oracle's kept_per_step
std::vector<std::vector<int>> kept_per_step(const Network& net,
                                            const std::vector<std::pair<int, int>>& steps);

// SplitMix64 counter generator (shared recipe with oracle/rng.py)
uint64_t splitmix64(uint64_t x);
struct Stream {
  uint64_t key, ctr = 0;
  Stream(uint64_t seed, uint64_t sid);
  uint64_t u64();
  double uniform();
  uint64_t below(uint64_t m) { return u64() % m; }
};
uint64_t child_stream(uint64_t sid, int side);

}  // namespace tn
