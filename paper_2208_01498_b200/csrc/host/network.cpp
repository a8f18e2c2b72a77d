// Circuit -> closed tensor network for <x|C|0>.
// PAPER.md "Classical Simulation of Quantum Circuits" l.115-125: single-qubit gates
// and boundary vectors are absorbed into the two-qubit gate tensors (l.116); each
// two-qubit gate is split into two rank-3 tensors joined by a bond of dimension
// <= 4 (l.122), placed at x_i + (x_j - x_i)/4, x_j + (x_i - x_j)/4, radius l/4 + eps.
// Readings R1-R4 are listed in DESIGN.md.
#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <stdexcept>

#include "tn_host.hpp"

namespace tn {

int Network::log2dim(int i) const {
  int d = dims[i], l = 0;
  while ((1 << l) < d) ++l;
  if ((1 << l) != d) throw std::runtime_error("index dimensions must be powers of two");
  return l;
}
bool Network::is_out(int i) const {
  return std::find(out_leg.begin(), out_leg.end(), i) != out_leg.end();
}
std::vector<int> Network::closed_inds(int t) const {
  std::vector<int> o;
  for (int i : tensors[t].inds)
    if (!is_out(i)) o.push_back(i);
  return o;
}

namespace {

// generic small pairwise contraction used by absorption (host, build time only):
// result axes = A's kept indices (A order) then B's new kept indices (B order).
Tensor merge_into(const Tensor& A, const Tensor& B, const std::set<int>& keep,
                  const std::vector<int>& dims) {
  std::vector<int> uni = A.inds;
  for (int i : B.inds)
    if (std::find(uni.begin(), uni.end(), i) == uni.end()) uni.push_back(i);
  std::vector<int> out;
  for (int i : A.inds)
    if (keep.count(i)) out.push_back(i);
  for (int i : B.inds)
    if (keep.count(i) && std::find(A.inds.begin(), A.inds.end(), i) == A.inds.end()) out.push_back(i);
  auto strides = [&](const std::vector<int>& inds) {
    std::vector<int64_t> s(inds.size());
    int64_t acc = 1;
    for (int k = (int)inds.size() - 1; k >= 0; --k) { s[k] = acc; acc *= dims[inds[k]]; }
    return std::make_pair(s, acc);
  };
  auto [sa, na] = strides(A.inds);
  auto [sb, nb] = strides(B.inds);
  auto [so, no] = strides(out);
  (void)na; (void)nb;
  Tensor R;
  R.inds = out;
  R.data.assign((size_t)no, cplx(0, 0));
  R.px = A.px; R.py = A.py; R.core = A.core; R.created = A.created;
  std::vector<int> val(uni.size(), 0);
  int64_t total = 1;
  for (int i : uni) total *= dims[i];
  auto pos_in = [&](const std::vector<int>& inds, const std::vector<int64_t>& st) {
    int64_t o = 0;
    for (size_t k = 0; k < inds.size(); ++k) {
      size_t u = std::find(uni.begin(), uni.end(), inds[k]) - uni.begin();
      o += st[k] * val[u];
    }
    return o;
  };
  for (int64_t it = 0; it < total; ++it) {
    int64_t r = it;
    for (int k = (int)uni.size() - 1; k >= 0; --k) { val[k] = (int)(r % dims[uni[k]]); r /= dims[uni[k]]; }
    R.data[pos_in(out, so)] += A.data[pos_in(A.inds, sa)] * B.data[pos_in(B.inds, sb)];
  }
  return R;
}

bool is_diag(const double* m, int d) {
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c)
      if (r != c && (m[2 * (r * d + c)] != 0.0 || m[2 * (r * d + c) + 1] != 0.0)) return false;
  return true;
}

}  // namespace

Network build_network(int n, const double* xy, int n_gates, const int32_t* gq, const double* mats,
                      bool diag_hyper, double eps_frac) {
  Network net;
  net.n_qubits = n;
  net.diag_hyper = diag_hyper;
  auto new_index = [&](int d) { net.dims.push_back(d); return (int)net.dims.size() - 1; };
  std::vector<int> wire(n);
  for (int q = 0; q < n; ++q) wire[q] = new_index(2);
  std::vector<Tensor> raw;
  auto add = [&](std::vector<int> inds, std::vector<cplx> data, double px, double py, bool core) {
    Tensor T;
    T.inds = std::move(inds); T.data = std::move(data);
    T.px = px; T.py = py; T.core = core; T.created = (int)raw.size();
    raw.push_back(std::move(T));
  };
  for (int q = 0; q < n; ++q) add({wire[q]}, {cplx(1, 0), cplx(0, 0)}, xy[2 * q], xy[2 * q + 1], false);
  double ltab = 0.0;
  std::vector<int> fcount(n, 0);
  size_t off = 0;
  for (int g = 0; g < n_gates; ++g) {
    int a = gq[2 * g], b = gq[2 * g + 1];
    if (b < 0) {
      const double* U = mats + off;
      off += 8;
      auto u = [&](int r, int c) { return cplx(U[2 * (2 * r + c)], U[2 * (2 * r + c) + 1]); };
      if (diag_hyper && is_diag(U, 2)) {
        add({wire[a]}, {u(0, 0), u(1, 1)}, xy[2 * a], xy[2 * a + 1], false);
      } else {
        int w = new_index(2);
        add({w, wire[a]}, {u(0, 0), u(0, 1), u(1, 0), u(1, 1)}, xy[2 * a], xy[2 * a + 1], false);
        wire[a] = w;
      }
      continue;
    }
    const double* U = mats + off;
    off += 32;
    auto u = [&](int r, int c) { return cplx(U[2 * (4 * r + c)], U[2 * (4 * r + c) + 1]); };
    fcount[a]++; fcount[b]++;
    double xa0 = xy[2 * a], xa1 = xy[2 * a + 1], xb0 = xy[2 * b], xb1 = xy[2 * b + 1];
    double dx = xa0 - xb0, dy = xa1 - xb1;
    ltab = std::max(ltab, std::sqrt(dx * dx + dy * dy));
    double pa0 = xa0 + (xb0 - xa0) / 4.0, pa1 = xa1 + (xb1 - xa1) / 4.0;
    double pb0 = xb0 + (xa0 - xb0) / 4.0, pb1 = xb1 + (xa1 - xb1) / 4.0;
    bool dg = is_diag(U, 4);
    if (dg && diag_hyper) {
      add({wire[a], wire[b]}, {u(0, 0), u(1, 1), u(2, 2), u(3, 3)}, pb0, pb1, true);
      continue;
    }
    int s, wa, wb;
    std::vector<cplx> X, Y;
    if (dg) {
      s = new_index(2); wa = new_index(2); wb = new_index(2);
      X.assign(8, cplx(0, 0)); Y.assign(8, cplx(0, 0));
      for (int i = 0; i < 2; ++i) {
        X[i * 4 + i * 2 + i] = 1.0;
        for (int k = 0; k < 2; ++k) Y[i * 4 + i * 2 + k] = u(2 * k + i, 2 * k + i);
      }
    } else {
      s = new_index(4); wa = new_index(2); wb = new_index(2);
      X.assign(16, cplx(0, 0)); Y.assign(16, cplx(0, 0));
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
          X[(i * 2 + j) * 4 + 2 * i + j] = 1.0;
          for (int k = 0; k < 4; ++k) Y[(i * 2 + j) * 4 + k] = u(2 * (k >> 1) + i, 2 * (k & 1) + j);
        }
    }
    add({wa, wire[a], s}, X, pa0, pa1, true);
    add({wb, wire[b], s}, Y, pb0, pb1, true);
    wire[a] = wa; wire[b] = wb;
  }
  net.out_leg = wire;
  std::set<int> outs(wire.begin(), wire.end());
  std::vector<char> alive(raw.size(), 1);
  std::map<int, std::set<int>> hold;
  for (size_t t = 0; t < raw.size(); ++t)
    for (int i : raw[t].inds) hold[i].insert((int)t);
  auto others = [&](int idx, int ex1, int ex2) {
    std::vector<int> o;
    auto it = hold.find(idx);
    if (it == hold.end()) return o;
    for (int h : it->second)
      if (h != ex1 && h != ex2) o.push_back(h);
    return o;
  };
  // absorption (R2)
  bool changed = true;
  while (changed) {
    changed = false;
    for (size_t t = 0; t < raw.size(); ++t) {
      if (!alive[t] || raw[t].core) continue;
      std::set<int> nb;
      for (int i : raw[t].inds)
        for (int h : others(i, (int)t, -1)) nb.insert(h);
      if (nb.empty()) continue;
      int tgt = -1;
      for (int h : nb)
        if (h > (int)t) { tgt = h; break; }
      if (tgt < 0) tgt = *nb.rbegin();
      std::set<int> keep;
      std::set<int> uni(raw[t].inds.begin(), raw[t].inds.end());
      uni.insert(raw[tgt].inds.begin(), raw[tgt].inds.end());
      for (int i : uni)
        if (outs.count(i) || !others(i, (int)t, tgt).empty()) keep.insert(i);
      Tensor R = merge_into(raw[tgt], raw[t], keep, net.dims);
      for (int i : raw[tgt].inds) hold[i].erase(tgt);
      for (int i : raw[t].inds) hold[i].erase((int)t);
      raw[tgt] = std::move(R);
      for (int i : raw[tgt].inds) hold[i].insert(tgt);
      alive[t] = 0;
      changed = true;
    }
  }
  for (size_t t = 0; t < raw.size(); ++t) {
    if (alive[t] && !raw[t].core) {
      int q = 0;
      for (; q < n; ++q)
        if (std::find(raw[t].inds.begin(), raw[t].inds.end(), wire[q]) != raw[t].inds.end()) break;
      raw[t].core = true;
      raw[t].px = xy[2 * q]; raw[t].py = xy[2 * q + 1];
    }
  }
  // R4: sum out indices held by a single tensor
  for (size_t t = 0; t < raw.size(); ++t) {
    if (!alive[t]) continue;
    std::vector<int> inds0 = raw[t].inds;
    for (int i : inds0) {
      if (outs.count(i) || !others(i, (int)t, -1).empty()) continue;
      Tensor& T = raw[t];
      std::set<int> keep;
      for (int j : T.inds)
        if (j != i) keep.insert(j);
      Tensor one;
      one.inds = {};
      one.data = {cplx(1, 0)};
      T = merge_into(T, one, keep, net.dims);
      hold[i].erase((int)t);
    }
  }
  for (size_t t = 0; t < raw.size(); ++t) {
    if (!alive[t]) continue;
    Tensor T = raw[t];
    // canonical axis order: output legs first, then ascending index id
    std::vector<int> order(T.inds.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = (int)k;
    std::sort(order.begin(), order.end(), [&](int x, int y) {
      bool ox = outs.count(T.inds[x]) > 0, oy = outs.count(T.inds[y]) > 0;
      if (ox != oy) return ox;
      return T.inds[x] < T.inds[y];
    });
    std::vector<int> ninds;
    for (int k : order) ninds.push_back(T.inds[k]);
    if (ninds != T.inds) {
      std::set<int> keep(ninds.begin(), ninds.end());
      Tensor one;
      one.data = {cplx(1, 0)};
      Tensor P;
      P.inds = ninds;
      // permute by re-merging with a scalar and reordering
      Tensor M = merge_into(T, one, keep, net.dims);  // same order as T
      std::vector<int64_t> st(T.inds.size());
      int64_t acc = 1;
      for (int k = (int)T.inds.size() - 1; k >= 0; --k) { st[k] = acc; acc *= net.dims[T.inds[k]]; }
      P.data.assign(M.data.size(), cplx(0, 0));
      std::vector<int> v(ninds.size(), 0);
      for (int64_t it = 0; it < acc; ++it) {
        int64_t r = it;
        for (int k = (int)ninds.size() - 1; k >= 0; --k) { v[k] = (int)(r % net.dims[ninds[k]]); r /= net.dims[ninds[k]]; }
        int64_t src = 0;
        for (size_t k = 0; k < ninds.size(); ++k) src += st[order[k]] * v[k];
        P.data[it] = M.data[src];
      }
      T.inds = ninds;
      T.data = std::move(P.data);
    }
    net.tensors.push_back(std::move(T));
  }
  net.out_owner.assign(n, -1);
  for (int q = 0; q < n; ++q)
    for (size_t t = 0; t < net.tensors.size(); ++t)
      if (std::find(net.tensors[t].inds.begin(), net.tensors[t].inds.end(), wire[q]) != net.tensors[t].inds.end()) {
        net.out_owner[q] = (int)t;
        break;
      }
  double rmin = INFINITY;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      double dx = xy[2 * i] - xy[2 * j], dy = xy[2 * i + 1] - xy[2 * j + 1];
      double d = std::sqrt(dx * dx + dy * dy);
      rmin = std::min(rmin, d);
    }
  if (!std::isfinite(rmin) || rmin <= 0) rmin = 1.0;
  net.l = ltab;
  net.r = rmin;
  net.radius = ltab / 4.0 + eps_frac * rmin;
  int F = 0;
  for (int f : fcount) F = std::max(F, f);
  net.F = F;
  double g = (ltab + rmin) / rmin;
  net.k_bound = std::max(1.0, (double)F * (g * g));
  return net;
}

}  // namespace tn
