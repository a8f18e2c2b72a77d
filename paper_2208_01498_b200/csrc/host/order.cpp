// Separator-based contraction order: SM Algorithm 1 applied
// recursively (Theorem 1 proof l.79-80, Fig. 2), greedy leaf planner (SM l.217),
// and index slicing (outlook l.178).  Readings R5-R11: DESIGN.md.
// Compiled with -ffp-contract=off: every floating-point decision is a plain
// IEEE-754 double operation in a fixed order.
#include <algorithm>
#include <atomic>
#include <exception>
#include <thread>
#include <cstdlib>
#include <cmath>
#include <map>
#include <numeric>
#include <stdexcept>
#include <tuple>
#include <unordered_map>

#include "tn_host.hpp"

namespace tn {

uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
Stream::Stream(uint64_t seed, uint64_t sid) : key(splitmix64(seed ^ splitmix64(sid))) {}
uint64_t Stream::u64() { return splitmix64(key + ctr++); }
double Stream::uniform() { return (double)(u64() >> 11) * (1.0 / 9007199254740992.0); }
uint64_t child_stream(uint64_t sid, int side) { return splitmix64(sid * 2 + (uint64_t)side + 1); }

namespace {

constexpr double BOX = 2.0, LP_TOL = 1e-9, PIV_TOL = 1e-12, SIDE_TOL = 1e-12;

bool inv4(const double B[4][4], double out[4][4]) {
  double M[4][8];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 8; ++c) M[r][c] = c < 4 ? B[r][c] : (c - 4 == r ? 1.0 : 0.0);
  for (int col = 0; col < 4; ++col) {
    int piv = col;
    double best = std::fabs(M[col][col]);
    for (int r = col + 1; r < 4; ++r)
      if (std::fabs(M[r][col]) > best) { best = std::fabs(M[r][col]); piv = r; }
    if (best == 0.0) return false;
    for (int c = 0; c < 8; ++c) std::swap(M[col][c], M[piv][c]);
    double p = M[col][col];
    for (int c = 0; c < 8; ++c) M[col][c] = M[col][c] / p;
    for (int r = 0; r < 4; ++r) {
      if (r == col) continue;
      double f = M[r][col];
      if (f != 0.0)
        for (int c = 0; c < 8; ++c) M[r][c] = M[r][c] - f * M[col][c];
    }
  }
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) out[r][c] = M[r][4 + c];
  return true;
}

// max t s.t. A x <= b (x = c0,c1,c2,t free), dual revised simplex, Bland's rule (R5)
bool lp_centerpoint(const std::vector<double>& A0, const std::vector<double>& A1,
                    const std::vector<double>& A2, const std::vector<double>& A3,
                    const std::vector<double>& b, double pi[4]) {
  int basis[4] = {0, 1, 2, 6};
  bool have = false;
  size_t m = b.size();
  for (int it = 0; it < 500; ++it) {
    double B[4][4], Bi[4][4];
    for (int c = 0; c < 4; ++c) {
      int j = basis[c];
      B[0][c] = A0[j]; B[1][c] = A1[j]; B[2][c] = A2[j]; B[3][c] = A3[j];
    }
    if (!inv4(B, Bi)) break;
    double cB[4];
    for (int r = 0; r < 4; ++r) cB[r] = b[basis[r]];
    for (int i = 0; i < 4; ++i) {
      double acc = cB[0] * Bi[0][i];
      for (int r = 1; r < 4; ++r) acc = acc + cB[r] * Bi[r][i];
      pi[i] = acc;
    }
    have = true;
    long e = -1;
    for (size_t j = 0; j < m; ++j) {
      if ((int)j == basis[0] || (int)j == basis[1] || (int)j == basis[2] || (int)j == basis[3]) continue;
      double d = b[j] - (((pi[0] * A0[j] + pi[1] * A1[j]) + pi[2] * A2[j]) + pi[3] * A3[j]);
      if (d < -LP_TOL) { e = (long)j; break; }
    }
    if (e < 0) break;
    double Ae[4] = {A0[e], A1[e], A2[e], A3[e]};
    int best_r = -1;
    double best_t = 0.0;
    for (int r = 0; r < 4; ++r) {
      double w = Bi[r][0] * Ae[0];
      for (int i = 1; i < 4; ++i) w = w + Bi[r][i] * Ae[i];
      if (w > PIV_TOL) {
        double th = Bi[r][3] / w;
        if (best_r < 0 || th < best_t || (th == best_t && basis[r] < basis[best_r])) { best_r = r; best_t = th; }
      }
    }
    if (best_r < 0) break;
    basis[best_r] = (int)e;
  }
  return have;
}

struct Vec3 { double x, y, z; };

Vec3 centerpoint(const std::vector<double>& P0, const std::vector<double>& P1,
                 const std::vector<double>& P2, Stream& rng, int a_max) {
  int s = (int)P0.size();
  int a = std::min(s, a_max);
  std::vector<int> perm(s);
  std::iota(perm.begin(), perm.end(), 0);
  for (int i = 0; i < a; ++i) {
    int j = i + (int)rng.below((uint64_t)(s - i));
    std::swap(perm[i], perm[j]);
  }
  std::vector<double> X(a), Y(a), Z(a);
  for (int i = 0; i < a; ++i) { X[i] = P0[perm[i]]; Y[i] = P1[perm[i]]; Z[i] = P2[perm[i]]; }
  std::vector<double> r0 = {1, 0, 0, -1, 0, 0, 0}, r1 = {0, 1, 0, 0, -1, 0, 0}, r2 = {0, 0, 1, 0, 0, -1, 0},
                      r3 = {0, 0, 0, 0, 0, 0, 1}, rb = {BOX, BOX, BOX, BOX, BOX, BOX, 1.0};
  if (a >= 3) {
    for (int i = 0; i < a; ++i)
      for (int j = i + 1; j < a; ++j)
        for (int k = j + 1; k < a; ++k) {
          double ux = X[j] - X[i], uy = Y[j] - Y[i], uz = Z[j] - Z[i];
          double vx = X[k] - X[i], vy = Y[k] - Y[i], vz = Z[k] - Z[i];
          double nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
          double nn2 = (nx * nx + ny * ny) + nz * nz;
          if (!(nn2 > 1e-24)) continue;
          double nrm = std::sqrt(nn2);
          nx = nx / nrm; ny = ny / nrm; nz = nz / nrm;
          double off = (nx * X[i] + ny * Y[i]) + nz * Z[i];
          int above = 0, below = 0;
          for (int l = 0; l < a; ++l) {
            double sd = ((nx * X[l] + ny * Y[l]) + nz * Z[l]) - off;
            if (sd > SIDE_TOL) ++above;
            if (sd < -SIDE_TOL) ++below;
          }
          if (above * 4 < a) { r0.push_back(nx); r1.push_back(ny); r2.push_back(nz); r3.push_back(1.0); rb.push_back(off); }
          if (below * 4 < a) { r0.push_back(-nx); r1.push_back(-ny); r2.push_back(-nz); r3.push_back(1.0); rb.push_back(-off); }
        }
  }
  double pi[4];
  if (!lp_centerpoint(r0, r1, r2, r3, rb, pi)) return {0, 0, 0};
  Vec3 c{pi[0], pi[1], pi[2]};
  double nc = std::sqrt((c.x * c.x + c.y * c.y) + c.z * c.z);
  if (nc > 0.999999) {
    double f = 0.999999 / nc;
    c = {c.x * f, c.y * f, c.z * f};
  }
  return c;
}

void rotation_to_pole(Vec3 c, double R[3][3], double& nc) {
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) R[r][k] = r == k ? 1.0 : 0.0;
  nc = std::sqrt((c.x * c.x + c.y * c.y) + c.z * c.z);
  if (nc < 1e-12) { nc = 0.0; return; }
  double w[3] = {c.x / nc, c.y / nc, c.z / nc - 1.0};
  double ww = (w[0] * w[0] + w[1] * w[1]) + w[2] * w[2];
  if (ww < 1e-24) return;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) R[r][k] = (r == k ? 1.0 : 0.0) - (2.0 * w[r] * w[k]) / ww;
}

Vec3 random_normal(Stream& rng) {
  for (;;) {
    double u0 = 2.0 * rng.uniform() - 1.0;
    double u1 = 2.0 * rng.uniform() - 1.0;
    double u2 = 2.0 * rng.uniform() - 1.0;
    double r2 = (u0 * u0 + u1 * u1) + u2 * u2;
    if (1e-6 < r2 && r2 <= 1.0) {
      double r = std::sqrt(r2);
      return {u0 / r, u1 / r, u2 / r};
    }
  }
}

struct Sep {
  bool ok = false, circle = true;
  double cx = 0, cy = 0, rho = 0, b0 = 0, b1 = 0, C0 = 0, nb = 0;
};

Sep separator_circle(Vec3 u, const double R[3][3], double alpha) {
  double a2 = alpha * alpha;
  double n[3] = {alpha * u.x, alpha * u.y, (u.z * (1.0 + a2)) / 2.0};
  double h = (u.z * (1.0 - a2)) / 2.0;
  double m[3];
  for (int i = 0; i < 3; ++i) m[i] = (R[0][i] * n[0] + R[1][i] * n[1]) + R[2][i] * n[2];
  double A = m[2] - h, b0 = m[0], b1 = m[1], C0 = m[2] + h;
  double scale = ((std::fabs(A) + std::fabs(b0)) + std::fabs(b1)) + std::fabs(C0);
  Sep s;
  if (std::fabs(A) > 1e-12 * scale) {
    s.cx = -b0 / A;
    s.cy = -b1 / A;
    double rho2 = (b0 * b0 + b1 * b1) / (A * A) + C0 / A;
    if (!(rho2 > 0.0)) return s;
    s.rho = std::sqrt(rho2);
    s.ok = true;
    return s;
  }
  double nb = std::sqrt(b0 * b0 + b1 * b1);
  if (nb == 0.0) return s;
  s.circle = false; s.b0 = b0; s.b1 = b1; s.C0 = C0; s.nb = nb; s.ok = true;
  return s;
}

struct Node {
  int nid;
  std::map<int, int> counts;  // index -> original holders inside
};

struct Ctx {
  const Network& net;
  uint64_t seed;
  OrderParams p;
  std::vector<std::vector<int>> inds;
  std::vector<int> l2;
  std::vector<double> PX, PY;
  std::vector<int> total;
  std::vector<std::pair<int, int>> steps;
  int n_leaves;
  int medians = 0;
  Ctx(const Network& n, uint64_t s, const OrderParams& pp) : net(n), seed(s), p(pp) {
    int T = (int)n.tensors.size();
    n_leaves = T;
    l2.resize(n.dims.size());
    for (size_t i = 0; i < n.dims.size(); ++i) l2[i] = n.log2dim((int)i);
    total.assign(n.dims.size(), 0);
    for (int t = 0; t < T; ++t) {
      inds.push_back(n.closed_inds(t));
      PX.push_back(n.tensors[t].px);
      PY.push_back(n.tensors[t].py);
      for (int i : inds.back()) total[i]++;
    }
  }
};

Node merge(Ctx& c, const Node& A, const Node& B) {
  Node R;
  R.counts = A.counts;
  for (auto& kv : B.counts) R.counts[kv.first] += kv.second;
  for (auto it = R.counts.begin(); it != R.counts.end();)
    if (it->second >= c.total[it->first]) it = R.counts.erase(it); else ++it;
  R.nid = c.n_leaves + (int)c.steps.size();
  c.steps.push_back({A.nid, B.nid});
  return R;
}

Node greedy_leaf(Ctx& c, const std::vector<int>& ids) {
  std::vector<Node> cur;
  for (int t : ids) {
    Node nd;
    nd.nid = t;
    for (int i : c.inds[t]) nd.counts[i] = 1;
    cur.push_back(nd);
  }
  while (cur.size() > 1) {
    bool share_any = false;
    std::vector<std::tuple<bool, int, int>> cands;
    for (size_t x = 0; x < cur.size(); ++x)
      for (size_t y = x + 1; y < cur.size(); ++y) {
        bool sh = false;
        for (auto& kv : cur[x].counts)
          if (cur[y].counts.count(kv.first)) { sh = true; break; }
        cands.emplace_back(sh, (int)x, (int)y);
        share_any = share_any || sh;
      }
    bool have = false;
    std::tuple<int, int, int, int> bk;
    int bx = -1, by = -1;
    for (auto& [sh, x, y] : cands) {
      if (share_any && !sh) continue;
      const Node &A = cur[x], &B = cur[y];
      int cost = 0, res = 0;
      for (auto& kv : A.counts) {
        cost += c.l2[kv.first];
        auto it = B.counts.find(kv.first);
        int cnt = kv.second + (it == B.counts.end() ? 0 : it->second);
        if (cnt < c.total[kv.first]) res += c.l2[kv.first];
      }
      for (auto& kv : B.counts) {
        if (A.counts.count(kv.first)) continue;
        cost += c.l2[kv.first];
        if (kv.second < c.total[kv.first]) res += c.l2[kv.first];
      }
      auto key = std::make_tuple(cost, res, std::min(A.nid, B.nid), std::max(A.nid, B.nid));
      if (!have || key < bk) { have = true; bk = key; bx = x; by = y; }
    }
    Node A = cur[bx], B = cur[by];
    if (A.nid > B.nid) std::swap(A, B);
    Node nd = merge(c, A, B);
    std::vector<Node> nxt;
    for (size_t j = 0; j < cur.size(); ++j)
      if ((int)j != bx && (int)j != by) nxt.push_back(cur[j]);
    nxt.push_back(nd);
    cur.swap(nxt);
  }
  return cur[0];
}

// Theorem 1 proof boundary assignment (R7); key = (max child open bits, cut) (R6)
void assign_boundary(Ctx& c, const std::vector<int>& ids, const std::vector<int>& lab,
                     std::vector<int>& E, std::vector<int>& I, std::pair<int, int>& key) {
  std::unordered_map<int, int> cE, cI;
  std::vector<int> O;
  E.clear(); I.clear();
  for (size_t k = 0; k < ids.size(); ++k) (lab[k] == 0 ? O : lab[k] == 1 ? E : I).push_back(ids[k]);
  for (int t : E) for (int i : c.inds[t]) cE[i]++;
  for (int t : I) for (int i : c.inds[t]) cI[i]++;
  for (int t : O) {
    int wE = 0, wI = 0;
    for (int i : c.inds[t]) {
      auto a = cE.find(i);
      if (a != cE.end() && a->second > 0) wE += c.l2[i];
      auto b = cI.find(i);
      if (b != cI.end() && b->second > 0) wI += c.l2[i];
    }
    int side;
    if (wE > wI) side = 1;
    else if (wI > wE) side = 2;
    else side = E.size() <= I.size() ? 1 : 2;
    if (side == 1) { E.push_back(t); for (int i : c.inds[t]) cE[i]++; }
    else { I.push_back(t); for (int i : c.inds[t]) cI[i]++; }
  }
  int cut = 0, oE = 0, oI = 0;
  for (auto& kv : cE) {
    auto b = cI.find(kv.first);
    if (b != cI.end() && b->second > 0) cut += c.l2[kv.first];
    if (kv.second < c.total[kv.first]) oE += c.l2[kv.first];
  }
  for (auto& kv : cI)
    if (kv.second < c.total[kv.first]) oI += c.l2[kv.first];
  std::sort(E.begin(), E.end());
  std::sort(I.begin(), I.end());
  key = {std::max(oE, oI), cut};
}

bool find_separator(Ctx& c, const std::vector<int>& ids, Stream& rng, std::vector<int>& bE,
                    std::vector<int>& bI) {
  int s = (int)ids.size();
  std::vector<double> PX(s), PY(s), P0(s), P1(s), P2(s);
  for (int k = 0; k < s; ++k) {
    PX[k] = c.PX[ids[k]]; PY[k] = c.PY[ids[k]];
    double ss = PX[k] * PX[k] + PY[k] * PY[k];
    double den = ss + 1.0;
    P0[k] = (2.0 * PX[k]) / den; P1[k] = (2.0 * PY[k]) / den; P2[k] = (ss - 1.0) / den;
  }
  double rad = c.net.radius, kb = c.net.k_bound;
  bool have = false;
  std::pair<int, int> bkey;
  int n_ok = 0;
  std::vector<int> lab(s), E, I;
  for (int round = 0; round < 2; ++round) {
    Vec3 cp = centerpoint(P0, P1, P2, rng, c.p.a_max);
    double R[3][3], nc;
    rotation_to_pole(cp, R, nc);
    double alpha = std::sqrt((1.0 - nc) / (1.0 + nc));
    for (int tr = 0; tr < c.p.max_tries; ++tr) {
      Vec3 u = random_normal(rng);
      Sep sp = separator_circle(u, R, alpha);
      if (!sp.ok) continue;
      int nO = 0, nE = 0, nI = 0;
      for (int k = 0; k < s; ++k) {
        int l = 0;
        if (sp.circle) {
          double dx = PX[k] - sp.cx, dy = PY[k] - sp.cy;
          double dist = std::sqrt(dx * dx + dy * dy);
          if (dist + rad < sp.rho) l = 2;
          if (dist - rad > sp.rho) l = 1;
        } else {
          double sd = (2.0 * (sp.b0 * PX[k] + sp.b1 * PY[k]) - sp.C0) / (2.0 * sp.nb);
          if (sd > rad) l = 1;
          if (sd < -rad) l = 2;
        }
        lab[k] = l;
        (l == 0 ? nO : l == 1 ? nE : nI)++;
      }
      // Eq. (1) with c_2 = 2, Eq. (2) with (d+1)/(d+2) = 3/4
      if (!((double)nO * (double)nO <= ((2.0 * 2.0) * kb) * (double)s)) continue;
      if (4 * nE > 3 * s || 4 * nI > 3 * s) continue;
      std::pair<int, int> key;
      assign_boundary(c, ids, lab, E, I, key);
      if (E.empty() || I.empty()) continue;
      ++n_ok;
      if (!have || key < bkey) { have = true; bkey = key; bE = E; bI = I; }
      if (n_ok >= c.p.n_valid) break;
    }
    if (have) break;
  }
  return have;
}

void median_split(Ctx& c, const std::vector<int>& ids, std::vector<int>& E, std::vector<int>& I) {
  double mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY;
  for (int t : ids) {
    mnx = std::min(mnx, c.PX[t]); mxx = std::max(mxx, c.PX[t]);
    mny = std::min(mny, c.PY[t]); mxy = std::max(mxy, c.PY[t]);
  }
  bool use_x = (mxx - mnx) >= (mxy - mny);
  std::vector<int> o(ids);
  std::sort(o.begin(), o.end(), [&](int a, int b) {
    double ka = use_x ? c.PX[a] : c.PY[a], kb = use_x ? c.PX[b] : c.PY[b];
    if (ka != kb) return ka < kb;
    return a < b;
  });
  size_t h = ids.size() / 2;
  E.assign(o.begin(), o.begin() + h);
  I.assign(o.begin() + h, o.end());
  std::sort(E.begin(), E.end());
  std::sort(I.begin(), I.end());
}

Node build(Ctx& c, const std::vector<int>& ids, uint64_t sid) {
  if ((int)ids.size() <= c.p.leaf_size) return greedy_leaf(c, ids);
  Stream rng(c.seed, sid);
  std::vector<int> E, I;
  if (!find_separator(c, ids, rng, E, I)) {
    median_split(c, ids, E, I);
    c.medians++;
  }
  Node nE = build(c, E, child_stream(sid, 0));
  Node nI = build(c, I, child_stream(sid, 1));
  return merge(c, nE, nI);
}

void costs(const Network& net, const std::vector<std::pair<int, int>>& steps, std::vector<int>& m,
           std::vector<int>& res) {
  int n = (int)net.tensors.size();
  std::vector<int> total(net.dims.size(), 0);
  std::unordered_map<int, std::map<int, int>> nodes;
  for (int t = 0; t < n; ++t) {
    for (int i : net.closed_inds(t)) { nodes[t][i] = 1; total[i]++; }
    if (!nodes.count(t)) nodes[t] = {};
  }
  m.clear(); res.clear();
  for (size_t k = 0; k < steps.size(); ++k) {
    auto A = std::move(nodes[steps[k].first]);
    auto B = std::move(nodes[steps[k].second]);
    nodes.erase(steps[k].first); nodes.erase(steps[k].second);
    std::map<int, int> cnt = A;
    for (auto& kv : B) cnt[kv.first] += kv.second;
    int mm = 0, rr = 0;
    std::map<int, int> kept;
    for (auto& kv : cnt) {
      mm += net.log2dim(kv.first);
      if (kv.second < total[kv.first]) { kept[kv.first] = kv.second; rr += net.log2dim(kv.first); }
    }
    nodes[n + (int)k] = kept;
    m.push_back(mm); res.push_back(rr);
  }
}

}  // namespace

std::vector<std::vector<int>> kept_per_step(const Network& net, const std::vector<std::pair<int, int>>& steps) {
  int n = (int)net.tensors.size();
  std::vector<int> total(net.dims.size(), 0);
  std::unordered_map<int, std::map<int, int>> nodes;
  for (int t = 0; t < n; ++t) {
    nodes[t] = {};
    for (int i : net.closed_inds(t)) { nodes[t][i] = 1; total[i]++; }
  }
  std::vector<std::vector<int>> out;
  for (size_t k = 0; k < steps.size(); ++k) {
    auto A = std::move(nodes[steps[k].first]);
    auto B = std::move(nodes[steps[k].second]);
    nodes.erase(steps[k].first); nodes.erase(steps[k].second);
    std::map<int, int> kept = A;
    for (auto& kv : B) kept[kv.first] += kv.second;
    std::vector<int> ks;
    for (auto it = kept.begin(); it != kept.end();) {
      if (it->second >= total[it->first]) it = kept.erase(it);
      else { ks.push_back(it->first); ++it; }
    }
    nodes[n + (int)k] = kept;
    out.push_back(ks);
  }
  return out;
}

std::vector<int> choose_slices(const Network& net, const std::vector<std::pair<int, int>>& steps,
                               int max_log2_size) {
  int n = (int)net.tensors.size();
  std::vector<int> l2(net.dims.size());
  for (size_t i = 0; i < net.dims.size(); ++i) l2[i] = net.log2dim((int)i);
  std::vector<std::vector<int>> tensors;
  for (int t = 0; t < n; ++t) {
    auto ii = net.closed_inds(t);
    std::sort(ii.begin(), ii.end());
    tensors.push_back(ii);
  }
  std::vector<int> total(net.dims.size(), 0);
  std::unordered_map<int, std::map<int, int>> nodes;
  for (int t = 0; t < n; ++t) {
    nodes[t] = {};
    for (int i : net.closed_inds(t)) { nodes[t][i] = 1; total[i]++; }
  }
  std::vector<std::vector<int>> unions;
  std::vector<int> sm;
  for (size_t k = 0; k < steps.size(); ++k) {
    auto A = std::move(nodes[steps[k].first]);
    auto B = std::move(nodes[steps[k].second]);
    nodes.erase(steps[k].first); nodes.erase(steps[k].second);
    std::map<int, int> cnt = A;
    for (auto& kv : B) cnt[kv.first] += kv.second;
    std::vector<int> u, kk;
    std::map<int, int> kept;
    int m = 0;
    for (auto& kv : cnt) {
      u.push_back(kv.first);
      m += l2[kv.first];
      if (kv.second < total[kv.first]) { kept[kv.first] = kv.second; kk.push_back(kv.first); }
    }
    nodes[n + (int)k] = kept;
    unions.push_back(u);
    sm.push_back(m);
    tensors.push_back(kk);
  }
  std::vector<char> sl(net.dims.size(), 0);
  auto bits = [&](const std::vector<int>& ii) {
    int b = 0;
    for (int i : ii) if (!sl[i]) b += l2[i];
    return b;
  };
  std::vector<int> out;
  for (;;) {
    int big = 0;
    for (auto& ii : tensors) big = std::max(big, bits(ii));
    if (big <= max_log2_size) break;
    std::vector<int> cands;
    for (auto& ii : tensors)
      if (bits(ii) == big)
        for (int i : ii) if (!sl[i]) cands.push_back(i);
    std::sort(cands.begin(), cands.end());
    cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
    int sb = 0;
    for (int i : out) sb += l2[i];
    bool have = false;
    double bw = 0;
    int bc = -1;
    for (int cnd : cands) {
      double w = 0.0;
      for (size_t k = 0; k < unions.size(); ++k) {
        int s = 0;
        for (int i : unions[k]) if (sl[i] || i == cnd) s += l2[i];
        w = w + std::ldexp(1.0, sm[k] - s);
      }
      w = w * std::ldexp(1.0, sb + l2[cnd]);
      if (!have || w < bw) { have = true; bw = w; bc = cnd; }
    }
    if (bc < 0) break;
    sl[bc] = 1;
    out.push_back(bc);
  }
  std::sort(out.begin(), out.end());
  return out;
}

// Eq. (3) work of all slices, W = 2^{sum sliced bits} * sum_k 2^{m_k - sliced bits of
// step k} (left to right, doubles) -- the quantity the greedy slicer minimises (R11).
double sliced_work(const Network& net, const std::vector<std::pair<int, int>>& steps, const std::vector<int>& slices) {
  const int n = (int)net.tensors.size();
  std::vector<int> l2(net.dims.size());
  for (size_t i = 0; i < net.dims.size(); ++i) l2[i] = net.log2dim((int)i);
  std::vector<char> sl(net.dims.size(), 0);
  int sb = 0;
  for (int i : slices) { sl[i] = 1; sb += l2[i]; }
  std::vector<int> total(net.dims.size(), 0);
  std::unordered_map<int, std::map<int, int>> nodes;
  for (int t = 0; t < n; ++t) {
    nodes[t] = {};
    for (int i : net.closed_inds(t)) { nodes[t][i] = 1; total[i]++; }
  }
  double w = 0.0;
  for (size_t k = 0; k < steps.size(); ++k) {
    auto A = std::move(nodes[steps[k].first]);
    auto B = std::move(nodes[steps[k].second]);
    nodes.erase(steps[k].first); nodes.erase(steps[k].second);
    std::map<int, int> cnt = A;
    for (auto& kv : B) cnt[kv.first] += kv.second;
    std::map<int, int> kept;
    int m = 0, s = 0;
    for (auto& kv : cnt) {
      m += l2[kv.first];
      if (sl[kv.first]) s += l2[kv.first];
      if (kv.second < total[kv.first]) kept[kv.first] = kv.second;
    }
    nodes[n + (int)k] = kept;
    w = w + std::ldexp(1.0, m - s);
  }
  return w * std::ldexp(1.0, sb);
}

Order find_order(const Network& net, uint64_t seed, const OrderParams& p) {
  // R10: the randomized hierarchy is built n_seeds times; keep the one with the smallest
  // Eq. (3) total -- of all slices when a slicing target is set (the slicer's overhead
  // differs by orders of magnitude between hierarchies of similar unsliced cost)
  // the hierarchies are independent (own root streams): built on host threads, then the
  // first one with the least work is kept -- the same choice as a serial loop
  std::vector<int> ids(net.tensors.size());
  std::iota(ids.begin(), ids.end(), 0);
  const int R = std::max(1, p.n_seeds);
  std::vector<Order> cand(R);
  std::vector<double> work(R, 0.0);
  auto one = [&](int r) {
    Ctx c(net, seed, p);
    if (!ids.empty()) build(c, ids, (uint64_t)(1 + r));
    Order& o = cand[r];
    costs(net, c.steps, o.step_m, o.step_res);
    double tot = 0.0;
    for (int mm : o.step_m) tot = tot + std::ldexp(1.0, mm + 1);
    o.total_2M = tot;
    o.median_fallbacks = c.medians;
    o.steps = std::move(c.steps);
    work[r] = tot;
    if (p.max_log2_size > 0) {
      o.slices = choose_slices(net, o.steps, p.max_log2_size);
      work[r] = sliced_work(net, o.steps, o.slices);
    }
  };
  // host threads: all cores, or TN_ORDER_THREADS (bench.py sets it to the cores per rank
  // when several ranks share a host); the choice does not depend on the thread count
  int hw = (int)std::thread::hardware_concurrency();
  if (const char* e = std::getenv("TN_ORDER_THREADS")) hw = std::atoi(e);
  const int T = std::max(1, std::min<int>(R, hw));
  std::atomic<int> next{0};
  std::vector<std::exception_ptr> err(T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      try {
        for (int r = next++; r < R; r = next++) one(r);
      } catch (...) {
        err[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : err) if (e) std::rethrow_exception(e);
  int best = 0;
  for (int r = 1; r < R; ++r) if (work[r] < work[best]) best = r;
  return std::move(cand[best]);
}

// An order given as explicit steps and sliced indices (tn_order_import: the order another
// rank found), validated by the caller as a full binary tree over the network's tensors;
// the per-step costs are recomputed here (the same Eq. (3) counts find_order keeps).
Order import_order(const Network& net, std::vector<std::pair<int, int>> steps, std::vector<int> slices,
                   int median_fallbacks) {
  Order o;
  costs(net, steps, o.step_m, o.step_res);
  double tot = 0.0;
  for (int mm : o.step_m) tot = tot + std::ldexp(1.0, mm + 1);
  o.total_2M = tot;
  o.median_fallbacks = median_fallbacks;
  o.steps = std::move(steps);
  o.slices = std::move(slices);
  return o;
}

}  // namespace tn
