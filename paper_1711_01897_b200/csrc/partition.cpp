// Bit-exact H-matrix partition on the host (hmatrix.py:105-211).
//
// Cluster tree: recursive longest-axis median bisection with a stable sort
// (hmatrix.py:122-137), nodes numbered in preorder, mid = start+(size+1)/2.
// Block tree: simultaneous descent, box admissibility
//   dist = |max(0, max(b_min - a_max, a_min - b_max))|,  adm iff dist > 0 and
//   min(diam_t, diam_s) <= eta * dist                     (hmatrix.py:66-69, 174-179)
// with children visited in (left, right) x (left, right) order
// (hmatrix.py:195-208).  np.linalg.norm of a 3-vector goes through BLAS ddot;
// norm_mode reproduces its float64 evaluation (see hbem_b200.h).
#include <algorithm>
#include <array>
#include <cmath>
#include <new>
#include <vector>

#include "../../include/hbem_b200.h"

namespace hb {
int set_error(int code, const char *fmt, ...);
void clear_error();
}  // namespace hb

struct hbem_tree {
  int64_t n = 0;
  std::vector<int64_t> perm;
  std::vector<std::array<int64_t, 5>> nodes;  // start, stop, level, left, right
  std::vector<std::array<double, 6>> bbox;    // min xyz, max xyz
};

struct hbem_blocks {
  std::vector<std::array<int64_t, 3>> leaves;
};

namespace {

inline double norm3(double x, double y, double z, int mode) {
  if (mode == 1) return std::sqrt(std::fma(z, z, std::fma(y, y, x * x)));
  volatile double xx = x * x, yy = y * y, zz = z * z;  // keep the numpy order
  return std::sqrt((xx + yy) + zz);
}

void build(hbem_tree &t, const double *pts, int64_t start, int64_t stop, int64_t level,
           int n_min, std::vector<std::pair<double, int64_t>> &scratch) {
  std::array<double, 6> bb;
  for (int c = 0; c < 3; ++c) {
    bb[c] = pts[3 * t.perm[start] + c];
    bb[3 + c] = bb[c];
  }
  for (int64_t i = start + 1; i < stop; ++i) {
    const double *p = pts + 3 * t.perm[i];
    for (int c = 0; c < 3; ++c) {
      if (p[c] < bb[c]) bb[c] = p[c];
      if (p[c] > bb[3 + c]) bb[3 + c] = p[c];
    }
  }
  const int64_t me = (int64_t)t.nodes.size();
  t.nodes.push_back({start, stop, level, -1, -1});
  t.bbox.push_back(bb);
  if (stop - start > n_min) {
    int axis = 0;
    double ext = bb[3] - bb[0];
    for (int c = 1; c < 3; ++c) {
      const double e = bb[3 + c] - bb[c];
      if (e > ext) {  // np.argmax: first maximum wins
        ext = e;
        axis = c;
      }
    }
    const int64_t n = stop - start;
    scratch.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t idx = t.perm[start + i];
      scratch[i] = {pts[3 * idx + axis], idx};
    }
    std::stable_sort(scratch.begin(), scratch.end(),
                     [](const std::pair<double, int64_t> &a,
                        const std::pair<double, int64_t> &b) { return a.first < b.first; });
    for (int64_t i = 0; i < n; ++i) t.perm[start + i] = scratch[i].second;
    const int64_t mid = start + (n + 1) / 2;
    build(t, pts, start, mid, level + 1, n_min, scratch);
    const int64_t left = me + 1;
    const int64_t right = (int64_t)t.nodes.size();
    build(t, pts, mid, stop, level + 1, n_min, scratch);
    t.nodes[me][3] = left;
    t.nodes[me][4] = right;
  }
}

}  // namespace

extern "C" {

int hbem_cluster_tree(const double *points, int64_t n, int32_t n_min, hbem_tree **out) {
  hb::clear_error();
  if (!points || !out) return hb::set_error(HBEM_ERR_ARG, "null argument");
  if (n < 1) return hb::set_error(HBEM_ERR_CONFIG, "cluster tree needs at least one DOF");
  if (n_min < 1) return hb::set_error(HBEM_ERR_CONFIG, "n_min must be >= 1, got %d", n_min);
  hbem_tree *t = new (std::nothrow) hbem_tree();
  if (!t) return hb::set_error(HBEM_ERR_CAPACITY, "out of host memory");
  t->n = n;
  t->perm.resize(n);
  for (int64_t i = 0; i < n; ++i) t->perm[i] = i;
  t->nodes.reserve(2 * (n / std::max<int64_t>(1, n_min / 2)) + 2);
  std::vector<std::pair<double, int64_t>> scratch;
  build(*t, points, 0, n, 0, n_min, scratch);
  *out = t;
  return HBEM_OK;
}

int hbem_tree_size(const hbem_tree *t, int64_t *n_points, int64_t *n_nodes) {
  if (!t) return hb::set_error(HBEM_ERR_ARG, "null tree");
  if (n_points) *n_points = t->n;
  if (n_nodes) *n_nodes = (int64_t)t->nodes.size();
  return HBEM_OK;
}

int hbem_tree_copy(const hbem_tree *t, int64_t *perm, int64_t *nodes, double *bbox) {
  if (!t) return hb::set_error(HBEM_ERR_ARG, "null tree");
  if (perm) std::copy(t->perm.begin(), t->perm.end(), perm);
  for (size_t i = 0; i < t->nodes.size(); ++i) {
    if (nodes)
      for (int k = 0; k < 5; ++k) nodes[5 * i + k] = t->nodes[i][k];
    if (bbox)
      for (int k = 0; k < 6; ++k) bbox[6 * i + k] = t->bbox[i][k];
  }
  return HBEM_OK;
}

int hbem_tree_destroy(hbem_tree *t) {
  delete t;
  return HBEM_OK;
}

int hbem_block_tree(const hbem_tree *rows, const hbem_tree *cols, double eta, int32_t norm_mode,
                    hbem_blocks **out) {
  hb::clear_error();
  if (!rows || !cols || !out) return hb::set_error(HBEM_ERR_ARG, "null argument");
  if (eta < 0.0) return hb::set_error(HBEM_ERR_CONFIG, "eta must be >= 0, got %g", eta);
  auto diam = [&](const hbem_tree *t) {
    std::vector<double> d(t->nodes.size());
    for (size_t i = 0; i < d.size(); ++i) {
      const auto &b = t->bbox[i];
      d[i] = norm3(b[3] - b[0], b[4] - b[1], b[5] - b[2], norm_mode);
    }
    return d;
  };
  const std::vector<double> dr = diam(rows);
  const std::vector<double> dc = (rows == cols) ? dr : diam(cols);
  hbem_blocks *B = new (std::nothrow) hbem_blocks();
  if (!B) return hb::set_error(HBEM_ERR_CAPACITY, "out of host memory");
  std::vector<std::pair<int64_t, int64_t>> stack;
  stack.push_back({0, 0});
  while (!stack.empty()) {
    auto [ti, si] = stack.back();
    stack.pop_back();
    const auto &a = rows->bbox[ti];
    const auto &b = cols->bbox[si];
    double g[3];
    for (int c = 0; c < 3; ++c) {
      const double u = b[c] - a[3 + c];  // b_min - a_max
      const double v = a[c] - b[3 + c];  // a_min - b_max
      const double w = u > v ? u : v;    // np.maximum (no NaN here)
      g[c] = w > 0.0 ? w : 0.0;
    }
    const double dist = norm3(g[0], g[1], g[2], norm_mode);
    bool adm = false;
    if (dist > 0.0) adm = std::min(dr[ti], dc[si]) <= eta * dist;
    const auto &tn = rows->nodes[ti];
    const auto &sn = cols->nodes[si];
    const bool tleaf = tn[3] < 0, sleaf = sn[3] < 0;
    if (adm) {
      B->leaves.push_back({ti, si, 1});
      continue;
    }
    if (tleaf && sleaf) {
      B->leaves.push_back({ti, si, 0});
      continue;
    }
    int64_t tk[2], sk[2];
    int nt = 0, ns = 0;
    if (tleaf) tk[nt++] = ti;
    else { tk[nt++] = tn[3]; tk[nt++] = tn[4]; }
    if (sleaf) sk[ns++] = si;
    else { sk[ns++] = sn[3]; sk[ns++] = sn[4]; }
    // push in reverse so (tk[0], sk[0]) is processed first
    for (int i = nt - 1; i >= 0; --i)
      for (int j = ns - 1; j >= 0; --j) stack.push_back({tk[i], sk[j]});
  }
  *out = B;
  return HBEM_OK;
}

int hbem_blocks_size(const hbem_blocks *b, int64_t *n_leaves) {
  if (!b) return hb::set_error(HBEM_ERR_ARG, "null blocks");
  *n_leaves = (int64_t)b->leaves.size();
  return HBEM_OK;
}

int hbem_blocks_copy(const hbem_blocks *b, int64_t *leaves) {
  if (!b) return hb::set_error(HBEM_ERR_ARG, "null blocks");
  for (size_t i = 0; i < b->leaves.size(); ++i)
    for (int k = 0; k < 3; ++k) leaves[3 * i + k] = b->leaves[i][k];
  return HBEM_OK;
}

int hbem_blocks_destroy(hbem_blocks *b) {
  delete b;
  return HBEM_OK;
}

}  // extern "C"
