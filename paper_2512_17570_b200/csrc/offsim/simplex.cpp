// Dense LP solver behind the planner (reference API: proj/include/offsim/
// simplex.hpp, solve_lp; algorithm restated, not translated, from
// proj/src/simplex.cpp:59-155): minimise c.x subject to A x <= b, x >= 0.
//
// Tableau form.  Row i becomes an equality with slack s_i; a row whose right-
// hand side is negative is negated (its slack coefficient becomes -1) and
// gets an artificial variable.  Phase 1 minimises the sum of artificials;
// phase 2 the objective over the remaining columns.  Pivots follow Bland's
// rule (smallest entering index, smallest basic index on ratio ties), which
// cannot cycle.  Each row is equilibrated by its largest |coefficient| first:
// the planner mixes byte counts (~1e10) with fractions in one system.
#include <algorithm>
#include <cmath>
#include <vector>

#include "offsim/offsim.hpp"

namespace offsim {

namespace {

constexpr double kEps = 1e-9;

struct Tableau {
  int rows = 0, cols = 0;          // constraint rows; columns excluding rhs
  std::vector<double> t;           // (rows + 1) x (cols + 1); last row = objective
  std::vector<int> basis;          // basic column of each constraint row
  double& at(int r, int c) { return t[static_cast<size_t>(r) * (cols + 1) + c]; }
  double& rhs(int r) { return at(r, cols); }

  void pivot(int pr, int pc) {
    const double inv = 1.0 / at(pr, pc);
    for (int c = 0; c <= cols; ++c) at(pr, c) *= inv;
    for (int r = 0; r <= rows; ++r) {
      if (r == pr) continue;
      const double f = at(r, pc);
      if (f == 0.0) continue;
      for (int c = 0; c <= cols; ++c) at(r, c) -= f * at(pr, c);
    }
    basis[static_cast<size_t>(pr)] = pc;
  }

  // Minimises the objective row over columns [0, active); false = unbounded.
  bool optimise(int active) {
    for (;;) {
      int pc = -1;
      for (int c = 0; c < active; ++c)
        if (at(rows, c) < -kEps) {
          pc = c;
          break;
        }
      if (pc < 0) return true;
      int pr = -1;
      double best = 0.0;
      for (int r = 0; r < rows; ++r) {
        const double a = at(r, pc);
        if (a <= kEps) continue;
        const double ratio = rhs(r) / a;
        if (pr < 0 || ratio < best - kEps ||
            (std::fabs(ratio - best) <= kEps && basis[static_cast<size_t>(r)] < basis[static_cast<size_t>(pr)])) {
          pr = r;
          best = ratio;
        }
      }
      if (pr < 0) return false;
      pivot(pr, pc);
    }
  }
};

}  // namespace

LpResult solve_lp(const std::vector<std::vector<double>>& A, const std::vector<double>& b,
                  const std::vector<double>& c) {
  const int m = static_cast<int>(A.size()), n = static_cast<int>(c.size());
  if (static_cast<int>(b.size()) != m) throw ValidationError("solve_lp: A and b row counts differ");
  for (const auto& row : A)
    if (static_cast<int>(row.size()) != n) throw ValidationError("solve_lp: ragged constraint matrix");

  // column layout: [x (n)] [slack (m)] [artificial (k)]
  std::vector<int> art_row;
  for (int i = 0; i < m; ++i)
    if (b[static_cast<size_t>(i)] < 0) art_row.push_back(i);
  const int k = static_cast<int>(art_row.size());
  Tableau T;
  T.rows = m;
  T.cols = n + m + k;
  T.t.assign(static_cast<size_t>(m + 1) * (T.cols + 1), 0.0);
  T.basis.assign(static_cast<size_t>(m), -1);
  int next_art = 0;
  for (int i = 0; i < m; ++i) {
    const auto& row = A[static_cast<size_t>(i)];
    double scale = std::fabs(b[static_cast<size_t>(i)]);
    for (double v : row) scale = std::max(scale, std::fabs(v));
    scale = scale > 0.0 ? 1.0 / scale : 1.0;
    const double sign = b[static_cast<size_t>(i)] < 0 ? -1.0 : 1.0;
    for (int j = 0; j < n; ++j) T.at(i, j) = sign * scale * row[static_cast<size_t>(j)];
    T.at(i, n + i) = sign;  // slack (+1, or -1 in a negated row)
    T.rhs(i) = sign * scale * b[static_cast<size_t>(i)];
    if (sign < 0) {
      T.at(i, n + m + next_art) = 1.0;
      T.basis[static_cast<size_t>(i)] = n + m + next_art;
      ++next_art;
    } else {
      T.basis[static_cast<size_t>(i)] = n + i;
    }
  }

  LpResult res;
  // phase 1: minimise the artificials (objective row = -sum of their rows)
  if (k > 0) {
    for (int c = 0; c <= T.cols; ++c) T.at(m, c) = 0.0;
    for (int r : art_row)
      for (int c = 0; c <= T.cols; ++c)
        if (c < n + m || c == T.cols) T.at(m, c) -= T.at(r, c);
    T.optimise(T.cols);
    if (-T.rhs(m) > 1e-7) return res;  // infeasible
    // move remaining (zero-valued) artificials out of the basis
    for (int r = 0; r < m; ++r) {
      if (T.basis[static_cast<size_t>(r)] < n + m) continue;
      for (int c = 0; c < n + m; ++c)
        if (std::fabs(T.at(r, c)) > kEps) {
          T.pivot(r, c);
          break;
        }
    }
  }
  res.feasible = true;
  // phase 2 objective in terms of the non-basic columns
  for (int c = 0; c <= T.cols; ++c) T.at(m, c) = 0.0;
  for (int j = 0; j < n; ++j) T.at(m, j) = c[static_cast<size_t>(j)];
  for (int r = 0; r < m; ++r) {
    const int bc = T.basis[static_cast<size_t>(r)];
    if (bc >= n + m) continue;  // redundant row kept with an artificial at 0
    const double f = T.at(m, bc);
    if (f == 0.0) continue;
    for (int c = 0; c <= T.cols; ++c) T.at(m, c) -= f * T.at(r, c);
  }
  if (!T.optimise(n + m)) {
    res.bounded = false;
    return res;
  }
  res.x.assign(static_cast<size_t>(n), 0.0);
  for (int r = 0; r < m; ++r) {
    const int bc = T.basis[static_cast<size_t>(r)];
    if (bc < n) res.x[static_cast<size_t>(bc)] = T.rhs(r);
  }
  res.objective = 0.0;
  for (int j = 0; j < n; ++j) res.objective += c[static_cast<size_t>(j)] * res.x[static_cast<size_t>(j)];
  return res;
}

}  // namespace offsim
