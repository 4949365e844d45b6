// Known-answer pins for the refcpu oracle (test infrastructure).
//
// Each TEST restates a known-answer / property test of the reference suite
// (proj/tests/*.cpp, cited per case) against the oracle. These are the pins
// that tie the Eigen-free restatement to the reference's documented results
// (SURVEY.md §8c). Inputs use the same std::mt19937 + uniform_real_distribution
// recipes as proj/tests/test_util.hpp so seeded inputs are identical.
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <numeric>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "../refcpu/solver.hpp"

using namespace refcpu;

static int g_fail = 0, g_checks = 0;
static const char* g_case = "";
#define CHECK(c)                                                                  \
  do {                                                                            \
    ++g_checks;                                                                   \
    if (!(c)) {                                                                   \
      ++g_fail;                                                                   \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #c); \
    }                                                                             \
  } while (0)
#define CHECK_THROWS(expr)            \
  do {                                \
    bool thrown = false;              \
    try {                             \
      (void)(expr);                   \
    } catch (const std::exception&) { \
      thrown = true;                  \
    }                                 \
    CHECK(thrown);                    \
  } while (0)
#define CHECK_THROWS_WITH(expr, sub)                              \
  do {                                                            \
    std::string msg;                                              \
    try {                                                         \
      (void)(expr);                                               \
    } catch (const std::exception& e) {                           \
      msg = e.what();                                             \
    }                                                             \
    CHECK(msg.find(sub) != std::string::npos);                    \
  } while (0)

static bool approx(Real a, Real b, Real eps) {
  return std::abs(a - b) <= eps * (std::max(std::abs(a), std::abs(b)));
}

// ---- builders (proj/tests/test_util.hpp:37-122) ----------------------------
static Csr tridiag(Index n, Real lo, Real di, Real up) {
  std::vector<Triplet> t;
  for (Index i = 0; i < n; ++i) {
    if (i > 0) t.push_back({i, i - 1, lo});
    t.push_back({i, i, di});
    if (i + 1 < n) t.push_back({i, i + 1, up});
  }
  return from_triplets(n, n, t);
}
static Csr laplace2d(Index nx, Index ny) {
  auto id = [nx](Index i, Index j) { return j * nx + i; };
  std::vector<Triplet> t;
  for (Index j = 0; j < ny; ++j)
    for (Index i = 0; i < nx; ++i) {
      t.push_back({id(i, j), id(i, j), 4.0});
      if (i > 0) t.push_back({id(i, j), id(i - 1, j), -1.0});
      if (i + 1 < nx) t.push_back({id(i, j), id(i + 1, j), -1.0});
      if (j > 0) t.push_back({id(i, j), id(i, j - 1), -1.0});
      if (j + 1 < ny) t.push_back({id(i, j), id(i, j + 1), -1.0});
    }
  return from_triplets(nx * ny, nx * ny, t);
}
static Csr laplace2d_aniso(Index nx, Index ny, Real eps) {
  auto id = [nx](Index i, Index j) { return j * nx + i; };
  std::vector<Triplet> t;
  for (Index j = 0; j < ny; ++j)
    for (Index i = 0; i < nx; ++i) {
      t.push_back({id(i, j), id(i, j), 2.0 + 2.0 * eps});
      if (i > 0) t.push_back({id(i, j), id(i - 1, j), -1.0});
      if (i + 1 < nx) t.push_back({id(i, j), id(i + 1, j), -1.0});
      if (j > 0) t.push_back({id(i, j), id(i, j - 1), -eps});
      if (j + 1 < ny) t.push_back({id(i, j), id(i, j + 1), -eps});
    }
  return from_triplets(nx * ny, nx * ny, t);
}
static Dense random_dense(std::mt19937& rng, Index r, Index c, Real lo = -1.0, Real hi = 1.0) {
  std::uniform_real_distribution<Real> d(lo, hi);
  Dense M(r, c);
  for (Index i = 0; i < r; ++i)
    for (Index j = 0; j < c; ++j) M(i, j) = d(rng);
  return M;
}
static Vec random_vec(std::mt19937& rng, Index n, Real lo = -1.0, Real hi = 1.0) {
  std::uniform_real_distribution<Real> d(lo, hi);
  Vec v(n);
  for (Index i = 0; i < n; ++i) v[i] = d(rng);
  return v;
}
static Csr random_nonsingular(std::mt19937& rng, Index n) {
  Dense M = random_dense(rng, n, n);
  for (Index i = 0; i < n; ++i) M(i, i) += static_cast<Real>(n);
  return dense_to_sparse(M);
}
static Csr random_sdd(std::mt19937& rng, Index n, Index extras = 3) {
  std::uniform_real_distribution<Real> d(-1.0, 1.0);
  std::uniform_int_distribution<Index> pick(0, n - 1);
  std::vector<Triplet> t;
  std::vector<Real> rs(n, 0.0);
  for (Index i = 0; i < n; ++i)
    for (Index k = 0; k < extras; ++k) {
      Index j = pick(rng);
      if (j == i) continue;
      t.push_back({i, j, d(rng)});
    }
  for (const auto& e : t) rs[e.r] += std::abs(e.v);
  Real diag = 1.0;
  for (Index i = 0; i < n; ++i) diag = std::max(diag, rs[i] + 1.0);
  for (Index i = 0; i < n; ++i) t.push_back({i, i, diag});
  return from_triplets(n, n, t);
}
static Csr dense2(Real a, Real b, Real c, Real d) {
  Dense M(2, 2);
  M(0, 0) = a; M(0, 1) = b; M(1, 0) = c; M(1, 1) = d;
  return dense_to_sparse(M);
}
static Vec axpby(Real a, const Vec& x, Real b, const Vec& y) {
  Vec r(x.size());
  for (size_t i = 0; i < x.size(); ++i) r[i] = a * x[i] + b * y[i];
  return r;
}
static Real dist(const Vec& a, const Vec& b) { return norm(sub(a, b)); }

// ---- sparse (proj/tests/test_sparse.cpp) -----------------------------------
static void test_sparse() {
  g_case = "sparse";
  Csr A = from_triplets(2, 2, {{0, 0, 1.0}, {0, 0, 2.0}, {1, 1, 5.0}});  // 15-20
  CHECK(A.coeff(0, 0) == 3.0);
  CHECK(A.nnz() == 2);
  validate(A);

  Csr I3 = identity(3);  // 22-46
  Vec x = {1, 2, 3};
  CHECK(dist(spmv(I3, x), x) == 0.0);
  Csr A2 = dense2(2, 1, 1, 3);
  Vec y = spmv(A2, {1, 0});
  CHECK(y[0] == 2.0 && y[1] == 1.0);
  Vec z = spmv(tridiag(4, -1, 2, -1), Vec(4, 1.0));
  CHECK(z[0] == 1.0 && z[1] == 0.0 && z[2] == 0.0 && z[3] == 1.0);
  CHECK_THROWS(spmv(A2, Vec(3, 1.0)));

  Csr B = from_triplets(5, 3, {{0, 0, 0.5}, {0, 2, -1.0}, {1, 1, 2.0}, {2, 0, 3.0}, {3, 2, -0.25},
                               {4, 1, 1.5}, {4, 2, 0.75}});  // 48-63
  CHECK(B.nnz() == 7);
  CHECK(same_matrix(transpose(transpose(B)), B));
  Csr T = transpose(from_triplets(2, 2, {{0, 1, 1.0}}));
  CHECK(T.coeff(1, 0) == 1.0 && T.coeff(0, 1) == 0.0);

  std::mt19937 rng(11);  // 65-99
  Csr R6 = dense_to_sparse(random_dense(rng, 6, 6));
  CHECK(same_matrix(matmul(R6, identity(6)), R6));
  Csr Pm = matmul(dense2(1, 1, 0, 1), dense2(1, 0, 1, 1));
  CHECK(Pm.coeff(0, 0) == 2.0 && Pm.coeff(0, 1) == 1.0 && Pm.coeff(1, 0) == 1.0 && Pm.coeff(1, 1) == 1.0);
  for (int trial = 0; trial < 5; ++trial) {
    Csr M1 = dense_to_sparse(random_dense(rng, 20, 20)), M2 = dense_to_sparse(random_dense(rng, 20, 20));
    Vec v = random_vec(rng, 20);
    Vec rhs = spmv(M1, spmv(M2, v));
    CHECK(dist(spmv(matmul(M1, M2), v), rhs) <= 1e-13 * (norm(rhs) + 1.0));
  }
  for (int trial = 0; trial < 5; ++trial) {
    Csr M1 = dense_to_sparse(random_dense(rng, 30, 30)), M2 = dense_to_sparse(random_dense(rng, 30, 30));
    Vec v = random_vec(rng, 30);
    Vec rhs = spmv(M1, spmv(M2, v));
    CHECK(dist(spmv(matmul(M1, M2), v), rhs) <= 1e-12 * norm(rhs));
  }
  CHECK_THROWS(matmul(dense_to_sparse(random_dense(rng, 3, 4)), dense_to_sparse(random_dense(rng, 3, 4))));

  CHECK(same_matrix(extract(identity(4), {0, 2}, {0, 2}), identity(2)));  // 101-130
  Csr sub1 = extract(dense2(4, 1, 1, 3), {0}, {1});
  CHECK(sub1.rows == 1 && sub1.cols == 1 && sub1.coeff(0, 0) == 1.0);
  std::mt19937 rng3(3);
  Csr R10 = dense_to_sparse(random_dense(rng3, 10, 10));
  IndexList F = {0, 3, 4, 7, 9}, C = complement(10, F);
  std::vector<Triplet> t;
  auto scatter = [&t](const Csr& M, const IndexList& rows, const IndexList& cols) {
    for (Index i = 0; i < M.rows; ++i)
      for (Index k = M.ptr[i]; k < M.ptr[i + 1]; ++k) t.push_back({rows[i], cols[M.col[k]], M.val[k]});
  };
  scatter(extract(R10, F, F), F, F);
  scatter(extract(R10, F, C), F, C);
  scatter(extract(R10, C, F), C, F);
  scatter(extract(R10, C, C), C, C);
  CHECK(same_matrix(from_triplets(10, 10, t), R10));
  CHECK_THROWS(extract(R10, {0, 10}, {0}));

  Vec dinv = diag_inverse(from_triplets(2, 2, {{0, 0, 2.0}, {1, 1, 4.0}}));  // 132-145
  CHECK(dinv[0] == 0.5 && dinv[1] == 0.25);
  CHECK_THROWS_WITH(diag_inverse(from_triplets(2, 2, {{0, 0, 1.0}, {1, 1, 0.0}, {1, 0, 1.0}})), "row 1");
  CHECK_THROWS_WITH(diag_inverse(from_triplets(2, 2, {{0, 0, 1.0}, {1, 0, 1.0}})), "row 1");

  DenseLU lu(to_dense(dense2(4, 1, 1, 3)));  // 147-181
  Vec xs = lu.solve(Vec{1, 0});
  CHECK(approx(xs[0], 3.0 / 11.0, 1e-14) && approx(xs[1], -1.0 / 11.0, 1e-14));
  std::mt19937 rng21(21);
  for (int trial = 0; trial < 100; ++trial) {
    Dense M = random_dense(rng21, 20, 20);
    for (Index i = 0; i < 20; ++i) M(i, i) += 20.0;
    Vec bb = random_vec(rng21, 20);
    Vec xx = DenseLU(M).solve(bb);
    CHECK(dist(spmv(dense_to_sparse(M), xx), bb) <= 1e-10 * norm(bb));
  }
  CHECK_THROWS(DenseLU(Dense(3, 3)));

  BlockDiagonalLU bl(dense2(4, 1, 1, 3), BlockLayout::from_sizes({2}));  // 183-214
  Vec zb = bl.solve({1, 0});
  CHECK(approx(zb[0], 3.0 / 11.0, 1e-14) && approx(zb[1], -1.0 / 11.0, 1e-14));
  CHECK_THROWS_WITH(BlockDiagonalLU(from_triplets(2, 2, {{0, 0, 1.0}}), BlockLayout::from_sizes({1, 1})),
                    "block 1");
}

// ---- relax (proj/tests/test_relax.cpp) -------------------------------------
static void test_relax() {
  g_case = "relax";
  Csr A = dense2(2, 1, 1, 2);
  Vec b(2, 1.0), x(2, 0.0);
  jacobi_sweep(A, b, x, 1.0);  // 22-48
  CHECK(x[0] == 0.5 && x[1] == 0.5);
  Vec g(2, 0.0);
  hybrid_l1_gs_sweep(A, b, g, true);  // 50-80
  CHECK(g[0] == 0.5 && g[1] == 0.25);
  Vec h(2, 0.0);
  hybrid_l1_gs_sweep(A, b, h, true, {{0, 1}, {1, 2}});
  CHECK(approx(h[0], 1.0 / 3.0, 1e-15) && approx(h[1], 1.0 / 3.0, 1e-15));
  Vec bw(2, 0.0);
  hybrid_l1_gs_sweep(A, b, bw, false);
  CHECK(bw[1] == 0.5 && bw[0] == 0.25);

  std::mt19937 rng(17);  // 82-99
  Csr S = random_sdd(rng, 30);
  Vec bb = random_vec(rng, 30), xx(30, 0.0), yy(30, 0.0);
  hybrid_l1_gs_sweep(S, bb, xx, true);
  Dense Sd = to_dense(S);
  for (Index i = 0; i < 30; ++i) {
    Real s = bb[i];
    for (Index j = 0; j < 30; ++j)
      if (j != i) s -= Sd(i, j) * yy[j];
    yy[i] = s / Sd(i, i);
  }
  CHECK(dist(xx, yy) <= 1e-13 * norm(yy));

  Vec d1 = l1_diagonal(A, {}), d2 = l1_diagonal(A, {{0, 1}, {1, 2}});  // 101-109
  CHECK(d1[0] == 2.0 && d1[1] == 2.0 && d2[0] == 3.0 && d2[1] == 3.0);

  std::mt19937 rng23(23);  // 139-160
  Csr S24 = random_sdd(rng23, 24);
  std::vector<SmootherSpec> specs = {
      {SmootherKind::jacobi, 2, 0.8, {}, {}, nullptr, false},
      {SmootherKind::l1_jacobi, 1, 1.0, {}, {}, nullptr, false},
      {SmootherKind::hybrid_l1_gs_forward, 2, 1.0, {}, {{0, 12}, {12, 24}}, nullptr, false},
      {SmootherKind::hybrid_l1_gs_backward, 1, 1.0, {}, {}, nullptr, false},
      {SmootherKind::dense_lu, 1, 1.0, {}, {}, nullptr, false},
      {SmootherKind::block_jacobi_exact, 1, 1.0, std::vector<Index>(12, 2), {}, nullptr, false}};
  Vec r1 = random_vec(rng23, 24), r2 = random_vec(rng23, 24);
  for (const auto& sp : specs) {
    BoundSmoother sm = BoundSmoother::bind(sp, S24);
    Vec lhs = sm.apply(axpby(2.5, r1, -0.75, r2));
    Vec rhs = axpby(2.5, sm.apply(r1), -0.75, sm.apply(r2));
    CHECK(dist(lhs, rhs) <= 1e-13 * (norm(rhs) + 1.0));
  }
  std::mt19937 rng5(5);  // 178-198
  Csr S10 = random_sdd(rng5, 10);
  Vec r = random_vec(rng5, 10);
  BoundSmoother jac = BoundSmoother::bind({SmootherKind::jacobi, 1, 1.0, {}, {}, nullptr, false}, S10);
  Vec di = diag_inverse(S10), ex(10);
  for (Index i = 0; i < 10; ++i) ex[i] = di[i] * r[i];
  CHECK(dist(jac.apply(r), ex) == 0.0);
  CHECK_THROWS(BoundSmoother::bind({SmootherKind::jacobi, 1, 2.5, {}, {}, nullptr, false}, S10));
  CHECK_THROWS(BoundSmoother::bind({SmootherKind::jacobi, 0, 1.0, {}, {}, nullptr, false}, S10));
  CHECK_THROWS(BoundSmoother::bind({SmootherKind::hybrid_l1_gs_forward, 1, 1.0, {}, {{0, 4}}, nullptr, false}, S10));
}

// ---- krylov (proj/tests/test_krylov.cpp) -----------------------------------
static void test_krylov() {
  g_case = "krylov";
  std::mt19937 rng(2);
  Vec b = random_vec(rng, 8), x(8, 0.0);
  KrylovConfig cfg;
  cfg.rel_tol = 1e-12;
  SolveReport rep = gmres(identity(8), b, x, cfg);  // 14-25
  CHECK(rep.converged && rep.iterations == 1);
  CHECK(dist(x, b) <= 1e-12 * norm(b));

  std::mt19937 rng77(77);  // 27-63
  for (Index n : {37, 120, 200}) {
    Csr A = random_nonsingular(rng77, n);
    DenseLU lu = factor_dense(A);
    Vec bb = random_vec(rng77, n), xx(n, 0.0);
    SolveReport r2 = gmres(A, bb, xx, cfg, [&lu](const Vec& v) { return lu.solve(v); });
    CHECK(r2.converged && r2.iterations == 1);
    CHECK(dist(spmv(A, xx), bb) <= 1e-12 * norm(bb));
  }
  {
    Csr L = tridiag(100, -1, 2, -1);  // 65-79
    std::mt19937 rng4(4);
    Vec bb = random_vec(rng4, 100), xx(100, 0.0);
    KrylovConfig c;
    c.rel_tol = 1e-8;
    c.max_iters = 2000;
    CHECK(gmres(L, bb, xx, c).converged);
    Vec xd = factor_dense(L).solve(bb);
    CHECK(dist(xx, xd) <= 1e-6 * norm(xd));
  }
  {
    Csr L = laplace2d(12, 12);  // 81-103
    std::mt19937 rng8(8);
    Vec bb = random_vec(rng8, L.rows);
    KrylovConfig c;
    c.rel_tol = 1e-9;
    c.max_iters = 1000;
    std::vector<Index> its;
    for (Real a : {1e-6, 1.0, 1e6}) {
      Vec xx(L.rows, 0.0), sb(bb.size());
      for (size_t i = 0; i < bb.size(); ++i) sb[i] = a * bb[i];
      SolveReport r3 = gmres(L, sb, xx, c);
      CHECK(r3.converged);
      its.push_back(r3.iterations);
    }
    CHECK(its[0] == its[1] && its[1] == its[2]);
  }
  {
    Csr L = tridiag(6, -1, 2, -1);  // 125-133
    Vec xx(6, 1.0);
    SolveReport r4 = gmres(L, Vec(6, 0.0), xx, KrylovConfig{});
    CHECK(r4.converged && r4.iterations == 0 && norm(xx) == 0.0);
  }
  {
    Csr S = from_triplets(3, 3, {{0, 0, 1.0}, {1, 1, 1.0}});  // 135-159
    KrylovConfig c;
    c.rel_tol = 1e-10;
    Vec bb = {0, 0, 1}, xx(3, 0.0);
    CHECK_THROWS(gmres(S, bb, xx, c));
    c.rel_tol = 1e-12;
    Vec b2 = {1, 1, 0}, x2(3, 0.0);
    SolveReport r5 = gmres(S, b2, x2, c);
    CHECK(r5.converged && dist(spmv(S, x2), b2) <= 1e-12 * norm(b2));
  }
  {
    Vec bb(3, 1.0), xx(3, 0.0);  // 161-168
    bb[1] = std::numeric_limits<Real>::quiet_NaN();
    CHECK_THROWS(gmres(identity(3), bb, xx, KrylovConfig{}));
  }
  {
    Csr L = laplace2d(8, 8);  // 181-194
    std::mt19937 rng31(31);
    Vec bb = random_vec(rng31, L.rows), xx(L.rows, 0.0);
    KrylovConfig c;
    c.rel_tol = 1e-9;
    SolveReport r6 = gmres(L, bb, xx, c);
    CHECK(r6.converged);
    const Real truth = dist(bb, spmv(L, xx)) / norm(bb);
    CHECK(approx(r6.final_residual, truth, 1e-10) && r6.final_residual <= c.rel_tol);
  }
}

// ---- amg (proj/tests/test_amg.cpp) -----------------------------------------
static Index amg_iters(const Csr& A, const AmgHierarchy& H, Real tol, Index maxit) {
  std::mt19937 rng(99);
  Vec b = random_vec(rng, A.rows), x(A.rows, 0.0);
  KrylovConfig c;
  c.rel_tol = tol;
  c.max_iters = maxit;
  SolveReport r = gmres(A, b, x, c, [&H](const Vec& v) { return amg_vcycle(H, v); });
  CHECK(r.converged);
  return r.iterations;
}

static void test_amg() {
  g_case = "amg";
  Csr L = tridiag(6, -1, 2, -1);  // 31-49
  CHECK(strength_graph(L, 0.25).nnz() == L.nnz() - 6);
  CHECK(strength_graph(from_triplets(3, 3, {{0, 0, 1.0}, {1, 1, 2.0}, {2, 2, 3.0}}), 0.25).nnz() == 0);
  Csr Sa = strength_graph(laplace2d_aniso(5, 5, 0.01), 0.25);
  bool only_x = Sa.nnz() > 0;
  for (Index i = 0; i < Sa.rows; ++i)
    for (Index k = Sa.ptr[i]; k < Sa.ptr[i + 1]; ++k) only_x = only_x && std::abs(Sa.col[k] - i) == 1;
  CHECK(only_x);

  IndexList C, F;  // 51-70
  Csr E;
  E.rows = E.cols = 4;
  E.ptr.assign(5, 0);
  pmis_coarsen(E, C, F);
  CHECK(C.size() == 4 && F.empty());
  pmis_coarsen(from_triplets(2, 2, {{0, 1, 1.0}, {1, 0, 1.0}}), C, F);
  CHECK(C.size() == 1 && F.size() == 1);
  pmis_coarsen(strength_graph(tridiag(9, -1, 2, -1), 0.25), C, F);
  CHECK(C.size() >= 3 && C.size() <= 5 && C.size() + F.size() == 9);

  Csr D = from_triplets(3, 3, {{0, 0, 2.0}, {1, 1, 2.0}, {2, 2, 2.0}});  // 72-118
  CHECK(same_matrix(classical_interp(D, strength_graph(D, 0.25), {0, 1, 2}, {}), identity(3)));
  Csr L3 = tridiag(3, -1, 2, -1);
  Csr P = classical_interp(L3, strength_graph(L3, 0.25), {0, 2}, {1});
  CHECK(P.coeff(0, 0) == 1.0 && P.coeff(2, 1) == 1.0);
  CHECK(approx(P.coeff(1, 0), 0.5, 1e-14) && approx(P.coeff(1, 1), 0.5, 1e-14));
  {
    std::mt19937 rng(13);
    const Index n = 40;
    std::uniform_int_distribution<Index> pick(0, n - 1);
    std::set<std::pair<Index, Index>> edges;
    for (Index i = 0; i < n; ++i) edges.insert({i, (i + 1) % n});
    for (int k = 0; k < 2 * n; ++k) {
      Index a = pick(rng), b = pick(rng);
      if (a != b) edges.insert({std::min(a, b), std::max(a, b)});
    }
    std::vector<Triplet> t;
    std::vector<Real> deg(n, 0.0);
    for (const auto& [a, b] : edges) {
      t.push_back({a, b, -1.0});
      t.push_back({b, a, -1.0});
      deg[a] += 1.0;
      deg[b] += 1.0;
    }
    for (Index i = 0; i < n; ++i) t.push_back({i, i, deg[i]});
    Csr M = from_triplets(n, n, t);
    Csr S = strength_graph(M, 0.25);
    IndexList Cm, Fm;
    pmis_coarsen(S, Cm, Fm);
    CHECK(!Fm.empty());
    Csr Pm = classical_interp(M, S, Cm, Fm);
    for (Index i : Fm) {
      Real s = 0.0;
      for (Index k = Pm.ptr[i]; k < Pm.ptr[i + 1]; ++k) s += Pm.val[k];
      CHECK(approx(s, 1.0, 1e-12));
    }
  }
  {
    AmgConfig cfg;  // 120-130
    cfg.coarse_size = 2;
    AmgHierarchy H = amg_setup(identity(30), cfg);
    CHECK(H.num_levels() == 1 && H.info.truncated);
  }
  {
    Csr A = laplace2d(20, 20);  // 132-143 Galerkin identity, bitwise
    AmgHierarchy H = amg_setup(A, AmgConfig{});
    CHECK(H.num_levels() >= 2);
    for (Index l = 0; l + 1 < H.num_levels(); ++l) {
      CHECK(same_matrix(matmul(H.levels[l].R, matmul(H.levels[l].A, H.levels[l].P)), H.levels[l + 1].A));
      CHECK(same_matrix(H.levels[l].R, transpose(H.levels[l].P)));
      CHECK(H.levels[l + 1].A.rows < H.levels[l].A.rows);
    }
  }
  {
    Csr A = laplace2d(12, 12);  // 145-154 linearity
    AmgHierarchy H = amg_setup(A, AmgConfig{});
    std::mt19937 rng(41);
    Vec r1 = random_vec(rng, A.rows), r2 = random_vec(rng, A.rows);
    Vec rhs = axpby(1.5, amg_vcycle(H, r1), -2.0, amg_vcycle(H, r2));
    CHECK(dist(amg_vcycle(H, axpby(1.5, r1, -2.0, r2)), rhs) <= 1e-12 * (norm(rhs) + 1.0));
  }
  {
    Csr A = laplace2d(32, 32);  // 156-162
    AmgHierarchy H = amg_setup(A, AmgConfig{});
    CHECK(amg_iters(A, H, 1e-8, 100) <= 20);
  }
  {
    std::vector<Index> counts;  // 164-176
    for (Index n : {16, 32, 64}) {
      Csr A = laplace2d(n, n);
      counts.push_back(amg_iters(A, amg_setup(A, AmgConfig{}), 1e-8, 200));
    }
    const Real lo = *std::min_element(counts.begin(), counts.end());
    const Real hi = *std::max_element(counts.begin(), counts.end());
    CHECK(hi / lo <= 1.5);
  }
  {
    Csr L1 = laplace2d(8, 8), L2 = tridiag(120, -1.0, 2.1, -1.0);  // 187-229
    const Index n1 = L1.rows, n2 = L2.rows;
    std::vector<Triplet> t;
    for (Index i = 0; i < n1; ++i)
      for (Index k = L1.ptr[i]; k < L1.ptr[i + 1]; ++k) t.push_back({i, L1.col[k], L1.val[k]});
    for (Index i = 0; i < n2; ++i)
      for (Index k = L2.ptr[i]; k < L2.ptr[i + 1]; ++k) t.push_back({n1 + i, n1 + L2.col[k], L2.val[k]});
    Csr A = from_triplets(n1 + n2, n1 + n2, t);
    AmgConfig sc;
    sc.unknown_map.assign(n1, 0);
    sc.unknown_map.insert(sc.unknown_map.end(), n2, 1);
    AmgHierarchy Hs = amg_setup(A, sc);
    AmgHierarchy H1 = amg_setup(L1, AmgConfig{}), H2 = amg_setup(L2, AmgConfig{});
    CHECK(Hs.num_levels() >= 2 && H1.num_levels() >= 2 && H2.num_levels() >= 2);
    const Csr& P1 = H1.levels[0].P;
    const Csr& P2 = H2.levels[0].P;
    std::vector<Triplet> tb;
    for (Index i = 0; i < P1.rows; ++i)
      for (Index k = P1.ptr[i]; k < P1.ptr[i + 1]; ++k) tb.push_back({i, P1.col[k], P1.val[k]});
    for (Index i = 0; i < P2.rows; ++i)
      for (Index k = P2.ptr[i]; k < P2.ptr[i + 1]; ++k) tb.push_back({n1 + i, P1.cols + P2.col[k], P2.val[k]});
    CHECK(same_matrix(Hs.levels[0].P, from_triplets(n1 + n2, P1.cols + P2.cols, tb)));
    const auto& cmap = Hs.levels[1].unknown_map;
    CHECK(static_cast<Index>(cmap.size()) == P1.cols + P2.cols);
    for (Index k = 0; k < static_cast<Index>(cmap.size()); ++k) CHECK(cmap[k] == (k < P1.cols ? 0 : 1));
  }
}

// ---- mgr (proj/tests/test_mgr.cpp) -----------------------------------------
static MgrLevelSpec level(std::vector<std::string> f, InterpKind i, RestrictKind r, SmootherSpec s) {
  MgrLevelSpec l;
  l.f_fields = std::move(f);
  l.interp = i;
  l.restrict_kind = r;
  l.f_relax = s;
  return l;
}

static void test_mgr() {
  g_case = "mgr";
  const SmootherSpec exact{SmootherKind::dense_lu, 1, 1.0, {}, {}, nullptr, false};
  const SmootherSpec jac{SmootherKind::jacobi, 1, 1.0, {}, {}, nullptr, false};
  DofPartition part = DofPartition::from_names({"p", "pi"}, {"p", "pi", "p", "pi"});  // 35-57
  IndexList F, C;
  split(part, {"pi"}, F, C);
  CHECK(F == IndexList({1, 3}) && C == IndexList({0, 2}));
  CHECK_THROWS(split(DofPartition::from_names({"p"}, {"p", "p"}), {"p"}, F, C));
  CHECK_THROWS(split(part, {"rho"}, F, C));

  Csr A = dense2(4, 1, 1, 3);  // 59-118
  Csr P = build_interp(A, {0}, {1}, InterpKind::jacobi);
  CHECK(P.coeff(0, 0) == -0.25 && P.coeff(1, 0) == 1.0);
  Csr Pd = build_interp(from_triplets(3, 3, {{0, 0, 2.0}, {1, 1, 3.0}, {2, 2, 4.0}}), {0}, {1, 2}, InterpKind::ideal);
  CHECK(Pd.nnz() == 2 && Pd.coeff(1, 0) == 1.0 && Pd.coeff(2, 1) == 1.0);
  Dense M3(3, 3);
  M3(0, 0) = 2; M3(0, 2) = 1; M3(1, 1) = 4; M3(1, 2) = 2; M3(2, 0) = 1; M3(2, 1) = 2; M3(2, 2) = 8;
  Csr A3 = dense_to_sparse(M3);
  Csr P3 = build_interp(A3, {0, 1}, {2}, InterpKind::ideal);
  CHECK(approx(P3.coeff(0, 0), -0.5, 1e-14) && approx(P3.coeff(1, 0), -0.5, 1e-14) && P3.coeff(2, 0) == 1.0);
  Csr Rinj = build_restrict(A, {0}, {1}, RestrictKind::injection);
  CHECK(Rinj.rows == 1 && Rinj.cols == 2 && Rinj.nnz() == 1 && Rinj.coeff(0, 1) == 1.0);
  Csr Rj = build_restrict(A, {0}, {1}, RestrictKind::jacobi);
  CHECK(Rj.coeff(0, 0) == -0.25 && Rj.coeff(0, 1) == 1.0);
  Csr R3 = build_restrict(A3, {0, 1}, {2}, RestrictKind::ideal);
  CHECK(approx(R3.coeff(0, 0), -0.5, 1e-14) && approx(R3.coeff(0, 1), -0.5, 1e-14) && R3.coeff(0, 2) == 1.0);

  Csr S = coarse_operator(A, build_restrict(A, {0}, {1}, RestrictKind::ideal),
                          build_interp(A, {0}, {1}, InterpKind::ideal));  // 96-118
  CHECK(S.rows == 1 && approx(S.coeff(0, 0), 2.75, 1e-14));
  CHECK(approx(coarse_operator(A3, R3, P3).coeff(0, 0), 6.5, 1e-14));

  {
    std::mt19937 rng(19);  // 120-142 ideal = dense Schur
    for (int trial = 0; trial < 5; ++trial) {
      Csr R = random_nonsingular(rng, 30);
      IndexList Fs, Cs;
      for (Index i = 0; i < 30; ++i) (i % 3 == 0 ? Fs : Cs).push_back(i);
      Csr Sc = coarse_operator(R, build_restrict(R, Fs, Cs, RestrictKind::ideal),
                               build_interp(R, Fs, Cs, InterpKind::ideal));
      Dense Aff = to_dense(extract(R, Fs, Fs)), Afc = to_dense(extract(R, Fs, Cs));
      Dense X = DenseLU(Aff).solve(Afc);
      Dense Acf = to_dense(extract(R, Cs, Fs)), Acc = to_dense(extract(R, Cs, Cs));
      Real err = 0.0, nrm = 0.0;
      for (Index i = 0; i < Acc.rows; ++i)
        for (Index j = 0; j < Acc.cols; ++j) {
          Real s = Acc(i, j);
          for (Index k = 0; k < Acf.cols; ++k) s -= Acf(i, k) * X(k, j);
          err += std::pow(Sc.coeff(i, j) - s, 2);
          nrm += s * s;
        }
      CHECK(std::sqrt(err) <= 1e-12 * std::sqrt(nrm));
    }
  }
  {
    std::mt19937 rng(23);  // 144-154
    Csr R = random_nonsingular(rng, 40);
    IndexList Fs, Cs;
    for (Index i = 0; i < 40; ++i) (i % 2 == 0 ? Fs : Cs).push_back(i);
    Dense a = to_dense(schur_jacobi_direct(R, Fs, Cs));
    Dense b = to_dense(coarse_operator(R, build_restrict(R, Fs, Cs, RestrictKind::injection),
                                       build_interp(R, Fs, Cs, InterpKind::jacobi)));
    Real e = 0, nb = 0;
    for (size_t k = 0; k < a.a.size(); ++k) {
      e += std::pow(a.a[k] - b.a[k], 2);
      nb += b.a[k] * b.a[k];
    }
    CHECK(std::sqrt(e) <= 1e-12 * std::sqrt(nb));
  }
  {
    DofPartition p6 = DofPartition::from_names({"a", "b"}, {"a", "b", "a", "b", "a", "b"});  // 194-230
    std::mt19937 rng(3);
    Csr R = random_nonsingular(rng, 6);
    MgrStrategy st;
    st.levels.push_back(level({"b"}, InterpKind::jacobi, RestrictKind::injection, jac));
    MgrHierarchy H1 = mgr_setup(R, p6, st), H2 = mgr_setup(R, p6, st);
    CHECK(H1.num_reduction_levels() == 1 && H1.A_coarse.rows == 3 && H1.levels[0].F.size() == 3);
    CHECK(H1.coarse_finest_ids == IndexList({0, 2, 4}));
    CHECK(same_matrix(H1.levels[0].P, H2.levels[0].P) && same_matrix(H1.A_coarse, H2.A_coarse));
    CHECK(same_matrix(H1.A_coarse, matmul(H1.levels[0].R, matmul(H1.levels[0].A, H1.levels[0].P))));
    MgrStrategy twice = st;
    twice.levels.push_back(st.levels[0]);
    CHECK_THROWS(mgr_setup(R, p6, twice));
  }
  {
    DofPartition pf = DofPartition::from_names({"f", "c"}, {"f", "c"});  // 244-269
    MgrStrategy st;
    st.levels.push_back(level({"f"}, InterpKind::ideal, RestrictKind::injection, exact));
    MgrHierarchy H = mgr_setup(A, pf, st);
    Vec z = mgr_apply(H, {1, 0});
    CHECK(approx(z[0], 3.0 / 11.0, 1e-14) && approx(z[1], -1.0 / 11.0, 1e-14));
    st.levels[0].interp = InterpKind::jacobi;
    CHECK(dist(mgr_apply(mgr_setup(A, pf, st), {1, 0}), z) <= 1e-15);
  }
  {
    std::mt19937 rng(47);  // 271-300 exactness
    for (Index n : {20, 97, 200}) {
      Csr R = random_nonsingular(rng, n);
      std::vector<std::string> names(n);
      for (Index i = 0; i < n; ++i) names[i] = (rng() % 2 == 0) ? "f" : "c";
      names[0] = "f";
      names[1] = "c";
      MgrStrategy st;
      st.levels.push_back(level({"f"}, InterpKind::ideal, RestrictKind::injection, exact));
      MgrHierarchy H = mgr_setup(R, DofPartition::from_names({"f", "c"}, names), st);
      Vec b = random_vec(rng, n), x(n, 0.0);
      KrylovConfig c;
      c.rel_tol = 1e-12;
      SolveReport rep = gmres(R, b, x, c, mgr_preconditioner(H));
      CHECK(rep.converged && rep.iterations == 1);
      CHECK(dist(b, spmv(R, x)) <= 1e-12 * norm(b));
    }
  }
  {
    std::mt19937 rng(61);  // 324-377 permutation equivariance
    const Index n = 60;
    Csr R = random_sdd(rng, n, 4);
    std::vector<std::string> names;
    for (Index i = 0; i < n; ++i) names.push_back(i % 2 == 0 ? "f" : "c");
    MgrStrategy st;
    st.levels.push_back(level({"f"}, InterpKind::jacobi, RestrictKind::injection, jac));
    std::mt19937 rngb(62);
    Vec b = random_vec(rngb, n);
    KrylovConfig c;
    c.rel_tol = 1e-9;
    c.max_iters = 400;
    MgrHierarchy H = mgr_setup(R, DofPartition::from_names({"f", "c"}, names), st);
    Vec x(n, 0.0);
    SolveReport rep = gmres(R, b, x, c, mgr_preconditioner(H));
    CHECK(rep.converged);
    std::vector<Index> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<Triplet> t;
    for (Index i = 0; i < n; ++i)
      for (Index k = R.ptr[i]; k < R.ptr[i + 1]; ++k) t.push_back({perm[i], perm[R.col[k]], R.val[k]});
    Csr Rp = from_triplets(n, n, t);
    std::vector<std::string> np(n);
    Vec bp(n);
    for (Index i = 0; i < n; ++i) {
      np[perm[i]] = names[i];
      bp[perm[i]] = b[i];
    }
    MgrHierarchy Hp = mgr_setup(Rp, DofPartition::from_names({"f", "c"}, np), st);
    Vec xp(n, 0.0);
    SolveReport rp = gmres(Rp, bp, xp, c, mgr_preconditioner(Hp));
    CHECK(rp.converged && rep.iterations == rp.iterations);
    Vec xu(n);
    for (Index i = 0; i < n; ++i) xu[i] = xp[perm[i]];
    CHECK(dist(xu, x) <= 1e-7 * norm(x));
  }
}

// ---- strategy json (proj/src/strategy_json.cpp) ------------------------------
static void test_json() {
  g_case = "json";
  MgrStrategy s = strategy_from_json_text(
      R"({"name":"mgr_pi","levels":[{"f_fields":["pi"],"interp":"ideal","restrict":"injection",
      "f_relax":{"kind":"jacobi","sweeps":1,"weight":1.0}}],"coarse":{"kind":"amg_vcycle","cycles":8,
      "amg":{"strength_theta":0.05}}})");
  CHECK(s.levels.size() == 1 && s.levels[0].interp == InterpKind::ideal && s.coarse.amg_cycles == 8);
  CHECK(s.coarse.amg.strength_theta == 0.05);
  CHECK(s.coarse.amg.pre_smoother.kind == SmootherKind::hybrid_l1_gs_forward);
  MgrStrategy back = strategy_from_json_text(strategy_to_json_text(s));
  CHECK(strategy_to_json_text(back) == strategy_to_json_text(s));
  CHECK_THROWS_WITH(strategy_from_json_text(R"({"levels":[{"f_fields":["p"],"bogus":1}]})"),
                    "levels[0]: unknown key 'bogus'");
  CHECK_THROWS_WITH(strategy_from_json_text(R"({"coarse":{"kind":"nope"}})"), "unknown coarse solver kind");
}

int main() {
  test_sparse();
  test_relax();
  test_krylov();
  test_amg();
  test_mgr();
  test_json();
  std::printf("refcpu pins: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
