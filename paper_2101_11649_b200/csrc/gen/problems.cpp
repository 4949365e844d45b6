// Synthetic problem generators for the BASELINE.json configs (SURVEY.md §8d,
// "Next #1"). These produce the input bundle (CSR matrix, rhs, field labels)
// that both the GPU path and the CPU oracle consume, so both see identical
// bits. They are host-side input producers, not part of the solve path.
//
// cfg1/cfg2 — hybrid mimetic FD (TPFA inner product) on a structured hex grid
// with unit cells, statically condensed to the two-field [p, pi] system the
// reference builds in proj/src/problems/mfd.cpp:337-458 (assemble_hybrid +
// static_condense). With the diagonal inner product B = diag(1/t_l) the
// fluxes eliminate cell by cell and the condensed rows are
//   cell c : (acc + sum_l t_l) p_c - sum_l t_l pi_{f(l)}
//   face f : -sum_{c ~ f} t_{c,l} p_c + (sum_{c ~ f} t_{c,l}) pi_f
// with half-transmissibility t_l = |f| (c_l . K n_l)/|c_l|^2 = 2 k_dir for
// unit cubes (mfd.cpp:272-285). All faces carry a multiplier dof (all
// no-flow) and the accumulation makes the system nonsingular.
//
// Dof numbering is slab-major in z: for each layer k, its cells
// (i fastest), its x-faces, its y-faces, its bottom z-faces, and for the top
// layer also the top z-faces. Every GPU count uses this one numbering.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

// Box-Muller standard normal on mt19937 (proj/src/problems/comp.cpp:20-31).
class Normal {
 public:
  explicit Normal(unsigned seed) : rng_(seed) {}
  double operator()() {
    const double u1 = (static_cast<double>(rng_()) + 0.5) * 0x1.0p-32;
    const double u2 = (static_cast<double>(rng_()) + 0.5) * 0x1.0p-32;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }

 private:
  std::mt19937 rng_;
};

// U(a,b) = a + (b-a)(u+0.5)2^-32.
class Uniform {
 public:
  explicit Uniform(unsigned seed) : rng_(seed) {}
  double operator()(double a, double b) {
    return a + (b - a) * ((static_cast<double>(rng_()) + 0.5) * 0x1.0p-32);
  }

 private:
  std::mt19937 rng_;
};

struct Problem {
  int n = 0;
  std::vector<int> ptr, col, labels, unknown_map;
  std::vector<double> val, rhs;
  std::vector<std::string> fields;
  std::string meta;  // JSON object with generator parameters
};

struct RowBuilder {
  // Rows are assembled as small (col, val) lists and sorted by column; the
  // generator never emits duplicate columns within a row.
  std::vector<std::pair<int, double>> e;
  void add(int c, double v) { e.push_back({c, v}); }
};

void finish_row(Problem& P, RowBuilder& rb) {
  std::sort(rb.e.begin(), rb.e.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  for (const auto& [c, v] : rb.e) {
    P.col.push_back(c);
    P.val.push_back(v);
  }
  P.ptr.push_back(static_cast<int>(P.col.size()));
  rb.e.clear();
}

struct MfdLayout {
  int nx, ny, nz;
  int64_t nc2, nfx, nfy, slab;
  int64_t off(int k) const { return slab * k; }
  int64_t cell(int i, int j, int k) const { return off(k) + i + int64_t(nx) * j; }
  int64_t xf(int i, int j, int k) const { return off(k) + nc2 + i + int64_t(nx + 1) * j; }
  int64_t yf(int i, int j, int k) const { return off(k) + nc2 + nfx + i + int64_t(nx) * j; }
  int64_t zf(int i, int j, int kz) const {
    const int64_t base = kz < nz ? off(kz) + nc2 + nfx + nfy : off(nz - 1) + nc2 + nfx + nfy + nc2;
    return base + i + int64_t(nx) * j;
  }
  int64_t total() const { return slab * nz + nc2; }
};

// field: 0 = i.i.d. ln k ~ N(0,1) per cell and direction (cfg1);
//        1 = layered: mu_k ~ U(-3,3) per layer, ln k = mu_k + sigma N(0,1) (cfg2).
Problem make_mfd(int nx, int ny, int nz, int field, double sigma, unsigned seed, double accum) {
  if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("mfd: dims must be >= 1");
  MfdLayout L{nx, ny, nz, int64_t(nx) * ny, int64_t(nx + 1) * ny, int64_t(nx) * (ny + 1), 0};
  L.slab = L.nc2 + L.nfx + L.nfy + L.nc2;
  if (L.total() > INT32_MAX / 2) throw std::invalid_argument("mfd: grid too large for int32 indices");
  const int64_t ncell = L.nc2 * nz;

  // Half transmissibilities per cell and direction: t = 2 k_dir (unit cube).
  std::vector<double> tx(ncell), ty(ncell), tz(ncell);
  {
    Normal nrm(seed);
    Uniform uni(seed ^ 0x5bd1e995u);
    for (int k = 0; k < nz; ++k) {
      const double mu = field == 1 ? uni(-3.0, 3.0) : 0.0;
      const double sg = field == 1 ? sigma : 1.0;
      for (int64_t q = 0; q < L.nc2; ++q) {
        const int64_t c = k * L.nc2 + q;
        tx[c] = 2.0 * std::exp(mu + sg * nrm());
        ty[c] = 2.0 * std::exp(mu + sg * nrm());
        tz[c] = 2.0 * std::exp(mu + sg * nrm());
      }
    }
  }
  auto cid = [&](int i, int j, int k) { return int64_t(k) * L.nc2 + i + int64_t(nx) * j; };

  Problem P;
  P.n = static_cast<int>(L.total());
  P.fields = {"p", "pi"};
  P.ptr.reserve(P.n + 1);
  P.ptr.push_back(0);
  P.labels.reserve(P.n);
  RowBuilder rb;

  auto face_row = [&](int64_t fdof, int64_t c0, double t0, int64_t dof0, int64_t c1, double t1,
                      int64_t dof1) {
    (void)c0;
    (void)c1;
    double d = 0.0;
    if (dof0 >= 0) {
      rb.add(static_cast<int>(dof0), -t0);
      d += t0;
    }
    if (dof1 >= 0) {
      rb.add(static_cast<int>(dof1), -t1);
      d += t1;
    }
    rb.add(static_cast<int>(fdof), d);
    finish_row(P, rb);
    P.labels.push_back(1);
  };

  for (int k = 0; k < nz; ++k) {
    // cells
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int64_t c = cid(i, j, k);
        const double t[6] = {tx[c], tx[c], ty[c], ty[c], tz[c], tz[c]};
        const int64_t f[6] = {L.xf(i, j, k), L.xf(i + 1, j, k), L.yf(i, j, k),
                              L.yf(i, j + 1, k), L.zf(i, j, k), L.zf(i, j, k + 1)};
        double d = accum;
        for (int l = 0; l < 6; ++l) {
          d += t[l];
          rb.add(static_cast<int>(f[l]), -t[l]);
        }
        rb.add(static_cast<int>(L.cell(i, j, k)), d);
        finish_row(P, rb);
        P.labels.push_back(0);
      }
    // x-faces of layer k
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        const bool has0 = i > 0, has1 = i < nx;
        face_row(L.xf(i, j, k), 0, has0 ? tx[cid(i - 1, j, k)] : 0.0, has0 ? L.cell(i - 1, j, k) : -1,
                 0, has1 ? tx[cid(i, j, k)] : 0.0, has1 ? L.cell(i, j, k) : -1);
      }
    // y-faces of layer k
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const bool has0 = j > 0, has1 = j < ny;
        face_row(L.yf(i, j, k), 0, has0 ? ty[cid(i, j - 1, k)] : 0.0, has0 ? L.cell(i, j - 1, k) : -1,
                 0, has1 ? ty[cid(i, j, k)] : 0.0, has1 ? L.cell(i, j, k) : -1);
      }
    // z-faces: bottom of layer k, plus the top boundary for the last layer
    for (int kz = k; kz <= (k == nz - 1 ? nz : k); ++kz)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          const bool has0 = kz > 0, has1 = kz < nz;
          face_row(L.zf(i, j, kz), 0, has0 ? tz[cid(i, j, kz - 1)] : 0.0,
                   has0 ? L.cell(i, j, kz - 1) : -1, 0, has1 ? tz[cid(i, j, kz)] : 0.0,
                   has1 ? L.cell(i, j, kz) : -1);
        }
  }
  if (static_cast<int64_t>(P.ptr.size()) != L.total() + 1)
    throw std::logic_error("mfd: row count mismatch");

  Uniform rhs(seed + 0x9e3779b9u);
  P.rhs.resize(P.n);
  for (int i = 0; i < P.n; ++i) P.rhs[i] = rhs(-1.0, 1.0);

  char buf[512];
  std::snprintf(buf, sizeof buf,
                "{\"problem\":\"mfd\",\"dims\":[%d,%d,%d],\"field\":\"%s\",\"sigma\":%.17g,"
                "\"seed\":%u,\"accumulation\":%.17g,\"inner_product\":\"tpfa\","
                "\"cells\":%lld,\"faces\":%lld,\"numbering\":\"slab-major-z\"}",
                nx, ny, nz, field == 1 ? "layered_lognormal" : "iid_lognormal", sigma, seed,
                accum, static_cast<long long>(ncell), static_cast<long long>(L.total() - ncell));
  P.meta = buf;
  return P;
}

// ---------------------------------------------------------------------------
// cfg3/cfg5 — compositional multiphase Jacobian with wells, restating the
// structure of proj/src/problems/comp.cpp:59-233 with the BASELINE knobs
// (SURVEY D5, D6, D9): 4 unknowns per cell (p, rho1, rho2, rho3) stored
// cell-interleaved (the 4x4 block layout), a 7-point pressure M-matrix with
// ln T ~ N(0, sigma_T^2) per face, density blocks that are mass-diagonal
// plus first-order upwind advection (per-face ratio U(0.1, 0.9) of the mass
// diagonal split over the 6 faces, so rows stay diagonally dominant), cross-
// field couplings on the own cell only, and rho3 as the strictly
// cell-diagonal volume constraint. Vertical wells: one element per layer,
// 5 dofs per element (p, rho1, rho2, rho3, rate), chained along the well,
// coupled to the perforated cells, with a rate-control row (stored zero
// diagonal) on the top element like the reference's control rows.
// Numbering is slab-major: each z-layer's cells, then (after all layers)
// the well block; the well field is never eliminated before the coarse grid.
Problem make_comp(int nx, int ny, int nz, int wells, double sigma_t, unsigned seed) {
  if (nx < 2 || ny < 2 || nz < 2) throw std::invalid_argument("comp: grid dims must be at least 2 each");
  if (wells < 0) throw std::invalid_argument("comp: negative well count");
  const int64_t N = int64_t(nx) * ny * nz;
  const int64_t Wd = int64_t(wells) * nz * 5;
  if (4 * N + Wd > INT32_MAX / 2) throw std::invalid_argument("comp: grid too large for int32 indices");
  const double acc = 1e-2, mass = 1.0, coupling = 0.1, gamma = 0.5;
  auto cid = [&](int i, int j, int k) { return int64_t(i) + int64_t(nx) * (j + int64_t(ny) * k); };
  auto dof = [&](int64_t c, int f) { return 4 * c + f; };
  const int64_t ow = 4 * N;
  auto wdof = [&](int w, int e, int f) { return ow + (int64_t(w) * nz + e) * 5 + f; };

  // face transmissibilities (x, y, z faces to the +neighbour) and upwind data
  Normal nrm(seed);
  Uniform uni(seed ^ 0x27d4eb2du);
  std::vector<double> Tf(3 * N, 0.0), rf(3 * N, 0.0);
  std::vector<signed char> upw(3 * N, 0);  // +1: cell c is upwind of its +neighbour
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int64_t c = cid(i, j, k);
        for (int d = 0; d < 3; ++d) {
          const bool has = (d == 0 && i + 1 < nx) || (d == 1 && j + 1 < ny) || (d == 2 && k + 1 < nz);
          if (!has) continue;
          Tf[3 * c + d] = std::exp(sigma_t * nrm());
          rf[3 * c + d] = uni(0.1, 0.9);
          // smooth analytic head h = cos(0.3 i) + sin(0.2 j) + 0.1 k drives the upwinding
          const double h0 = std::cos(0.3 * i) + std::sin(0.2 * j) + 0.1 * k;
          const double h1 = std::cos(0.3 * (i + (d == 0))) + std::sin(0.2 * (j + (d == 1))) + 0.1 * (k + (d == 2));
          upw[3 * c + d] = h0 >= h1 ? 1 : -1;
        }
      }
  auto nbr = [&](int i, int j, int k, int d, int sgn) -> int64_t {
    const int ii = i + (d == 0) * sgn, jj = j + (d == 1) * sgn, kk = k + (d == 2) * sgn;
    if (ii < 0 || jj < 0 || kk < 0 || ii >= nx || jj >= ny || kk >= nz) return -1;
    return cid(ii, jj, kk);
  };
  // well columns on the areal diagonal (proj/src/problems/comp.cpp:49-56)
  std::vector<std::pair<int, int>> wcol(wells);
  for (int w = 0; w < wells; ++w) {
    const int ix = std::min(int((w + 1) * int64_t(nx) / (wells + 1)), nx - 1);
    const int iy = std::min(int((w + 1) * int64_t(ny) / (wells + 1)), ny - 1);
    wcol[w] = {ix, iy};
  }
  auto perf_well = [&](int i, int j) {
    for (int w = 0; w < wells; ++w)
      if (wcol[w].first == i && wcol[w].second == j) return w;
    return -1;
  };

  Problem P;
  P.n = static_cast<int>(4 * N + Wd);
  P.fields = {"p", "rho1", "rho2", "rho3", "well"};
  if (wells == 0) P.fields.pop_back();
  P.ptr.reserve(P.n + 1);
  P.ptr.push_back(0);
  P.labels.reserve(P.n);
  RowBuilder rb;
  const double gp = gamma, g1 = 0.1 * gamma;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int64_t c = cid(i, j, k);
        const int pw = k >= 1 ? perf_well(i, j) : -1;  // layer 0 faces the control element
        // --- pressure row
        {
          double d = acc;
          for (int dd = 0; dd < 3; ++dd)
            for (int sgn : {-1, 1}) {
              const int64_t m = nbr(i, j, k, dd, sgn);
              if (m < 0) continue;
              const double T = sgn > 0 ? Tf[3 * c + dd] : Tf[3 * m + dd];
              d += T;
              rb.add(static_cast<int>(dof(m, 0)), -T);
            }
          rb.add(static_cast<int>(dof(c, 1)), coupling * acc);
          rb.add(static_cast<int>(dof(c, 2)), 0.5 * coupling * acc);
          rb.add(static_cast<int>(dof(c, 3)), 0.25 * coupling * acc);
          if (pw >= 0) {
            d += gp;
            rb.add(static_cast<int>(wdof(pw, k, 0)), -gp);
          }
          rb.add(static_cast<int>(dof(c, 0)), d);
          finish_row(P, rb);
          P.labels.push_back(0);
        }
        // --- density rows rho1, rho2 (upwind advection within the field)
        for (int f = 1; f <= 2; ++f) {
          double d = mass;
          for (int dd = 0; dd < 3; ++dd)
            for (int sgn : {-1, 1}) {
              const int64_t m = nbr(i, j, k, dd, sgn);
              if (m < 0) continue;
              const int64_t fc = sgn > 0 ? c : m;  // face owner (minus side)
              const double a = rf[3 * fc + dd] * mass / 6.0;
              const bool c_upwind = (sgn > 0) ? (upw[3 * fc + dd] > 0) : (upw[3 * fc + dd] < 0);
              if (c_upwind) d += a;                                   // outflow on the diagonal
              else rb.add(static_cast<int>(dof(m, f)), -a);          // inflow from the upwind cell
            }
          rb.add(static_cast<int>(dof(c, 0)), (f == 1 ? -1.0 : -0.5) * coupling * mass);
          if (f == 1) rb.add(static_cast<int>(dof(c, 2)), 0.5 * coupling * mass);
          else rb.add(static_cast<int>(dof(c, 1)), 0.25 * coupling * mass);
          if (pw >= 0) {
            d += (f == 1 ? g1 : 0.5 * g1);
            rb.add(static_cast<int>(wdof(pw, k, f)), -(f == 1 ? g1 : 0.5 * g1));
          }
          rb.add(static_cast<int>(dof(c, f)), d);
          finish_row(P, rb);
          P.labels.push_back(f);
        }
        // --- volume constraint rho3: strictly cell-diagonal
        rb.add(static_cast<int>(dof(c, 0)), 0.2);
        rb.add(static_cast<int>(dof(c, 1)), 0.3);
        rb.add(static_cast<int>(dof(c, 2)), 0.3);
        rb.add(static_cast<int>(dof(c, 3)), 1.0);
        finish_row(P, rb);
        P.labels.push_back(3);
      }
  // --- wells: chained elements, rate control on the top element
  for (int w = 0; w < wells; ++w) {
    const auto [ix, iy] = wcol[w];
    for (int e = 0; e < nz; ++e) {
      const int64_t c = cid(ix, iy, e);
      // pressure
      if (e == 0) {
        rb.add(static_cast<int>(wdof(w, 0, 0)), 0.0);  // stored zero diagonal (control row)
        rb.add(static_cast<int>(wdof(w, 0, 4)), 1.0);
        if (nz > 1) rb.add(static_cast<int>(wdof(w, 1, 4)), 0.25);
      } else {
        rb.add(static_cast<int>(wdof(w, e, 0)), 4.0 + gp);
        rb.add(static_cast<int>(wdof(w, e - 1, 0)), -1.0);
        if (e + 1 < nz) rb.add(static_cast<int>(wdof(w, e + 1, 0)), -1.0);
        rb.add(static_cast<int>(wdof(w, e, 4)), 1.0);
        rb.add(static_cast<int>(wdof(w, e - 1, 4)), -1.0);
        rb.add(static_cast<int>(dof(c, 0)), -gp);
      }
      finish_row(P, rb);
      P.labels.push_back(4);
      // densities
      for (int f = 1; f <= 3; ++f) {
        const double g = f == 1 ? g1 : (f == 2 ? 0.5 * g1 : 0.0);
        rb.add(static_cast<int>(wdof(w, e, f)), 3.0 + g);
        if (e > 0) rb.add(static_cast<int>(wdof(w, e - 1, f)), -0.75);
        if (e + 1 < nz) rb.add(static_cast<int>(wdof(w, e + 1, f)), -0.75);
        rb.add(static_cast<int>(wdof(w, e, 0)), 0.3);
        if (g > 0.0 && e > 0) rb.add(static_cast<int>(dof(c, f)), -g);
        finish_row(P, rb);
        P.labels.push_back(4);
      }
      // rate
      rb.add(static_cast<int>(wdof(w, e, 4)), 2.0);
      if (e > 0) rb.add(static_cast<int>(wdof(w, e - 1, 4)), -0.4);
      if (e + 1 < nz) rb.add(static_cast<int>(wdof(w, e + 1, 4)), -0.4);
      rb.add(static_cast<int>(wdof(w, e, 0)), 1.0);
      if (e + 1 < nz) rb.add(static_cast<int>(wdof(w, e + 1, 0)), -1.0);
      finish_row(P, rb);
      P.labels.push_back(4);
    }
  }
  if (static_cast<int64_t>(P.ptr.size()) != P.n + 1) throw std::logic_error("comp: row count mismatch");
  Uniform rhs(seed + 0x9e3779b9u);
  P.rhs.resize(P.n);
  for (int i = 0; i < P.n; ++i) P.rhs[i] = rhs(-1.0, 1.0);
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "{\"problem\":\"comp\",\"dims\":[%d,%d,%d],\"wells\":%d,\"well_elements\":%d,"
                "\"dofs_per_cell\":4,\"dofs_per_well_element\":5,\"sigma_lnT\":%.17g,\"seed\":%u,"
                "\"layout\":\"cell-interleaved 4x4 blocks, wells last\"}",
                nx, ny, nz, wells, nz, sigma_t, seed);
  P.meta = buf;
  return P;
}

// ---------------------------------------------------------------------------
// cfg4 — hydraulic fracturing: 3-D Q1 hex elasticity coupled to lubrication
// flow on a planar fracture, the 3-D restatement of proj/src/problems/
// frac.cpp:75-168 (2-D Q4 there). Unit cube, m^3 nodes (m per
// side), bottom (k = 0) and top (k = m-1) node planes fixed and eliminated.
// The fracture is the mid node plane km = m/2 over all (m-1)^2 face
// elements: interior plane nodes are duplicated (elements above use the
// copies), perimeter nodes are shared tips. Nondimensional units: E per
// element log-normal with median 1 (<-> 10 GPa) and sigma_lnE 0.5, nu 0.25.
// Fracture element e: pressure dof with storage c_s h^2, cubic-law
// transmissibility between neighbours T = harmonic((w/w_ref)^3 / 12),
// w ~ U(1e-4, 1e-3) m, w_ref = 1e-3. Coupling: the element pressure loads its
// face corners equally and oppositely (-/+ h^2/4 on u_z of top copy /
// original), the pressure row takes the transposed jump rate (rate/dt).
// Dofs: u node-interleaved (x, y, z) in slab-major node order (each node
// plane's originals, then for km its copies), then the fracture pressures;
// unknown_map = displacement component (0 on p), fields {u, p}.
void q1_stiffness(double h, double nu, double Ke[24][24]) {
  // isotropic D for E = 1
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), mu = 0.5 / (1.0 + nu);
  double D[6][6] = {};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) D[a][b] = lam + (a == b ? 2.0 * mu : 0.0);
  for (int a = 3; a < 6; ++a) D[a][a] = mu;
  const int sgn[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                         {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
  for (int a = 0; a < 24; ++a)
    for (int b = 0; b < 24; ++b) Ke[a][b] = 0.0;
  const double g = 1.0 / std::sqrt(3.0);
  const double jdet = (h / 2) * (h / 2) * (h / 2), dinv = 2.0 / h;
  for (int qx = -1; qx <= 1; qx += 2)
    for (int qy = -1; qy <= 1; qy += 2)
      for (int qz = -1; qz <= 1; qz += 2) {
        const double xi[3] = {qx * g, qy * g, qz * g};
        double dN[8][3];
        for (int a = 0; a < 8; ++a)
          for (int d = 0; d < 3; ++d) {
            double v = 0.125 * sgn[a][d];
            for (int e = 0; e < 3; ++e)
              if (e != d) v *= 1.0 + sgn[a][e] * xi[e];
            dN[a][d] = v * dinv;
          }
        double B[6][24] = {};
        for (int a = 0; a < 8; ++a) {
          B[0][3 * a] = dN[a][0];
          B[1][3 * a + 1] = dN[a][1];
          B[2][3 * a + 2] = dN[a][2];
          B[3][3 * a] = dN[a][1];
          B[3][3 * a + 1] = dN[a][0];
          B[4][3 * a + 1] = dN[a][2];
          B[4][3 * a + 2] = dN[a][1];
          B[5][3 * a] = dN[a][2];
          B[5][3 * a + 2] = dN[a][0];
        }
        for (int a = 0; a < 24; ++a)
          for (int b = 0; b < 24; ++b) {
            double s = 0.0;
            for (int r = 0; r < 6; ++r)
              for (int c = 0; c < 6; ++c) s += B[r][a] * D[r][c] * B[c][b];
            Ke[a][b] += s * jdet;
          }
      }
  for (int a = 0; a < 24; ++a)  // exact symmetry
    for (int b = a + 1; b < 24; ++b) Ke[a][b] = Ke[b][a] = 0.5 * (Ke[a][b] + Ke[b][a]);
}

Problem make_frac(int m, double sigma_e, unsigned seed) {
  if (m < 4 || m % 2 != 0) throw std::invalid_argument("frac: nodes per side must be even and >= 4");
  const int ne = m - 1, km = m / 2;
  const double h = 1.0 / ne, nu = 0.25;
  const int64_t nplane = int64_t(m) * m;
  auto nid = [&](int i, int j, int k) { return int64_t(i) + int64_t(m) * (j + int64_t(m) * k); };
  const int64_t nn = nplane * m;
  auto interior = [&](int i, int j) { return i > 0 && i < m - 1 && j > 0 && j < m - 1; };
  // node numbering (free nodes only): planes 1..m-2; plane km followed by copies
  std::vector<int64_t> nodeid(nn + nplane, -1);  // [0,nn): originals, [nn, nn+nplane): copies
  int64_t nf = 0;
  for (int k = 1; k < m - 1; ++k) {
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) nodeid[nid(i, j, k)] = nf++;
    if (k == km)
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i)
          if (interior(i, j)) nodeid[nn + i + int64_t(m) * j] = nf++;
  }
  const int64_t nu_dofs = 3 * nf, np = int64_t(ne) * ne;
  if (nu_dofs + np > INT32_MAX / 2) throw std::invalid_argument("frac: too large for int32 indices");

  double Ke[24][24];
  q1_stiffness(h, nu, Ke);
  Normal nrm(seed);
  Uniform uni(seed ^ 0x85ebca6bu);
  std::vector<double> E(int64_t(ne) * ne * ne);
  for (auto& e : E) e = std::exp(sigma_e * nrm());
  std::vector<double> w(np);
  for (auto& x : w) x = uni(1e-4, 1e-3);

  // node-block accumulation: per free node a small list of (col node, 3x3)
  struct Blk {
    int64_t col;
    double v[9];
  };
  std::vector<std::vector<Blk>> rows(nf);
  auto add_block = [&](int64_t r, int64_t c, const double* v9, double scale) {
    auto& R = rows[r];
    for (auto& b : R)
      if (b.col == c) {
        for (int q = 0; q < 9; ++q) b.v[q] += scale * v9[q];
        return;
      }
    Blk b;
    b.col = c;
    for (int q = 0; q < 9; ++q) b.v[q] = scale * v9[q];
    R.push_back(b);
  };
  const int off[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
  for (int ez = 0; ez < ne; ++ez)
    for (int ey = 0; ey < ne; ++ey)
      for (int ex = 0; ex < ne; ++ex) {
        int64_t nd[8];
        for (int a = 0; a < 8; ++a) {
          const int i = ex + off[a][0], j = ey + off[a][1], k = ez + off[a][2];
          int64_t g = nodeid[nid(i, j, k)];
          if (k == km && ez == km && interior(i, j)) g = nodeid[nn + i + int64_t(m) * j];  // copy above
          nd[a] = g;
        }
        const double Ee = E[ex + int64_t(ne) * (ey + int64_t(ne) * ez)];
        for (int a = 0; a < 8; ++a) {
          if (nd[a] < 0) continue;
          for (int b2 = 0; b2 < 8; ++b2) {
            if (nd[b2] < 0) continue;
            double v9[9];
            for (int r = 0; r < 3; ++r)
              for (int c = 0; c < 3; ++c) v9[3 * r + c] = Ke[3 * a + r][3 * b2 + c];
            add_block(nd[a], nd[b2], v9, Ee);
          }
        }
      }
  // fracture coupling lists: for every u_z dof, (p index, coefficient)
  std::vector<std::vector<std::pair<int64_t, double>>> up(nf);
  const double load = h * h / 4.0;
  auto fe = [&](int i, int j) { return int64_t(i) + int64_t(ne) * j; };
  for (int j = 0; j < ne; ++j)
    for (int i = 0; i < ne; ++i)
      for (int a = 0; a < 4; ++a) {
        const int ii = i + (a == 1 || a == 2), jj = j + (a >= 2);
        if (!interior(ii, jj)) continue;  // shared tip: no jump
        const int64_t top = nodeid[nn + ii + int64_t(m) * jj], bot = nodeid[nid(ii, jj, km)];
        up[top].push_back({fe(i, j), -load});
        up[bot].push_back({fe(i, j), load});
      }

  Problem P;
  P.n = static_cast<int>(nu_dofs + np);
  P.fields = {"u", "p"};
  P.ptr.reserve(P.n + 1);
  P.ptr.push_back(0);
  P.labels.reserve(P.n);
  P.unknown_map.reserve(P.n);
  RowBuilder rb;
  for (int64_t r = 0; r < nf; ++r)
    for (int cr = 0; cr < 3; ++cr) {
      for (const auto& b : rows[r])
        for (int cc = 0; cc < 3; ++cc) rb.add(static_cast<int>(3 * b.col + cc), b.v[3 * cr + cc]);
      if (cr == 2)
        for (const auto& [pe, v] : up[r]) {
          bool merged = false;
          for (auto& e : rb.e)
            if (e.first == static_cast<int>(nu_dofs + pe)) {
              e.second += v;
              merged = true;
            }
          if (!merged) rb.add(static_cast<int>(nu_dofs + pe), v);
        }
      finish_row(P, rb);
      P.labels.push_back(0);
      P.unknown_map.push_back(cr);
    }
  // pressure rows: storage + cubic-law flow + transposed jump rate
  std::vector<std::vector<std::pair<int64_t, double>>> pu(np);
  for (int64_t r = 0; r < nf; ++r)
    for (const auto& [pe, v] : up[r]) pu[pe].push_back({3 * r + 2, -v});  // rate/dt with dt = 1
  const double cs = 1e-2 * h * h;
  for (int j = 0; j < ne; ++j)
    for (int i = 0; i < ne; ++i) {
      const int64_t e = fe(i, j);
      auto kk = [&](int64_t q) { const double r = w[q] / 1e-3; return r * r * r / 12.0; };
      double d = cs;
      const int nbi[4] = {i - 1, i + 1, i, i};
      const int nbj[4] = {j, j, j - 1, j + 1};
      for (int q = 0; q < 4; ++q) {
        if (nbi[q] < 0 || nbj[q] < 0 || nbi[q] >= ne || nbj[q] >= ne) continue;
        const int64_t o = fe(nbi[q], nbj[q]);
        const double T = 2.0 * kk(e) * kk(o) / (kk(e) + kk(o));
        d += T;
        rb.add(static_cast<int>(nu_dofs + o), -T);
      }
      rb.add(static_cast<int>(nu_dofs + e), d);
      for (const auto& [c, v] : pu[e]) {
        bool merged = false;
        for (auto& x : rb.e)
          if (x.first == static_cast<int>(c)) {
            x.second += v;
            merged = true;
          }
        if (!merged) rb.add(static_cast<int>(c), v);
      }
      finish_row(P, rb);
      P.labels.push_back(1);
      P.unknown_map.push_back(0);
    }
  Uniform rhs(seed + 0x9e3779b9u);
  P.rhs.resize(P.n);
  for (int i = 0; i < P.n; ++i) P.rhs[i] = rhs(-1.0, 1.0);
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "{\"problem\":\"frac\",\"nodes_per_side\":%d,\"elements\":%lld,\"fracture_elements\":%lld,"
                "\"u_dofs\":%lld,\"sigma_lnE\":%.17g,\"nu\":0.25,\"seed\":%u,"
                "\"units\":\"nondimensional, E median 1 <-> 10 GPa\",\"bc\":\"bottom and top node planes fixed\"}",
                m, static_cast<long long>(ne) * ne * ne, static_cast<long long>(np),
                static_cast<long long>(nu_dofs), sigma_e, seed);
  P.meta = buf;
  return P;
}

}  // namespace

extern "C" {

void* mgrx_gen_frac(int m, double sigma_e, unsigned seed) {
  try {
    return new Problem(make_frac(m, sigma_e, seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* mgrx_gen_comp(int nx, int ny, int nz, int wells, double sigma_t, unsigned seed) {
  try {
    return new Problem(make_comp(nx, ny, nz, wells, sigma_t, seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

const char* mgrx_gen_last_error() { return g_err.c_str(); }

void* mgrx_gen_mfd(int nx, int ny, int nz, int field, double sigma, unsigned seed, double accum) {
  try {
    return new Problem(make_mfd(nx, ny, nz, field, sigma, seed, accum));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int mgrx_gen_n(void* h) { return static_cast<Problem*>(h)->n; }
long long mgrx_gen_nnz(void* h) { return static_cast<long long>(static_cast<Problem*>(h)->col.size()); }
int mgrx_gen_nfields(void* h) { return static_cast<int>(static_cast<Problem*>(h)->fields.size()); }
const char* mgrx_gen_field(void* h, int k) { return static_cast<Problem*>(h)->fields[k].c_str(); }
const char* mgrx_gen_meta(void* h) { return static_cast<Problem*>(h)->meta.c_str(); }
int mgrx_gen_has_unknown_map(void* h) { return static_cast<Problem*>(h)->unknown_map.empty() ? 0 : 1; }

void mgrx_gen_copy(void* h, int* ptr, int* col, double* val, int* labels, double* rhs, int* umap) {
  const Problem* P = static_cast<Problem*>(h);
  if (ptr) std::memcpy(ptr, P->ptr.data(), sizeof(int) * P->ptr.size());
  if (col) std::memcpy(col, P->col.data(), sizeof(int) * P->col.size());
  if (val) std::memcpy(val, P->val.data(), sizeof(double) * P->val.size());
  if (labels) std::memcpy(labels, P->labels.data(), sizeof(int) * P->labels.size());
  if (rhs) std::memcpy(rhs, P->rhs.data(), sizeof(double) * P->rhs.size());
  if (umap && !P->unknown_map.empty())
    std::memcpy(umap, P->unknown_map.data(), sizeof(int) * P->unknown_map.size());
}

void mgrx_gen_free(void* h) { delete static_cast<Problem*>(h); }

}  // extern "C"
