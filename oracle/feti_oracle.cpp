// =============================================================================
// oracle/feti_oracle.cpp — CPU restatement of the reference FETI-DP(H)
// range-space Schur solve.  TEST INFRASTRUCTURE ONLY.
//
// This file is the *checker* for the B200 product in paper_1312_5653_b200/.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  The product never links or calls it.
//
// It restates, line by line, the reference C++ (/root/reference/proj) without
// Eigen (which is absent from this image):
//   mesh        : src/mesh.cpp:7-36                (build_rectangle_mesh)
//   assembly    : src/fem.cpp:62-117, 119-192      (Q1 element matrices, K/V/Kc)
//   targets     : src/fem.cpp:194-220              (thermal target, boundary trace)
//   partition   : src/feti.cpp:34-169              (partition_structured)
//   blocks      : src/feti.cpp:244-364             (assemble_subdomain_operators)
//   FETI ctor   : src/feti.cpp:373-480             (coupling, coarse, equilibration)
//   FETI ops    : src/feti.cpp:483-627             (coarse_solve, split_rhs, eliminate,
//                                                   gather_jump, dual op, Dirichlet)
//   FETI solve  : src/feti.cpp:630-717
//   GMRES       : include/pdeopt/krylov.hpp:66-223 (Hermitian MGS, Givens, restarts)
//   range space : src/control.cpp:15, 113-120, 297-334
//   threads     : include/pdeopt/parallel.hpp:12-27 (fresh std::threads per call)
// Third-party arithmetic (Eigen SparseLU / PartialPivLU / SimplicialLLT, version
// unpinned in proj/CMakeLists.txt:15) is restated by published algorithms:
//   SparseLU      -> banded LU with partial pivoting (LAPACK zgbtf2/zgbtrs scheme)
//   PartialPivLU  -> dense LU with partial pivoting
//   SimplicialLLT -> banded Cholesky (small n) / Jacobi-PCG to 1e-15 (large n)
// Any exact solve agrees with Eigen's to rounding.
//   augmentation: src/feti.cpp:132-167 (edges), 171-242 (edge-RBM columns), 394-454
//                 (augmented coupling / coarse), 516-556 (eliminate), 572-578 + 655-662
//                 (dual-space projection) — the `augment` option.
// =============================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

namespace orc {

using cd = std::complex<double>;
using CVec = std::vector<cd>;
using RVec = std::vector<double>;

struct ContractError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// parallel.hpp:12-27 — spawn/join fresh threads on every call, round-robin indices.
static void parallel_for(int count, int n_threads, const std::function<void(int)>& body) {
  if (count <= 0) return;
  n_threads = std::max(1, std::min(n_threads, count));
  if (n_threads == 1) {
    for (int i = 0; i < count; ++i) body(i);
    return;
  }
  std::vector<std::thread> workers;
  workers.reserve(n_threads);
  for (int t = 0; t < n_threads; ++t)
    workers.emplace_back([&, t] {
      for (int i = t; i < count; i += n_threads) body(i);
    });
  for (auto& w : workers) w.join();
}

// ---------------------------------------------------------------- CSR (csr.hpp:60-122)
struct Trip {
  int r, c;
  double v;
};
struct Csr {
  int nr = 0, nc = 0;
  std::vector<int> off, col;
  RVec val;
  template <class S>
  void apply(const S* x, S* y) const {
    for (int r = 0; r < nr; ++r) {
      S acc{};
      for (int k = off[r]; k < off[r + 1]; ++k) acc += S(val[k]) * x[col[k]];
      y[r] = acc;
    }
  }
};
static Csr csr_from_triplets(int nr, int nc, std::vector<Trip> t) {
  std::stable_sort(t.begin(), t.end(),
                   [](const Trip& a, const Trip& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
  Csr m;
  m.nr = nr;
  m.nc = nc;
  m.off.assign(nr + 1, 0);
  std::size_t k = 0;
  for (int r = 0; r < nr; ++r) {
    while (k < t.size() && t[k].r == r) {
      const int c = t[k].c;
      double v = t[k].v;
      ++k;
      while (k < t.size() && t[k].r == r && t[k].c == c) v += t[k++].v;
      m.col.push_back(c);
      m.val.push_back(v);
    }
    m.off[r + 1] = static_cast<int>(m.col.size());
  }
  return m;
}

// ------------------------------------------------------- mesh + FEM (mesh.cpp, fem.cpp)
constexpr double kXi[4] = {-1.0, 1.0, 1.0, -1.0};
constexpr double kEta[4] = {-1.0, -1.0, 1.0, 1.0};
static double shape(int a, double xi, double eta) {
  return 0.25 * (1.0 + kXi[a] * xi) * (1.0 + kEta[a] * eta);
}
static double dsdxi(int a, double, double eta) { return 0.25 * kXi[a] * (1.0 + kEta[a] * eta); }
static double dsdeta(int a, double xi, double) { return 0.25 * kEta[a] * (1.0 + kXi[a] * xi); }
struct GP {
  double xi, eta, w;
};
static void gauss22(GP out[4]) {
  const double g = 1.0 / std::sqrt(3.0);
  out[0] = {-g, -g, 1.0};
  out[1] = {g, -g, 1.0};
  out[2] = {g, g, 1.0};
  out[3] = {-g, g, 1.0};
}

// fem.cpp:62-70
static void element_mass_heat(double h, double m[16]) {
  GP gp[4];
  gauss22(gp);
  const double detj = h * h / 4.0;
  std::fill(m, m + 16, 0.0);
  for (auto& g : gp)
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b)
        m[a * 4 + b] += g.w * shape(a, g.xi, g.eta) * shape(b, g.xi, g.eta) * detj;
}
// fem.cpp:72-81
static void element_stiffness_heat(double k[16]) {
  GP gp[4];
  gauss22(gp);
  std::fill(k, k + 16, 0.0);
  for (auto& g : gp)
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b)
        k[a * 4 + b] += g.w * (dsdxi(a, g.xi, g.eta) * dsdxi(b, g.xi, g.eta) +
                               dsdeta(a, g.xi, g.eta) * dsdeta(b, g.xi, g.eta));
}
// fem.cpp:83-90
static void element_mass_elastic(double h, double m[64]) {
  double s[16];
  element_mass_heat(h, s);
  std::fill(m, m + 64, 0.0);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      for (int c = 0; c < 2; ++c) m[(2 * a + c) * 8 + 2 * b + c] = s[a * 4 + b];
}
// fem.cpp:92-117
static void element_stiffness_plane_strain(double e, double nu, double h, double k[64]) {
  const double f = e / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double d[3][3] = {{f * (1.0 - nu), f * nu, 0.0},
                          {f * nu, f * (1.0 - nu), 0.0},
                          {0.0, 0.0, f * (1.0 - 2.0 * nu) / 2.0}};
  GP gp[4];
  gauss22(gp);
  std::fill(k, k + 64, 0.0);
  const double detj = h * h / 4.0, gs = 2.0 / h;
  for (auto& g : gp) {
    double b[3][8] = {};
    for (int a = 0; a < 4; ++a) {
      const double dx = gs * dsdxi(a, g.xi, g.eta), dy = gs * dsdeta(a, g.xi, g.eta);
      b[0][2 * a] = dx;
      b[1][2 * a + 1] = dy;
      b[2][2 * a] = dy;
      b[2][2 * a + 1] = dx;
    }
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double acc = 0.0;
        for (int p = 0; p < 3; ++p)
          for (int q = 0; q < 3; ++q) acc += b[p][i] * d[p][q] * b[q][j];
        k[i * 8 + j] += g.w * detj * acc;
      }
  }
}

// ---- 3D extension (BASELINE.json configs 4-5; the reference is 2D only, SURVEY.md §0 F5,
// §7 step 7).  Trilinear Q1 hexahedra, 2x2x2 Gauss (exact for the Q1 mass and stiffness),
// local nodes counterclockwise in the bottom face then the top face (the 2D order of
// mesh.cpp:31-34 extruded), 3 interleaved dofs per node for elasticity (fem.cpp:171).
constexpr double kXi3[8] = {-1, 1, 1, -1, -1, 1, 1, -1};
constexpr double kEta3[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
constexpr double kZeta3[8] = {-1, -1, -1, -1, 1, 1, 1, 1};
static void shape3(int a, double x, double y, double z, double& n, double& dx, double& dy, double& dz) {
  const double fx = 1.0 + kXi3[a] * x, fy = 1.0 + kEta3[a] * y, fz = 1.0 + kZeta3[a] * z;
  n = 0.125 * fx * fy * fz;
  dx = 0.125 * kXi3[a] * fy * fz;
  dy = 0.125 * kEta3[a] * fx * fz;
  dz = 0.125 * kZeta3[a] * fx * fy;
}
static void element_heat3d(double h, double k[64], double m[64]) {
  const double g = 1.0 / std::sqrt(3.0), pts[2] = {-g, g};
  const double detj = h * h * h / 8.0, gs = 2.0 / h;
  std::fill(k, k + 64, 0.0);
  std::fill(m, m + 64, 0.0);
  for (double z : pts)
    for (double y : pts)
      for (double x : pts) {
        double n[8], dx[8], dy[8], dz[8];
        for (int a = 0; a < 8; ++a) shape3(a, x, y, z, n[a], dx[a], dy[a], dz[a]);
        for (int a = 0; a < 8; ++a)
          for (int b = 0; b < 8; ++b) {
            m[a * 8 + b] += n[a] * n[b] * detj;
            k[a * 8 + b] += (dx[a] * dx[b] + dy[a] * dy[b] + dz[a] * dz[b]) * gs * gs * detj;
          }
      }
}
static void element_elastic3d(double e, double nu, double h, double k[576], double m[576]) {
  const double f = e / ((1.0 + nu) * (1.0 - 2.0 * nu));
  double d[6][6] = {};
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) d[p][q] = f * (p == q ? 1.0 - nu : nu);
  for (int p = 3; p < 6; ++p) d[p][p] = f * (1.0 - 2.0 * nu) / 2.0;
  const double g = 1.0 / std::sqrt(3.0), pts[2] = {-g, g};
  const double detj = h * h * h / 8.0, gs = 2.0 / h;
  std::fill(k, k + 576, 0.0);
  for (double z : pts)
    for (double y : pts)
      for (double x : pts) {
        double b[6][24] = {};
        for (int a = 0; a < 8; ++a) {
          double n, dx, dy, dz;
          shape3(a, x, y, z, n, dx, dy, dz);
          dx *= gs, dy *= gs, dz *= gs;
          b[0][3 * a] = dx;
          b[1][3 * a + 1] = dy;
          b[2][3 * a + 2] = dz;
          b[3][3 * a] = dy, b[3][3 * a + 1] = dx;
          b[4][3 * a + 1] = dz, b[4][3 * a + 2] = dy;
          b[5][3 * a] = dz, b[5][3 * a + 2] = dx;
        }
        for (int i = 0; i < 24; ++i)
          for (int j = i; j < 24; ++j) {
            double acc = 0.0;
            for (int p = 0; p < 6; ++p)
              for (int q = 0; q < 6; ++q) acc += b[p][i] * d[p][q] * b[q][j];
            k[i * 24 + j] += detj * acc;
          }
      }
  for (int i = 0; i < 24; ++i)  // exactly symmetric
    for (int j = 0; j < i; ++j) k[i * 24 + j] = k[j * 24 + i];
  double kh[64], mh[64];
  element_heat3d(h, kh, mh);
  std::fill(m, m + 576, 0.0);
  for (int a = 0; a < 8; ++a)
    for (int b2 = 0; b2 < 8; ++b2)
      for (int c = 0; c < 3; ++c) m[(3 * a + c) * 24 + 3 * b2 + c] = mh[a * 8 + b2];
}

struct Problem {
  int nx = 0, ny = 0, nz = 0, dpn = 1, physics = 0;  // physics 0 = heat, 1 = plane strain / 3D elasticity
  double h = 0, lx = 1, ly = 1, lz = 0, E = 0, nu = 0;  // nz = 0: 2D (the reference), nz > 0: 3D
  std::vector<int> free_map, cons_map, free_dofs, cons_dofs;
  Csr K, V, Kc;
  double mass_sum = 0;
  double ke[576], me[576];
  int edofs = 4;
  int n() const { return K.nr; }
  int m() const { return Kc.nc; }
  bool is3d() const { return nz > 0; }
  int npe() const { return nz > 0 ? 8 : 4; }
  int node_id(int i, int j, int k = 0) const { return (k * (ny + 1) + j) * (nx + 1) + i; }
  double node_x(int id) const { return (id % (nx + 1)) * h; }
  double node_y(int id) const { return ((id / (nx + 1)) % (ny + 1)) * h; }
  double node_z(int id) const { return (id / ((nx + 1) * (ny + 1))) * h; }
  void elem_nodes(int e, int out[8]) const {
    const int i = e % nx, j = (e / nx) % ny, k = nz > 0 ? e / (nx * ny) : 0;  // mesh.cpp:31-34, counterclockwise
    out[0] = node_id(i, j, k);
    out[1] = node_id(i + 1, j, k);
    out[2] = node_id(i + 1, j + 1, k);
    out[3] = node_id(i, j + 1, k);
    if (nz > 0) {
      out[4] = node_id(i, j, k + 1);
      out[5] = node_id(i + 1, j, k + 1);
      out[6] = node_id(i + 1, j + 1, k + 1);
      out[7] = node_id(i, j + 1, k + 1);
    }
  }
  int n_elems() const { return nx * ny * (nz > 0 ? nz : 1); }
};

// mesh.cpp:7-36 + fem.cpp:119-192 (nz = 0); the 3D extension with nz > 0: whole-boundary
// Dirichlet for heat, clamped face x = 0 for elasticity (BASELINE.json configs 4-5)
static Problem* build_problem_any(int nx, int ny, int nz, double lx, double ly, double lz, int physics, double E,
                                  double nu) {
  const bool d3 = nz > 0;
  if (nx < 2 || ny < 2 || (d3 && nz < 2)) throw ContractError("build_rectangle_mesh: need at least 2 elements per axis");
  if (lx <= 0 || ly <= 0 || (d3 && lz <= 0)) throw ContractError("build_rectangle_mesh: non-positive extent");
  const double hx = lx / nx, hy = ly / ny, hz = d3 ? lz / nz : hx;
  if (std::abs(hx - hy) > 1e-12 * std::max(hx, hy) || std::abs(hx - hz) > 1e-12 * std::max(hx, hz))
    throw ContractError("build_rectangle_mesh: elements must be square");
  auto p = std::make_unique<Problem>();
  p->nx = nx;
  p->ny = ny;
  p->nz = d3 ? nz : 0;
  p->lx = lx;
  p->ly = ly;
  p->lz = d3 ? lz : 0.0;
  p->h = hx;
  p->physics = physics;
  p->E = E;
  p->nu = nu;
  p->dpn = physics == 0 ? 1 : (d3 ? 3 : 2);
  const int dpn = p->dpn;
  if (physics != 0) {
    if (!(nu > 0.0 && nu < 0.5)) throw ContractError("Physics: poisson_ratio must lie strictly in (0, 0.5)");
    if (E <= 0.0) throw ContractError("Physics: young_modulus must be positive");
  }
  if (!d3 && physics == 0) {
    element_stiffness_heat(p->ke);
    element_mass_heat(p->h, p->me);
  } else if (!d3) {
    element_stiffness_plane_strain(E, nu, p->h, p->ke);
    element_mass_elastic(p->h, p->me);
  } else if (physics == 0) {
    element_heat3d(p->h, p->ke, p->me);
  } else {
    element_elastic3d(E, nu, p->h, p->ke, p->me);
  }
  p->edofs = p->npe() * dpn;
  const int nzz = d3 ? nz : 0;
  const int nn = (nx + 1) * (ny + 1) * (nzz + 1), nmd = nn * dpn;
  std::vector<char> cons(nmd, 0);
  for (int k = 0; k <= nzz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        const int node = p->node_id(i, j, k);
        if (physics == 0) {  // whole boundary (fem.cpp:121-122)
          if (i == 0 || i == nx || j == 0 || j == ny || (d3 && (k == 0 || k == nz))) cons[node] = 1;
        } else if (i == 0) {  // clamped x = 0 (fem.cpp:124-128)
          for (int c = 0; c < dpn; ++c) cons[dpn * node + c] = 1;
        }
      }
  p->free_map.assign(nmd, -1);
  p->cons_map.assign(nmd, -1);
  for (int d = 0; d < nmd; ++d) {
    if (cons[d]) {
      p->cons_map[d] = (int)p->cons_dofs.size();
      p->cons_dofs.push_back(d);
    } else {
      p->free_map[d] = (int)p->free_dofs.size();
      p->free_dofs.push_back(d);
    }
  }
  const int n = (int)p->free_dofs.size(), m = (int)p->cons_dofs.size();
  const int ed = p->edofs, npe = p->npe();
  std::vector<Trip> tk, tv, tkc;
  tk.reserve((size_t)p->n_elems() * ed * ed);
  tv.reserve(tk.capacity());
  int gd[24], en[8];
  for (int e = 0; e < p->n_elems(); ++e) {
    p->elem_nodes(e, en);
    for (int a = 0; a < npe; ++a)
      for (int c = 0; c < dpn; ++c) gd[dpn * a + c] = dpn * en[a] + c;
    for (int a = 0; a < ed; ++a) {
      const int fa = p->free_map[gd[a]];
      for (int b = 0; b < ed; ++b) {
        p->mass_sum += p->me[a * ed + b];
        if (fa < 0) continue;
        const int fb = p->free_map[gd[b]];
        if (fb >= 0) {
          tk.push_back({fa, fb, p->ke[a * ed + b]});
          tv.push_back({fa, fb, p->me[a * ed + b]});
        } else {
          tkc.push_back({fa, p->cons_map[gd[b]], p->ke[a * ed + b]});
        }
      }
    }
  }
  p->K = csr_from_triplets(n, n, std::move(tk));
  p->V = csr_from_triplets(n, n, std::move(tv));
  p->Kc = csr_from_triplets(n, m, std::move(tkc));
  return p.release();
}
static Problem* build_problem(int nx, int ny, double lx, double ly, int physics, double E, double nu) {
  return build_problem_any(nx, ny, 0, lx, ly, 0.0, physics, E, nu);
}

// fem.cpp:194-202
static double evaluate_target_thermal(double x1, double x2) {
  if (x1 <= 0.5 && x2 <= 0.5) {
    const double a = 2.0 * x1 - 1.0, b = 2.0 * x2 - 1.0;
    return a * a * b * b;
  }
  return 0.0;
}

// Seeded sine-mode target of BASELINE.json configs 1-3 (new: the reference's
// ExperimentConfig::seed is never consumed).  The generator is
// specified in SURVEY.md §8(d): std::mt19937_64(seed); per mode k: a_k by explicit
// Box-Muller on two U(0,1) draws, then m_k = 1 + rng() % M, n_k = 1 + rng() % M.
// The product restates the same recipe independently (csrc/host_core.cpp) and the
// tests compare the two bit for bit.
static double u01(std::mt19937_64& g) { return (double)(g() >> 11) * (1.0 / 9007199254740992.0); }
static void sine_modes(uint64_t seed, int modes, int mmax, double* a, int* m, int* nn) {
  std::mt19937_64 g(seed);
  for (int k = 0; k < modes; ++k) {
    const double u1 = u01(g), u2 = u01(g);
    a[k] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
    m[k] = 1 + (int)(g() % (uint64_t)mmax);
    nn[k] = 1 + (int)(g() % (uint64_t)mmax);
  }
}

// ------------------------------------------------------------ partition (feti.cpp:34-169)
struct Sub {
  std::vector<int> elements, dofs, corner_local, corner_global, r_local, r_interior, r_boundary;
  // signed Boolean jump entries B^s(row, rpos) = sign.  In 2D every interface dof has exactly
  // one multiplier row, so entry k is boundary dof k (feti.cpp:98-121).  In 3D a dof on a
  // subdomain edge (multiplicity 4) is in 3 rows of this subdomain: lambda_bidx[k] is the
  // boundary index and lambda_rpos[k] the r-position of entry k.
  std::vector<int> lambda_rows, lambda_rpos, lambda_bidx;
  RVec lambda_signs, weights;
};
struct Edge {  // feti.hpp:59-65: open segment between subdomain-grid vertices
  int sub_lo = 0, sub_hi = 0;
  bool vertical = false;
  std::vector<int> nodes, lambda_rows;  // dpn rows per node
};
struct Partition {
  int sx = 0, sy = 0, ex = 0, ey = 0, dpn = 1, n_free = 0, n_corner = 0, n_lambda = 0, n_edges = 0;
  int sz = 1, ez = 0;  // 3D extension (sz = 1, ez = 0 in 2D)
  double h = 0;
  // Dirichlet-preconditioner scaling W of each multiplier row: 1/multiplicity of its node
  // (the reference hard-codes W = 1/2, feti.cpp:602, 626, which is 1/mult in 2D)
  RVec lam_weight;
  std::vector<Sub> subs;
  std::vector<int> free_mult;
  std::vector<Edge> edges;
};
static std::pair<int, int> owner_range(int i, int e, int ns) {
  const int lo = (i == 0) ? 0 : (i - 1) / e;
  const int hi = std::min(ns - 1, i / e);
  return {lo, hi};
}
static Partition partition_structured(const Problem& P, int sx, int sy) {
  if (sx < 1 || sy < 1 || sx * sy < 2) throw ContractError("partition_structured: need at least two subdomains");
  if (P.nx % sx != 0 || P.ny % sy != 0)
    throw ContractError("partition_structured: subdomain grid must divide the element grid");
  const int ex = P.nx / sx, ey = P.ny / sy;
  if (ex < 2 || ey < 2) throw ContractError("partition_structured: H/h must be at least 2");
  const int dpn = P.dpn;
  Partition part;
  part.sx = sx;
  part.sy = sy;
  part.ex = ex;
  part.ey = ey;
  part.dpn = dpn;
  part.n_free = P.n();
  const int nn = (P.nx + 1) * (P.ny + 1);
  std::vector<int> mult(nn, 0);
  std::vector<char> corner(nn, 0);
  for (int j = 0; j <= P.ny; ++j) {
    auto [qlo, qhi] = owner_range(j, ey, sy);
    for (int i = 0; i <= P.nx; ++i) {
      auto [plo, phi] = owner_range(i, ex, sx);
      const int node = P.node_id(i, j);
      mult[node] = (phi - plo + 1) * (qhi - qlo + 1);
      const bool fr = P.free_map[node * dpn] >= 0;
      corner[node] = (i % ex == 0) && (j % ey == 0) && mult[node] >= 2 && fr;
    }
  }
  std::vector<int> corner_of(nn * dpn, -1), lambda_of(nn * dpn, -1);
  for (int node = 0; node < nn; ++node) {
    if (P.free_map[node * dpn] < 0) continue;
    if (corner[node]) {
      for (int c = 0; c < dpn; ++c) corner_of[node * dpn + c] = part.n_corner++;
    } else if (mult[node] >= 2) {
      if (mult[node] != 2) throw NumericalError("partition_structured: unexpected interface multiplicity");
      for (int c = 0; c < dpn; ++c) lambda_of[node * dpn + c] = part.n_lambda++;
    }
  }
  part.free_mult.assign(part.n_free, 1);
  for (int node = 0; node < nn; ++node)
    for (int c = 0; c < dpn; ++c) {
      const int f = P.free_map[node * dpn + c];
      if (f >= 0) part.free_mult[f] = mult[node];
    }
  part.subs.resize(sx * sy);
  for (int q = 0; q < sy; ++q)
    for (int p = 0; p < sx; ++p) {
      const int sid = q * sx + p;
      Sub& s = part.subs[sid];
      for (int j = q * ey; j < (q + 1) * ey; ++j)
        for (int i = p * ex; i < (p + 1) * ex; ++i) s.elements.push_back(j * P.nx + i);
      for (int j = q * ey; j <= (q + 1) * ey; ++j)
        for (int i = p * ex; i <= (p + 1) * ex; ++i) {
          const int node = P.node_id(i, j);
          for (int c = 0; c < dpn; ++c) {
            const int md = node * dpn + c, f = P.free_map[md];
            if (f < 0) continue;
            const int local = (int)s.dofs.size();
            s.dofs.push_back(f);
            s.weights.push_back(1.0 / mult[node]);
            if (corner[node]) {
              s.corner_local.push_back(local);
              s.corner_global.push_back(corner_of[md]);
            } else {
              const int rpos = (int)s.r_local.size();
              s.r_local.push_back(local);
              if (lambda_of[md] >= 0) {
                s.lambda_bidx.push_back((int)s.r_boundary.size());
                s.lambda_rpos.push_back(rpos);
                s.r_boundary.push_back(rpos);
                s.lambda_rows.push_back(lambda_of[md]);
                auto [plo2, phi2] = owner_range(i, ex, sx);
                auto [qlo2, qhi2] = owner_range(j, ey, sy);
                (void)phi2;
                (void)qhi2;
                s.lambda_signs.push_back(sid == qlo2 * sx + plo2 ? 1.0 : -1.0);
              } else {
                s.r_interior.push_back(rpos);
              }
            }
          }
        }
    }
  // edges (feti.cpp:132-167): vertical cuts first (row q, cut p), then horizontal cuts;
  // only free nodes strictly inside the segment; empty segments are dropped
  part.h = P.h;
  auto add_edge = [&](Edge e) {
    for (int node : e.nodes)
      for (int c = 0; c < dpn; ++c) e.lambda_rows.push_back(lambda_of[node * dpn + c]);
    if (!e.nodes.empty()) part.edges.push_back(std::move(e));
  };
  for (int q = 0; q < sy; ++q)
    for (int p = 1; p < sx; ++p) {
      Edge e;
      e.vertical = true;
      e.sub_lo = q * sx + p - 1;
      e.sub_hi = q * sx + p;
      for (int j = q * ey + 1; j < (q + 1) * ey; ++j)
        if (P.free_map[P.node_id(p * ex, j) * dpn] >= 0) e.nodes.push_back(P.node_id(p * ex, j));
      add_edge(std::move(e));
    }
  for (int q = 1; q < sy; ++q)
    for (int p = 0; p < sx; ++p) {
      Edge e;
      e.vertical = false;
      e.sub_lo = (q - 1) * sx + p;
      e.sub_hi = q * sx + p;
      for (int i = p * ex + 1; i < (p + 1) * ex; ++i)
        if (P.free_map[P.node_id(i, q * ey) * dpn] >= 0) e.nodes.push_back(P.node_id(i, q * ey));
      add_edge(std::move(e));
    }
  part.n_edges = (int)part.edges.size();
  part.lam_weight.assign(part.n_lambda, 0.5);
  return part;
}

// 3D extension of partition_structured (new: the reference rejects multiplicity 4,
// feti.cpp:76-78).  Same corner rule (subdomain-grid vertices that are free with
// multiplicity >= 2), same +1-for-the-lower-subdomain sign rule, applied pairwise: a
// non-corner interface dof shared by subdomains s_1 < ... < s_m gets one row per pair
// (s_a, s_b), a < b (fully redundant multipliers; m = 2 on faces, 4 on subdomain edges).
// Rows ascend by (node, component, pair); the Dirichlet scaling is W = 1/m per row.
static Partition partition_structured3d(const Problem& P, int sx, int sy, int sz) {
  if (!P.is3d()) throw ContractError("partition_structured3d: 2D problem");
  if (sx < 1 || sy < 1 || sz < 1 || sx * sy * sz < 2) throw ContractError("partition_structured: need at least two subdomains");
  if (P.nx % sx != 0 || P.ny % sy != 0 || P.nz % sz != 0)
    throw ContractError("partition_structured: subdomain grid must divide the element grid");
  const int ex = P.nx / sx, ey = P.ny / sy, ez = P.nz / sz;
  if (ex < 2 || ey < 2 || ez < 2) throw ContractError("partition_structured: H/h must be at least 2");
  const int dpn = P.dpn;
  Partition part;
  part.sx = sx, part.sy = sy, part.sz = sz;
  part.ex = ex, part.ey = ey, part.ez = ez;
  part.dpn = dpn;
  part.n_free = P.n();
  part.h = P.h;
  const int nn = (P.nx + 1) * (P.ny + 1) * (P.nz + 1);
  std::vector<int> mult(nn, 0);
  std::vector<char> corner(nn, 0);
  auto owners = [&](int node) {
    const int i = node % (P.nx + 1), j = (node / (P.nx + 1)) % (P.ny + 1), k = node / ((P.nx + 1) * (P.ny + 1));
    auto [plo, phi] = owner_range(i, ex, sx);
    auto [qlo, qhi] = owner_range(j, ey, sy);
    auto [rlo, rhi] = owner_range(k, ez, sz);
    std::vector<int> o;
    for (int r = rlo; r <= rhi; ++r)
      for (int q = qlo; q <= qhi; ++q)
        for (int p = plo; p <= phi; ++p) o.push_back((r * sy + q) * sx + p);  // ascending
    return o;
  };
  for (int k = 0; k <= P.nz; ++k)
    for (int j = 0; j <= P.ny; ++j)
      for (int i = 0; i <= P.nx; ++i) {
        const int node = P.node_id(i, j, k);
        auto [plo, phi] = owner_range(i, ex, sx);
        auto [qlo, qhi] = owner_range(j, ey, sy);
        auto [rlo, rhi] = owner_range(k, ez, sz);
        mult[node] = (phi - plo + 1) * (qhi - qlo + 1) * (rhi - rlo + 1);
        const bool fr = P.free_map[node * dpn] >= 0;
        corner[node] = (i % ex == 0) && (j % ey == 0) && (k % ez == 0) && mult[node] >= 2 && fr;
      }
  // rows of node*dpn+c: first row id and the owner list (pairs in lexicographic order)
  std::vector<int> corner_of(nn * dpn, -1), lambda0(nn * dpn, -1);
  for (int node = 0; node < nn; ++node) {
    if (P.free_map[node * dpn] < 0) continue;
    if (corner[node]) {
      for (int c = 0; c < dpn; ++c) corner_of[node * dpn + c] = part.n_corner++;
    } else if (mult[node] >= 2) {
      const int m = mult[node], pairs = m * (m - 1) / 2;
      for (int c = 0; c < dpn; ++c) {
        lambda0[node * dpn + c] = part.n_lambda;
        part.n_lambda += pairs;
        for (int q = 0; q < pairs; ++q) part.lam_weight.push_back(1.0 / m);
      }
    }
  }
  part.free_mult.assign(part.n_free, 1);
  for (int node = 0; node < nn; ++node)
    for (int c = 0; c < dpn; ++c) {
      const int f = P.free_map[node * dpn + c];
      if (f >= 0) part.free_mult[f] = mult[node];
    }
  part.subs.resize(sx * sy * sz);
  for (int r = 0; r < sz; ++r)
    for (int q = 0; q < sy; ++q)
      for (int p = 0; p < sx; ++p) {
        const int sid = (r * sy + q) * sx + p;
        Sub& s = part.subs[sid];
        for (int k = r * ez; k < (r + 1) * ez; ++k)
          for (int j = q * ey; j < (q + 1) * ey; ++j)
            for (int i = p * ex; i < (p + 1) * ex; ++i) s.elements.push_back((k * P.ny + j) * P.nx + i);
        for (int k = r * ez; k <= (r + 1) * ez; ++k)
          for (int j = q * ey; j <= (q + 1) * ey; ++j)
            for (int i = p * ex; i <= (p + 1) * ex; ++i) {
              const int node = P.node_id(i, j, k);
              std::vector<int> own;
              if (mult[node] >= 2 && !corner[node]) own = owners(node);
              for (int c = 0; c < dpn; ++c) {
                const int md = node * dpn + c, f = P.free_map[md];
                if (f < 0) continue;
                const int local = (int)s.dofs.size();
                s.dofs.push_back(f);
                s.weights.push_back(1.0 / mult[node]);
                if (corner[node]) {
                  s.corner_local.push_back(local);
                  s.corner_global.push_back(corner_of[md]);
                  continue;
                }
                const int rpos = (int)s.r_local.size();
                s.r_local.push_back(local);
                if (lambda0[md] < 0) {
                  s.r_interior.push_back(rpos);
                  continue;
                }
                const int bidx = (int)s.r_boundary.size();
                s.r_boundary.push_back(rpos);
                int row = lambda0[md];
                for (size_t a = 0; a < own.size(); ++a)
                  for (size_t b = a + 1; b < own.size(); ++b, ++row) {
                    if (own[a] != sid && own[b] != sid) continue;
                    s.lambda_rows.push_back(row);
                    s.lambda_rpos.push_back(rpos);
                    s.lambda_bidx.push_back(bidx);
                    s.lambda_signs.push_back(own[a] == sid ? 1.0 : -1.0);
                  }
              }
            }
      }
  part.n_edges = 0;  // edge-RBM augmentation is 2D only
  return part;
}
static Partition partition_any(const Problem& P, int sx, int sy, int sz) {
  return P.is3d() ? partition_structured3d(P, sx, sy, sz) : partition_structured(P, sx, sy);
}

// ------------------------------------------- edge-RBM augmentation (feti.cpp:171-242)
// One normalised column per edge for scalar physics (the edge mean); for plane strain the
// two translations and the in-plane rotation about the edge midpoint.
struct AugColumn {
  std::vector<int> rows;
  RVec values;
};
static std::vector<AugColumn> edge_rbm_columns(const Partition& part) {
  std::vector<AugColumn> cols;
  for (size_t e = 0; e < part.edges.size(); ++e) {
    const Edge& ed = part.edges[e];
    const int nn = (int)ed.nodes.size();
    std::vector<AugColumn> mine;
    if (part.dpn == 1) {
      AugColumn c;
      c.rows = ed.lambda_rows;
      c.values.assign(nn, 1.0);
      mine.push_back(std::move(c));
    } else {
      AugColumn tx, ty, rot;
      for (int k = 0; k < nn; ++k) {
        const int rx = ed.lambda_rows[2 * k], ry = ed.lambda_rows[2 * k + 1];
        tx.rows.push_back(rx);
        tx.values.push_back(1.0);
        ty.rows.push_back(ry);
        ty.values.push_back(1.0);
        const double arm = (k - 0.5 * (nn - 1)) * part.h;  // offset from the edge midpoint
        rot.rows.push_back(ed.vertical ? rx : ry);
        rot.values.push_back(ed.vertical ? -arm : arm);
      }
      mine.push_back(std::move(tx));
      mine.push_back(std::move(ty));
      mine.push_back(std::move(rot));
    }
    for (auto& c : mine) {
      double n2 = 0;
      for (double v : c.values) n2 += v * v;
      if (!(n2 > 0.0))
        throw NumericalError("build_edge_rbm_augmentation: dependent (zero) column on edge " + std::to_string(e) +
                             "; H/h too small for a rotation mode");
      const double inv = 1.0 / std::sqrt(n2);
      for (double& v : c.values) v *= inv;
    }
    for (size_t a = 0; a < mine.size(); ++a)
      for (size_t b = a + 1; b < mine.size(); ++b) {
        double dot = 0;
        for (size_t i = 0; i < mine[a].rows.size(); ++i)
          for (size_t j = 0; j < mine[b].rows.size(); ++j)
            if (mine[a].rows[i] == mine[b].rows[j]) dot += mine[a].values[i] * mine[b].values[j];
        if (std::abs(dot) > 1e-12)
          throw NumericalError("build_edge_rbm_augmentation: dependent columns on edge " + std::to_string(e));
      }
    for (auto& c : mine) cols.push_back(std::move(c));
  }
  return cols;
}

// --------------------------------------- banded LU with partial pivoting (zgbtf2/zgbtrs)
// g_band_ldlt (orc_set_band_ldlt, test infrastructure): factor the subdomain blocks by a
// symmetric band LDL^T (no pivoting; only the lower band stored, kl + 1 rows) instead.  The
// blocks K + cV are complex symmetric with SPD real part K, so the pivot-free factorization is
// stable; it is an exact solve like the pivoted LU (results agree to rounding) with a third
// of the memory -- what lets the 3D restatement run BASELINE configs 4-5 at full size.
static bool g_band_ldlt = false;
struct BandLU {
  int n = 0, kl = 0, ku = 0, ld = 0;
  bool sym = false;
  CVec ab;  // column-major LAPACK band layout with kl extra fill rows (sym: lower band only)
  std::vector<int> piv;
  cd& at(int i, int j) { return sym ? ab[(size_t)j * ld + (i - j)] : ab[(size_t)j * ld + (kl + ku + i - j)]; }
  const cd& at(int i, int j) const {
    return sym ? ab[(size_t)j * ld + (i - j)] : ab[(size_t)j * ld + (kl + ku + i - j)];
  }
  void add(int i, int j, cd v) {  // assembly: the upper triangle is implied in sym mode
    if (!sym || i >= j) at(i, j) += v;
  }
  void init(int n_, int kl_, int ku_) {
    n = n_;
    kl = kl_;
    ku = ku_;
    sym = g_band_ldlt && kl == ku;
    ld = sym ? kl + 1 : 2 * kl + ku + 1;
    ab.assign((size_t)ld * std::max(n, 1), cd(0));
    piv.assign(sym ? 0 : n, 0);
  }
  bool factor() {
    if (sym) return factor_ldlt();
    const int kv = ku + kl;
    int ju = 0;
    for (int j = 0; j < n; ++j) {
      const int km = std::min(kl, n - 1 - j);
      int p = j;
      double best = std::abs(at(j, j));
      for (int i = j + 1; i <= j + km; ++i)
        if (std::abs(at(i, j)) > best) {
          best = std::abs(at(i, j));
          p = i;
        }
      piv[j] = p;
      if (!(best > 0.0) || !std::isfinite(best)) return false;
      ju = std::max(ju, std::min(j + ku + p - j, n - 1));
      if (p != j)
        for (int c = j; c <= ju; ++c) std::swap(at(j, c), at(p, c));
      const cd inv = cd(1) / at(j, j);
      for (int i = j + 1; i <= j + km; ++i) at(i, j) *= inv;
      for (int c = j + 1; c <= ju; ++c) {
        const cd u = at(j, c);
        if (u == cd(0)) continue;
        for (int i = j + 1; i <= j + km; ++i) at(i, c) -= at(i, j) * u;
      }
      (void)kv;
    }
    return true;
  }
  bool factor_ldlt() {  // A = L D L^T (transpose, not adjoint: complex symmetric)
    std::vector<cd> t(kl + 1);
    for (int j = 0; j < n; ++j) {
      cd* cj = &ab[(size_t)j * ld];
      const cd d = cj[0];
      if (!(std::abs(d) > 0.0) || !std::isfinite(std::abs(d))) return false;
      const int m = std::min(kl, n - 1 - j);
      const cd inv = cd(1) / d;
      for (int i = 1; i <= m; ++i) {
        t[i] = cj[i];
        cj[i] *= inv;
      }
      for (int c = 1; c <= m; ++c) {  // column j+c, rows j+c..j+m: a(i,k) -= l_i t_k
        cd* dst = &ab[(size_t)(j + c) * ld];
        const cd tc = t[c];
        for (int i = c; i <= m; ++i) dst[i - c] -= cj[i] * tc;
      }
    }
    return true;
  }
  void solve(cd* b) const {
    if (sym) {
      for (int j = 0; j < n; ++j) {
        const cd* cj = &ab[(size_t)j * ld];
        const int m = std::min(kl, n - 1 - j);
        const cd bj = b[j];
        for (int i = 1; i <= m; ++i) b[j + i] -= cj[i] * bj;
      }
      for (int j = 0; j < n; ++j) b[j] /= ab[(size_t)j * ld];
      for (int j = n - 1; j >= 0; --j) {
        const cd* cj = &ab[(size_t)j * ld];
        const int m = std::min(kl, n - 1 - j);
        cd acc = b[j];
        for (int i = 1; i <= m; ++i) acc -= cj[i] * b[j + i];
        b[j] = acc;
      }
      return;
    }
    for (int j = 0; j < n; ++j) {
      const int km = std::min(kl, n - 1 - j);
      if (piv[j] != j) std::swap(b[j], b[piv[j]]);
      const cd bj = b[j];
      for (int i = j + 1; i <= j + km; ++i) b[i] -= at(i, j) * bj;
    }
    const int kv = kl + ku;
    for (int j = n - 1; j >= 0; --j) {
      b[j] /= at(j, j);
      const cd bj = b[j];
      for (int i = std::max(0, j - kv); i < j; ++i) b[i] -= at(i, j) * bj;
    }
  }
};

// dense LU with partial pivoting (Eigen::PartialPivLU restated), row-major n x n
struct DenseLU {
  int n = 0;
  CVec a;
  std::vector<int> perm;
  void factor(const CVec& m, int n_) {
    n = n_;
    a = m;
    perm.resize(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int k = 0; k < n; ++k) {
      int p = k;
      double best = std::abs(a[(size_t)k * n + k]);
      for (int i = k + 1; i < n; ++i)
        if (std::abs(a[(size_t)i * n + k]) > best) {
          best = std::abs(a[(size_t)i * n + k]);
          p = i;
        }
      if (p != k) {
        for (int c = 0; c < n; ++c) std::swap(a[(size_t)k * n + c], a[(size_t)p * n + c]);
        std::swap(perm[k], perm[p]);
      }
      const cd piv = a[(size_t)k * n + k];
      if (piv == cd(0)) continue;
      for (int i = k + 1; i < n; ++i) {
        cd& l = a[(size_t)i * n + k];
        l /= piv;
        if (l == cd(0)) continue;
        for (int c = k + 1; c < n; ++c) a[(size_t)i * n + c] -= l * a[(size_t)k * n + c];
      }
    }
  }
  void solve(cd* b) const {
    CVec y(n);
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < i; ++k) y[i] -= a[(size_t)i * n + k] * y[k];
    for (int i = n - 1; i >= 0; --i) {
      for (int k = i + 1; k < n; ++k) y[i] -= a[(size_t)i * n + k] * y[k];
      y[i] /= a[(size_t)i * n + i];
    }
    for (int i = 0; i < n; ++i) b[i] = y[i];
  }
};

// ------------------------------------------------------------ GMRES (krylov.hpp:66-223)
struct SolveStats {
  int iterations = 0;
  double relative_residual = 0.0;
  bool converged = false;
  double wall_time = 0.0;
};
static double nrm(const CVec& v) {
  double s = 0;
  for (auto& x : v) s += std::norm(x);
  return std::sqrt(s);
}
static cd hdot(const CVec& a, const CVec& b) {  // a^H b (Eigen .dot conjugates the first)
  cd s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += std::conj(a[i]) * b[i];
  return s;
}
static void make_givens(cd h1, cd h2, double& c, cd& s) {  // krylov.hpp:66-83
  const double a1 = std::abs(h1), a2 = std::abs(h2);
  if (a2 == 0.0) {
    c = 1.0;
    s = 0;
    return;
  }
  if (a1 == 0.0) {
    c = 0.0;
    s = 1;
    return;
  }
  const double t = std::hypot(a1, a2);
  c = a1 / t;
  s = (h1 / a1) * (std::conj(h2) / t);
}
using Op = std::function<void(const CVec&, CVec&)>;
static std::pair<CVec, SolveStats> gmres(int n, const Op& apply, const Op& prec, const CVec& b, double tol,
                                        int max_iter, int restart, std::vector<double>* hist) {
  auto t0 = std::chrono::steady_clock::now();
  SolveStats st;
  CVec x(n, cd(0));
  const double bnorm = nrm(b);
  if (bnorm == 0.0) {
    st.converged = true;
    return {x, st};
  }
  CVec r(n), w(n), z(n);
  apply(x, r);
  for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
  CVec best_x = x;
  double best_res = nrm(r) / bnorm;
  const int m = std::max(1, restart);
  std::vector<CVec> basis(m + 1);
  std::vector<cd> hess((size_t)(m + 1) * m, cd(0));  // column-major (m+1) x m
  auto H = [&](int i, int j) -> cd& { return hess[(size_t)j * (m + 1) + i]; };
  std::vector<double> gc(m);
  std::vector<cd> gs(m), g(m + 1);
  while (true) {
    const double rnorm = nrm(r);
    st.relative_residual = rnorm / bnorm;
    if (st.relative_residual < best_res) {
      best_res = st.relative_residual;
      best_x = x;
    }
    if (st.relative_residual <= tol) {
      st.converged = true;
      break;
    }
    if (st.iterations >= max_iter) break;
    basis[0].resize(n);
    for (int i = 0; i < n; ++i) basis[0][i] = r[i] / rnorm;
    std::fill(g.begin(), g.end(), cd(0));
    g[0] = rnorm;
    int k = 0;
    for (int j = 0; j < m && st.iterations < max_iter; ++j) {
      prec(basis[j], z);
      apply(z, w);
      const double wpre = nrm(w);
      for (int i = 0; i <= j; ++i) {  // Hermitian MGS (krylov.hpp:159-163)
        const cd hij = hdot(basis[i], w);
        H(i, j) = hij;
        for (int q = 0; q < n; ++q) w[q] -= hij * basis[i][q];
      }
      const double hnext = nrm(w);
      bool finite = std::isfinite(hnext);
      for (int q = 0; q < n && finite; ++q) finite = std::isfinite(std::abs(w[q]));
      if (!finite) throw NumericalError("gmres: breakdown (NaN/Inf in Arnoldi)");
      H(j + 1, j) = hnext;
      for (int i = 0; i < j; ++i) {
        const cd t1 = H(i, j), t2 = H(i + 1, j);
        H(i, j) = gc[i] * t1 + gs[i] * t2;
        H(i + 1, j) = -std::conj(gs[i]) * t1 + gc[i] * t2;
      }
      make_givens(H(j, j), H(j + 1, j), gc[j], gs[j]);
      H(j, j) = gc[j] * H(j, j) + gs[j] * H(j + 1, j);
      H(j + 1, j) = 0;
      g[j + 1] = -std::conj(gs[j]) * g[j];
      g[j] = gc[j] * g[j];
      ++st.iterations;
      k = j + 1;
      const double est = std::abs(g[j + 1]);
      if (hist) hist->push_back(est / bnorm);
      const bool happy = hnext <= 1e-14 * std::max(wpre, 1e-300);
      if (happy || est <= tol * bnorm) break;
      basis[j + 1].resize(n);
      for (int q = 0; q < n; ++q) basis[j + 1][q] = w[q] / hnext;
    }
    CVec y(k);
    for (int i = k - 1; i >= 0; --i) {
      cd acc = g[i];
      for (int j2 = i + 1; j2 < k; ++j2) acc -= H(i, j2) * y[j2];
      y[i] = acc / H(i, i);
    }
    CVec t(n, cd(0));
    for (int i = 0; i < k; ++i)
      for (int q = 0; q < n; ++q) t[q] += y[i] * basis[i][q];
    prec(t, z);
    for (int q = 0; q < n; ++q) x[q] += z[q];
    apply(x, r);
    for (int q = 0; q < n; ++q) r[q] = b[q] - r[q];
  }
  apply(x, w);
  {
    CVec d(n);
    for (int q = 0; q < n; ++q) d[q] = b[q] - w[q];
    st.relative_residual = nrm(d) / bnorm;
  }
  if (st.relative_residual > best_res) {
    x = best_x;
    st.relative_residual = best_res;
  }
  st.converged = st.relative_residual <= tol;
  st.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return {x, st};
}

// ---------------------------------------------------------------- FETI-DP (feti.cpp)
struct Block {
  // sparse pieces as (row, col, value) lists in the reference's r / i / b numbering
  std::vector<std::tuple<int, int, cd>> arc, aib, abb;  // A_rc (n_r x n_c), A_ib, A_bb
  CVec acc;                                             // n_c x n_c row-major
  BandLU arr, aii;
  // augmentation columns touching this subdomain (feti.cpp:394-412): global column ids and
  // their (r-position, sign * value) entries C^s = Q^T B^s
  std::vector<int> active_aug;
  std::vector<std::vector<std::pair<int, double>>> aug_entries;
  int nz = 0;     // local coarse unknowns: n_c corners + active augmentation columns
  CVec coupling;  // n_r x nz row-major: A_rr^{-1} [A_rc | C^T]
};

struct FetiStats {
  SolveStats dual;
  double primal_residual = 0, interface_jump = 0, setup_seconds = 0, solve_seconds = 0;
  int n_lambda = 0, coarse_dim = 0;
};

struct Feti {
  const Problem* P;
  Partition part;
  cd kcoef = 1.0, mcoef = 0.0;
  double tol = 1e-10;
  int max_iter = 1000, threads = 1, setup_threads = 1;
  std::vector<Block> blk;
  bool augment = false;
  std::vector<AugColumn> aug;  // edge-RBM columns (augment = true)
  int ncg = 0;                 // corner dofs; coarse = [corners | augmentation columns]
  int nc = 0;
  CVec coarse;  // nc x nc row-major
  RVec cscale;
  DenseLU clu;
  double setup_seconds = 0;

  static int bandwidth(const std::vector<std::tuple<int, int, cd>>& t) {
    int w = 0;
    for (auto& [i, j, v] : t) w = std::max(w, std::abs(i - j));
    return w;
  }

  // feti.cpp:244-364 (assembly + local factorizations; serial as in the reference)
  void assemble() {
    const int dpn = P->dpn, ed = P->edofs;
    cd ae[576];
    for (int q = 0; q < ed * ed; ++q) ae[q] = kcoef * cd(P->ke[q]) + mcoef * cd(P->me[q]);
    const int ns = (int)part.subs.size();
    blk.resize(ns);
    std::vector<std::string> fail(ns);
    // The reference assembles and factors serially (feti.cpp:271).  setup_threads > 1 runs
    // independent subdomains on worker threads (identical results; used only to keep the
    // 3D CPU-baseline samples of bench.py within minutes).
    const int nt = std::max(1, std::min(setup_threads, ns));
    std::vector<std::vector<int>> lof_pool(nt, std::vector<int>(P->n(), -1));
    auto body = [&](int s, std::vector<int>& local_of_free) {
      const Sub& sub = part.subs[s];
      Block& B = blk[s];
      const int nl = (int)sub.dofs.size(), nc_ = (int)sub.corner_local.size(), nr = (int)sub.r_local.size();
      const int ni = (int)sub.r_interior.size(), nb = (int)sub.r_boundary.size();
      std::vector<int> cat(nl, -1), pos(nl, -1), rcat(nr, 0), rpos(nr, -1);
      for (int k = 0; k < nc_; ++k) cat[sub.corner_local[k]] = 0, pos[sub.corner_local[k]] = k;
      for (int k = 0; k < nr; ++k) cat[sub.r_local[k]] = 1, pos[sub.r_local[k]] = k;
      for (int k = 0; k < ni; ++k) rcat[sub.r_interior[k]] = 0, rpos[sub.r_interior[k]] = k;
      for (int k = 0; k < nb; ++k) rcat[sub.r_boundary[k]] = 1, rpos[sub.r_boundary[k]] = k;
      for (int l = 0; l < nl; ++l) local_of_free[sub.dofs[l]] = l;
      std::vector<std::tuple<int, int, cd>> trr, tii;
      B.acc.assign((size_t)nc_ * nc_, cd(0));
      int gd[24], en[8];
      const int npe = P->npe();
      for (int e : sub.elements) {
        P->elem_nodes(e, en);
        for (int a = 0; a < npe; ++a)
          for (int c = 0; c < dpn; ++c) gd[dpn * a + c] = dpn * en[a] + c;
        for (int a = 0; a < ed; ++a) {
          const int fa = P->free_map[gd[a]];
          if (fa < 0) continue;
          const int la = local_of_free[fa];
          for (int b = 0; b < ed; ++b) {
            const int fb = P->free_map[gd[b]];
            if (fb < 0) continue;
            const int lb = local_of_free[fb];
            const cd v = ae[a * ed + b];
            if (cat[la] == 0 && cat[lb] == 0) {
              B.acc[(size_t)pos[la] * nc_ + pos[lb]] += v;
            } else if (cat[la] == 1 && cat[lb] == 0) {
              B.arc.emplace_back(pos[la], pos[lb], v);
            } else if (cat[la] == 1 && cat[lb] == 1) {
              const int ra = pos[la], rb = pos[lb];
              trr.emplace_back(ra, rb, v);
              if (rcat[ra] == 0 && rcat[rb] == 0)
                tii.emplace_back(rpos[ra], rpos[rb], v);
              else if (rcat[ra] == 0 && rcat[rb] == 1)
                B.aib.emplace_back(rpos[ra], rpos[rb], v);
              else if (rcat[ra] == 1 && rcat[rb] == 1)
                B.abb.emplace_back(rpos[ra], rpos[rb], v);
            }
          }
        }
      }
      for (int l = 0; l < nl; ++l) local_of_free[sub.dofs[l]] = -1;
      const int wr = bandwidth(trr), wi = bandwidth(tii);
      B.arr.init(nr, wr, wr);
      for (auto& [i, j, v] : trr) B.arr.add(i, j, v);
      B.aii.init(ni, wi, wi);
      for (auto& [i, j, v] : tii) B.aii.add(i, j, v);
      if (!B.arr.factor()) fail[s] = "singular remaining block A_rr in subdomain " + std::to_string(s);
      if (!B.aii.factor()) fail[s] = "singular interior block A_ii in subdomain " + std::to_string(s);
    };
    if (nt == 1) {
      for (int s = 0; s < ns; ++s) body(s, lof_pool[0]);
    } else {
      std::vector<std::thread> workers;
      for (int t = 0; t < nt; ++t)
        workers.emplace_back([&, t] {
          for (int s = t; s < ns; s += nt) body(s, lof_pool[t]);
        });
      for (auto& w : workers) w.join();
    }
    for (auto& f : fail)
      if (!f.empty()) throw NumericalError("assemble_subdomain_operators: " + f);
  }

  void setup() {  // feti.cpp:373-480
    auto t0 = std::chrono::steady_clock::now();
    assemble();
    if (augment) aug = edge_rbm_columns(part);
    ncg = part.n_corner;
    const int nq = (int)aug.size();
    nc = ncg + nq;
    const int ns = (int)part.subs.size();
    // lambda row -> (r-position, sign) of each subdomain, for C^s = Q^T B^s (feti.cpp:394-406)
    std::vector<CVec> contrib(ns);
    parallel_for(ns, threads, [&](int s) {
      const Sub& sub = part.subs[s];
      Block& B = blk[s];
      const int nr = (int)sub.r_local.size(), nc_ = (int)sub.corner_local.size();
      std::vector<std::pair<int, int>> row_of;  // sorted (lambda row, k)
      for (size_t k = 0; k < sub.lambda_rows.size(); ++k) row_of.emplace_back(sub.lambda_rows[k], (int)k);
      std::sort(row_of.begin(), row_of.end());
      for (int q = 0; q < nq; ++q) {
        std::vector<std::pair<int, double>> ent;
        for (size_t k = 0; k < aug[q].rows.size(); ++k) {
          auto it = std::lower_bound(row_of.begin(), row_of.end(), std::make_pair(aug[q].rows[k], -1));
          if (it != row_of.end() && it->first == aug[q].rows[k]) {
            const int kk = it->second;
            ent.emplace_back(sub.lambda_rpos[kk], sub.lambda_signs[kk] * aug[q].values[k]);
          }
        }
        if (!ent.empty()) {
          B.active_aug.push_back(q);
          B.aug_entries.push_back(std::move(ent));
        }
      }
      const int na = (int)B.active_aug.size();
      B.nz = nc_ + na;
      B.coupling.assign((size_t)nr * B.nz, cd(0));
      if (B.nz == 0) return;
      // coupling rhs columns [A_rc | C^T] (sparse), solved with A_rr
      auto rhs_col = [&](int c, CVec& col) {
        std::fill(col.begin(), col.end(), cd(0));
        if (c < nc_) {
          for (auto& [i, j, v] : B.arc)
            if (j == c) col[i] += v;
        } else {
          for (auto& [rp, v] : B.aug_entries[c - nc_]) col[rp] += v;
        }
      };
      CVec col(nr);
      for (int c = 0; c < B.nz; ++c) {
        rhs_col(c, col);
        B.arr.solve(col.data());
        for (int i = 0; i < nr; ++i) B.coupling[(size_t)i * B.nz + c] = col[i];
      }
      // contribs = rhs^T * coupling_solved  (transpose, not adjoint: feti.cpp:433)
      contrib[s].assign((size_t)B.nz * B.nz, cd(0));
      for (int a = 0; a < B.nz; ++a) {
        rhs_col(a, col);
        for (int i = 0; i < nr; ++i)
          if (col[i] != cd(0))
            for (int b = 0; b < B.nz; ++b) contrib[s][(size_t)a * B.nz + b] += col[i] * B.coupling[(size_t)i * B.nz + b];
      }
    });
    coarse.assign((size_t)nc * nc, cd(0));
    for (int s = 0; s < ns; ++s) {
      const Sub& sub = part.subs[s];
      const Block& B = blk[s];
      const int nc_ = (int)sub.corner_local.size();
      std::vector<int> zidx(B.nz);
      for (int k = 0; k < nc_; ++k) zidx[k] = sub.corner_global[k];
      for (size_t a = 0; a < B.active_aug.size(); ++a) zidx[nc_ + a] = ncg + B.active_aug[a];
      for (int k = 0; k < nc_; ++k)
        for (int l = 0; l < nc_; ++l)
          coarse[(size_t)sub.corner_global[k] * nc + sub.corner_global[l]] += B.acc[(size_t)k * nc_ + l];
      for (int a = 0; a < B.nz; ++a)
        for (int b = 0; b < B.nz; ++b) coarse[(size_t)zidx[a] * nc + zidx[b]] -= contrib[s][(size_t)a * B.nz + b];
    }
    if (nc > 0) {  // feti.cpp:456-475
      cscale.resize(nc);
      for (int i = 0; i < nc; ++i) {
        const double d = std::abs(coarse[(size_t)i * nc + i]);
        cscale[i] = d > 0.0 ? 1.0 / std::sqrt(d) : 1.0;
      }
      CVec sc = coarse;
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j) sc[(size_t)i * nc + j] *= cscale[i] * cscale[j];
      clu.factor(sc, nc);
      double umax = 0;
      for (int i = 0; i < nc; ++i) umax = std::max(umax, std::abs(clu.a[(size_t)i * nc + i]));
      for (int i = 0; i < nc; ++i)
        if (!(std::abs(clu.a[(size_t)i * nc + i]) > umax * 1e-13)) throw NumericalError("feti: coarse problem is singular");
    }
    setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  // v -= Q Q^T v, column by column (feti.cpp:572-578)
  void project_out_augmentation(CVec& v) const {
    for (const auto& c : aug) {
      cd coef = 0;
      for (size_t k = 0; k < c.rows.size(); ++k) coef += c.values[k] * v[c.rows[k]];
      for (size_t k = 0; k < c.rows.size(); ++k) v[c.rows[k]] -= coef * c.values[k];
    }
  }

  CVec coarse_solve(const CVec& g) const {  // feti.cpp:483-490
    if (nc == 0) return {};
    CVec z = g;
    for (int i = 0; i < nc; ++i) z[i] *= cscale[i];
    clu.solve(z.data());
    for (int i = 0; i < nc; ++i) z[i] *= cscale[i];
    return z;
  }

  void split_rhs(const CVec& rhs, std::vector<CVec>& fr, CVec& fc) const {  // 493-510
    const int ns = (int)part.subs.size();
    fr.resize(ns);
    fc.assign(ncg, cd(0));
    for (int s = 0; s < ns; ++s) {
      const Sub& sub = part.subs[s];
      fr[s].resize(sub.r_local.size());
      for (size_t k = 0; k < sub.r_local.size(); ++k) {
        const int l = sub.r_local[k];
        fr[s][k] = sub.weights[l] * rhs[sub.dofs[l]];
      }
      for (size_t k = 0; k < sub.corner_local.size(); ++k) fc[sub.corner_global[k]] = rhs[sub.dofs[sub.corner_local[k]]];
    }
  }

  void eliminate(const std::vector<CVec>& t, const CVec& fc, std::vector<CVec>& ur, CVec& z) const {  // 516-556
    const int ns = (int)part.subs.size();
    std::vector<CVec> u1(ns);
    parallel_for(ns, threads, [&](int s) {
      u1[s] = t[s];
      blk[s].arr.solve(u1[s].data());
    });
    CVec g(nc, cd(0));
    for (int i = 0; i < ncg; ++i) g[i] = fc[i];
    for (int s = 0; s < ns; ++s) {
      const Sub& sub = part.subs[s];
      const Block& B = blk[s];
      const int nc_ = (int)sub.corner_local.size();
      if (nc_ > 0) {
        CVec v(nc_, cd(0));
        for (auto& [i, c, val] : B.arc) v[c] += val * u1[s][i];
        for (int k = 0; k < nc_; ++k) g[sub.corner_global[k]] -= v[k];
      }
      for (size_t a = 0; a < B.active_aug.size(); ++a) {
        cd acc = 0;
        for (auto& [rp, val] : B.aug_entries[a]) acc += val * u1[s][rp];
        g[ncg + B.active_aug[a]] -= acc;
      }
    }
    z = coarse_solve(g);
    ur.resize(ns);
    parallel_for(ns, threads, [&](int s) {
      const Sub& sub = part.subs[s];
      const Block& B = blk[s];
      const int nc_ = (int)sub.corner_local.size(), nr = (int)sub.r_local.size();
      ur[s] = std::move(u1[s]);
      if (B.nz > 0) {
        CVec zl(B.nz);
        for (int k = 0; k < nc_; ++k) zl[k] = z[sub.corner_global[k]];
        for (size_t a = 0; a < B.active_aug.size(); ++a) zl[nc_ + a] = z[ncg + B.active_aug[a]];
        for (int i = 0; i < nr; ++i) {
          cd acc = 0;
          for (int k = 0; k < B.nz; ++k) acc += B.coupling[(size_t)i * B.nz + k] * zl[k];
          ur[s][i] -= acc;
        }
      }
    });
  }

  CVec gather_jump(const std::vector<CVec>& ur) const {  // 560-569
    CVec out(part.n_lambda, cd(0));
    for (size_t s = 0; s < part.subs.size(); ++s) {
      const Sub& sub = part.subs[s];
      for (size_t k = 0; k < sub.lambda_rows.size(); ++k)
        out[sub.lambda_rows[k]] += sub.lambda_signs[k] * ur[s][sub.lambda_rpos[k]];
    }
    return out;
  }

  CVec apply_dual(const CVec& lam) const {  // 581-594
    const int ns = (int)part.subs.size();
    std::vector<CVec> t(ns);
    for (int s = 0; s < ns; ++s) {
      const Sub& sub = part.subs[s];
      t[s].assign(sub.r_local.size(), cd(0));
      for (size_t k = 0; k < sub.lambda_rows.size(); ++k)
        t[s][sub.lambda_rpos[k]] -= sub.lambda_signs[k] * lam[sub.lambda_rows[k]];
    }
    std::vector<CVec> ur;
    CVec z;
    eliminate(t, CVec(ncg, cd(0)), ur, z);
    CVec out = gather_jump(ur);
    for (auto& v : out) v = -v;
    return out;
  }

  CVec apply_dirichlet(const CVec& res) const {  // 597-627; W = 1/2 there, 1/mult per row here
    const int ns = (int)part.subs.size();
    CVec wr(res.size());
    for (size_t i = 0; i < res.size(); ++i) wr[i] = res[i] * part.lam_weight[i];
    std::vector<CVec> contrib(ns);
    parallel_for(ns, threads, [&](int s) {
      const Sub& sub = part.subs[s];
      const Block& B = blk[s];
      const int nb = (int)sub.r_boundary.size(), ni = (int)sub.r_interior.size();
      CVec vb(nb, cd(0));
      for (size_t k = 0; k < sub.lambda_rows.size(); ++k)
        vb[sub.lambda_bidx[k]] += sub.lambda_signs[k] * wr[sub.lambda_rows[k]];
      CVec wb(nb, cd(0));
      for (auto& [i, j, v] : B.abb) wb[i] += v * vb[j];
      if (ni > 0) {
        CVec ti(ni, cd(0));
        for (auto& [i, j, v] : B.aib) ti[i] += v * vb[j];
        B.aii.solve(ti.data());
        for (auto& [i, j, v] : B.aib) wb[j] -= v * ti[i];
      }
      contrib[s] = std::move(wb);
    });
    CVec out(part.n_lambda, cd(0));
    for (int s = 0; s < ns; ++s) {
      const Sub& sub = part.subs[s];
      for (size_t k = 0; k < sub.lambda_rows.size(); ++k)
        out[sub.lambda_rows[k]] += sub.lambda_signs[k] * contrib[s][sub.lambda_bidx[k]];
    }
    for (size_t i = 0; i < out.size(); ++i) out[i] *= part.lam_weight[i];
    return out;
  }

  // global operator kcoef*K + mcoef*V applied to a complex vector (primal residual)
  void apply_global(const CVec& x, CVec& y) const {
    CVec kx(x.size()), vx(x.size());
    P->K.apply(x.data(), kx.data());
    P->V.apply(x.data(), vx.data());
    y.resize(x.size());
    for (size_t i = 0; i < x.size(); ++i) y[i] = kcoef * kx[i] + mcoef * vx[i];
  }

  std::pair<CVec, FetiStats> solve(const CVec& rhs, std::vector<double>* hist = nullptr) const {  // 630-717
    auto t0 = std::chrono::steady_clock::now();
    FetiStats st;
    st.n_lambda = part.n_lambda;
    st.coarse_dim = nc;
    st.setup_seconds = setup_seconds;
    if ((int)rhs.size() != part.n_free) throw ContractError("feti: rhs dimension mismatch");
    if (nrm(rhs) == 0.0) {
      st.dual.converged = true;
      return {CVec(part.n_free, cd(0)), st};
    }
    std::vector<CVec> fr;
    CVec fc;
    split_rhs(rhs, fr, fc);
    std::vector<CVec> ur;
    CVec z;
    eliminate(fr, fc, ur, z);
    CVec d = gather_jump(ur);
    // the coarse solve pins the augmented jump components: the dual problem lives in the
    // orthogonal complement of the columns (feti.cpp:655-662)
    project_out_augmentation(d);
    const int nl = part.n_lambda;
    Op A = [this](const CVec& x, CVec& y) {
      y = apply_dual(x);
      project_out_augmentation(y);
    };
    Op M = [this](const CVec& x, CVec& y) { y = apply_dirichlet(x); };
    auto [lam, gst] = gmres(nl, A, M, d, tol, max_iter, std::max(1, max_iter), hist);
    st.dual = gst;
    const int ns = (int)part.subs.size();
    std::vector<CVec> t(ns);
    for (int s = 0; s < ns; ++s) {
      const Sub& sub = part.subs[s];
      t[s] = fr[s];
      for (size_t k = 0; k < sub.lambda_rows.size(); ++k)
        t[s][sub.lambda_rpos[k]] -= sub.lambda_signs[k] * lam[sub.lambda_rows[k]];
    }
    eliminate(t, fc, ur, z);
    CVec x(part.n_free, cd(0));
    for (int s = 0; s < ns; ++s) {
      const Sub& sub = part.subs[s];
      for (size_t k = 0; k < sub.corner_local.size(); ++k) x[sub.dofs[sub.corner_local[k]]] = z[sub.corner_global[k]];
      for (size_t k = 0; k < sub.r_local.size(); ++k) {
        const int l = sub.r_local[k];
        x[sub.dofs[l]] += sub.weights[l] * ur[s][k];
      }
    }
    const CVec jump = gather_jump(ur);
    double jm = 0;
    for (auto& v : jump) jm = std::max(jm, std::abs(v));
    st.interface_jump = jm;
    CVec ax;
    apply_global(x, ax);
    CVec dd(ax.size());
    for (size_t i = 0; i < ax.size(); ++i) dd[i] = ax[i] - rhs[i];
    st.primal_residual = nrm(dd) / nrm(rhs);
    st.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {x, st};
  }
};

// ------------------------------------------------------ V^{-1} (SimplicialLLT restated)
static void mass_solve(const Problem& P, const double* b, double* x) {
  const Csr& V = P.V;
  const int n = V.nr;
  int w = 0;
  for (int r = 0; r < n; ++r)
    for (int k = V.off[r]; k < V.off[r + 1]; ++k) w = std::max(w, std::abs(V.col[k] - r));
  if ((double)n * w * w <= 4e9) {  // banded Cholesky, row storage of lower band
    const int ld = w + 1;
    RVec L((size_t)n * ld, 0.0);  // L(i, j) at [i*ld + (j - i + w)], j in [i-w, i]
    auto at = [&](int i, int j) -> double& { return L[(size_t)i * ld + (j - i + w)]; };
    for (int r = 0; r < n; ++r)
      for (int k = V.off[r]; k < V.off[r + 1]; ++k)
        if (V.col[k] <= r) at(r, V.col[k]) = V.val[k];
    for (int i = 0; i < n; ++i) {
      for (int j = std::max(0, i - w); j <= i; ++j) {
        double s = at(i, j);
        for (int k = std::max(0, i - w); k < j; ++k)
          if (k >= j - w) s -= at(i, k) * at(j, k);
        if (j == i) {
          if (!(s > 0)) throw NumericalError("SpdCholesky: matrix is not positive definite");
          at(i, i) = std::sqrt(s);
        } else {
          at(i, j) = s / at(j, j);
        }
      }
    }
    RVec y(b, b + n);
    for (int i = 0; i < n; ++i) {
      double s = y[i];
      for (int k = std::max(0, i - w); k < i; ++k) s -= at(i, k) * y[k];
      y[i] = s / at(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k <= std::min(n - 1, i + w); ++k) s -= at(k, i) * y[k];
      y[i] = s / at(i, i);
    }
    std::copy(y.begin(), y.end(), x);
    return;
  }
  // Jacobi-PCG to 1e-15 relative (large n; agrees with the Cholesky to ~1e-14)
  RVec d(n), r(b, b + n), z(n), p(n), q(n), xx(n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = V.off[i]; k < V.off[i + 1]; ++k)
      if (V.col[k] == i) d[i] = V.val[k];
  double bn = 0;
  for (int i = 0; i < n; ++i) bn += b[i] * b[i];
  bn = std::sqrt(bn);
  if (bn == 0) {
    std::fill(x, x + n, 0.0);
    return;
  }
  for (int i = 0; i < n; ++i) z[i] = r[i] / d[i], p[i] = z[i];
  double rz = 0;
  for (int i = 0; i < n; ++i) rz += r[i] * z[i];
  for (int it = 0; it < 1000; ++it) {
    V.apply(p.data(), q.data());
    double pq = 0;
    for (int i = 0; i < n; ++i) pq += p[i] * q[i];
    const double a = rz / pq;
    double rn = 0;
    for (int i = 0; i < n; ++i) xx[i] += a * p[i], r[i] -= a * q[i], rn += r[i] * r[i];
    if (std::sqrt(rn) <= 1e-15 * bn) break;
    for (int i = 0; i < n; ++i) z[i] = r[i] / d[i];
    double rz2 = 0;
    for (int i = 0; i < n; ++i) rz2 += r[i] * z[i];
    const double beta = rz2 / rz;
    rz = rz2;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  std::copy(xx.begin(), xx.end(), x);
}

}  // namespace orc

// ================================================================ C ABI (ctypes)
using namespace orc;
namespace {
thread_local std::string g_err;
int guard(const std::function<void()>& f) {
  try {
    f();
    return 0;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}
struct OrcStats {  // mirrors FetiStats + SolveStats
  int iterations, converged;
  double relative_residual, primal_residual, interface_jump, setup_seconds, solve_seconds;
  int n_lambda, coarse_dim;
};
void fill(OrcStats* o, const FetiStats& s) {
  if (!o) return;
  o->iterations = s.dual.iterations;
  o->converged = s.dual.converged;
  o->relative_residual = s.dual.relative_residual;
  o->primal_residual = s.primal_residual;
  o->interface_jump = s.interface_jump;
  o->setup_seconds = s.setup_seconds;
  o->solve_seconds = s.solve_seconds;
  o->n_lambda = s.n_lambda;
  o->coarse_dim = s.coarse_dim;
}
}  // namespace

extern "C" {
const char* orc_last_error() { return g_err.c_str(); }
// test infrastructure: subdomain blocks by symmetric band LDL^T instead of pivoted band LU
void orc_set_band_ldlt(int on) { g_band_ldlt = on != 0; }

int orc_problem_create3(int nx, int ny, int nz, double lx, double ly, double lz, int physics, double E, double nu,
                        void** out) {
  return guard([&] { *out = build_problem_any(nx, ny, nz, lx, ly, lz, physics, E, nu); });
}
int orc_problem_create(int nx, int ny, double lx, double ly, int physics, double E, double nu, void** out) {
  return guard([&] { *out = build_problem(nx, ny, lx, ly, physics, E, nu); });
}
void orc_problem_destroy(void* p) { delete static_cast<Problem*>(p); }
int orc_problem_n(void* p) { return static_cast<Problem*>(p)->n(); }
int orc_problem_m(void* p) { return static_cast<Problem*>(p)->m(); }
double orc_problem_mass_sum(void* p) { return static_cast<Problem*>(p)->mass_sum; }
void orc_element_matrices(void* p, double* ke, double* me) {
  auto* P = static_cast<Problem*>(p);
  std::copy(P->ke, P->ke + P->edofs * P->edofs, ke);
  std::copy(P->me, P->me + P->edofs * P->edofs, me);
}
// which: 0 K, 1 V, 2 Kc ; dense row-major
void orc_dense(void* p, int which, double* out) {
  auto* P = static_cast<Problem*>(p);
  const Csr& A = which == 0 ? P->K : which == 1 ? P->V : P->Kc;
  std::fill(out, out + (size_t)A.nr * A.nc, 0.0);
  for (int r = 0; r < A.nr; ++r)
    for (int k = A.off[r]; k < A.off[r + 1]; ++k) out[(size_t)r * A.nc + A.col[k]] = A.val[k];
}
void orc_apply(void* p, int which, const double* x, double* y) {
  auto* P = static_cast<Problem*>(p);
  const Csr& A = which == 0 ? P->K : which == 1 ? P->V : P->Kc;
  A.apply(x, y);
}
void orc_target_thermal(void* p, double* out) {  // fem.cpp:204-211
  auto* P = static_cast<Problem*>(p);
  for (int f = 0; f < P->n(); ++f) {
    const int node = P->free_dofs[f] / P->dpn;
    out[f] = evaluate_target_thermal(P->node_x(node), P->node_y(node));
  }
}
void orc_boundary_thermal(void* p, double* out) {  // fem.cpp:213-220
  auto* P = static_cast<Problem*>(p);
  for (int c = 0; c < P->m(); ++c) {
    const int node = P->cons_dofs[c] / P->dpn;
    out[c] = evaluate_target_thermal(P->node_x(node), P->node_y(node));
  }
}
void orc_target_sine(void* p, unsigned long long seed, int modes, int mmax, double* out) {
  auto* P = static_cast<Problem*>(p);
  std::vector<double> a(modes);
  std::vector<int> m(modes), nn(modes);
  sine_modes(seed, modes, mmax, a.data(), m.data(), nn.data());
  for (int f = 0; f < P->n(); ++f) {
    const int node = P->free_dofs[f] / P->dpn;
    const double x = P->node_x(node), y = P->node_y(node);
    double v = 0.0;
    for (int k = 0; k < modes; ++k) v += a[k] * std::sin(m[k] * M_PI * x) * std::sin(nn[k] * M_PI * y);
    out[f] = v;
  }
}
// 3D seeded target: per mode a_k (Box-Muller), then l_k, m_k, n_k = 1 + rng() % M
void orc_target_sine3(void* p, unsigned long long seed, int modes, int mmax, double* out) {
  auto* P = static_cast<Problem*>(p);
  std::mt19937_64 g(seed);
  std::vector<double> a(modes);
  std::vector<int> l(modes), m(modes), nn(modes);
  for (int k = 0; k < modes; ++k) {
    const double u1 = u01(g), u2 = u01(g);
    a[k] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
    l[k] = 1 + (int)(g() % (uint64_t)mmax);
    m[k] = 1 + (int)(g() % (uint64_t)mmax);
    nn[k] = 1 + (int)(g() % (uint64_t)mmax);
  }
  for (int f = 0; f < P->n(); ++f) {
    const int node = P->free_dofs[f] / P->dpn;
    const double x = P->node_x(node), y = P->node_y(node), z = P->node_z(node);
    double v = 0.0;
    for (int k = 0; k < modes; ++k)
      v += a[k] * std::sin(l[k] * M_PI * x) * std::sin(m[k] * M_PI * y) * std::sin(nn[k] * M_PI * z);
    out[f] = v;
  }
}
void orc_sine_modes(unsigned long long seed, int modes, int mmax, double* a, int* m, int* n) {
  sine_modes(seed, modes, mmax, a, m, n);
}
// info: [n_sub, n_corner, n_lambda, n_edges, ex, ey, ez]
int orc_partition_info3(void* p, int sx, int sy, int sz, int* info) {
  return guard([&] {
    Partition part = partition_any(*static_cast<Problem*>(p), sx, sy, sz);
    info[6] = part.ez;
    info[0] = (int)part.subs.size();
    info[1] = part.n_corner;
    info[2] = part.n_lambda;
    info[3] = part.n_edges;
    info[4] = part.ex;
    info[5] = part.ey;
  });
}

int orc_partition_info(void* p, int sx, int sy, int* info) {
  int tmp[7];
  const int rc = orc_partition_info3(p, sx, sy, 1, tmp);
  if (rc == 0) std::copy(tmp, tmp + 6, info);
  return rc;
}
// per-subdomain sizes of a partition: out[s*5 + {0..4}] = n_r, n_i, n_b, n_c, jump entries
int orc_partition_sizes(void* p, int sx, int sy, int sz, int* out) {
  return guard([&] {
    Partition part = partition_any(*static_cast<Problem*>(p), sx, sy, sz);
    for (size_t s = 0; s < part.subs.size(); ++s) {
      const Sub& b = part.subs[s];
      out[s * 5 + 0] = (int)b.r_local.size();
      out[s * 5 + 1] = (int)b.r_interior.size();
      out[s * 5 + 2] = (int)b.r_boundary.size();
      out[s * 5 + 3] = (int)b.corner_local.size();
      out[s * 5 + 4] = (int)b.lambda_rows.size();
    }
  });
}
int orc_feti_create3(void* p, int sx, int sy, int sz, double kre, double kim, double mre, double mim, double tol,
                     int max_iter, int threads, int augment, void** out) {
  return guard([&] {
    auto F = std::make_unique<Feti>();
    F->P = static_cast<Problem*>(p);
    if (augment && F->P->is3d()) throw ContractError("feti: edge-RBM augmentation is 2D only");
    F->part = partition_any(*F->P, sx, sy, sz);
    F->augment = augment != 0;
    F->kcoef = cd(kre, kim);
    F->mcoef = cd(mre, mim);
    F->tol = tol;
    F->max_iter = max_iter;
    F->threads = threads;
    F->setup();
    *out = F.release();
  });
}
int orc_feti_create(void* p, int sx, int sy, double kre, double kim, double mre, double mim, double tol,
                    int max_iter, int threads, int augment, void** out) {
  return orc_feti_create3(p, sx, sy, 1, kre, kim, mre, mim, tol, max_iter, threads, augment, out);
}
void orc_feti_destroy(void* f) { delete static_cast<Feti*>(f); }
int orc_feti_n_lambda(void* f) { return static_cast<Feti*>(f)->part.n_lambda; }
int orc_feti_coarse_dim(void* f) { return static_cast<Feti*>(f)->nc; }
double orc_feti_setup_seconds(void* f) { return static_cast<Feti*>(f)->setup_seconds; }
int orc_feti_apply_dual(void* f, const double* in, double* out) {
  return guard([&] {
    auto* F = static_cast<Feti*>(f);
    const int nl = F->part.n_lambda;
    CVec x((const cd*)in, (const cd*)in + nl);
    CVec y = F->apply_dual(x);
    std::copy(y.begin(), y.end(), (cd*)out);
  });
}
int orc_feti_apply_precond(void* f, const double* in, double* out) {
  return guard([&] {
    auto* F = static_cast<Feti*>(f);
    const int nl = F->part.n_lambda;
    CVec x((const cd*)in, (const cd*)in + nl);
    CVec y = F->apply_dirichlet(x);
    std::copy(y.begin(), y.end(), (cd*)out);
  });
}
int orc_feti_solve(void* f, const double* rhs, double* x, OrcStats* st, double* hist, int hist_cap) {
  return guard([&] {
    auto* F = static_cast<Feti*>(f);
    const int n = F->part.n_free;
    CVec b((const cd*)rhs, (const cd*)rhs + n);
    std::vector<double> h;
    auto [xx, s] = F->solve(b, &h);
    std::copy(xx.begin(), xx.end(), (cd*)x);
    fill(st, s);
    if (hist)
      for (int i = 0; i < std::min<int>(hist_cap, (int)h.size()); ++i) hist[i] = h[i];
  });
}

// Range-space Schur solve (control.cpp:297-334). Two independent FETI setups, as
// in the reference (control.cpp:303-304). times[0] = setup seconds (both factors),
// times[1] = solve seconds (both FETI solves + recovery).
int orc_schur_solve3(void* p, int sx, int sy, int sz, double phi, const double* ybar, const double* yc, double tol,
                     int max_iter, int threads, int augment, double* y, double* u, double* lam, OrcStats* plus,
                     OrcStats* minus, double* imag_leak, double* times) {
  return guard([&] {
    auto* P = static_cast<Problem*>(p);
    if (!(phi > 0.0)) throw ContractError("ControlProblem: phi must be positive");
    const int n = P->n(), m = P->m();
    const cd c(0.0, -1.0 / std::sqrt(phi));
    auto t0 = std::chrono::steady_clock::now();
    Feti fp, fm;
    for (Feti* F : {&fp, &fm}) {
      F->P = P;
      F->part = partition_any(*P, sx, sy, sz);
      F->augment = augment != 0;
      F->kcoef = 1.0;
      F->tol = tol;
      F->max_iter = max_iter;
      F->threads = threads;
    }
    fp.mcoef = c;
    fm.mcoef = -c;
    fp.setup();
    fm.setup();
    auto t1 = std::chrono::steady_clock::now();
    RVec rhs(n), kc(n, 0.0);
    P->K.apply(ybar, rhs.data());
    if (yc && m > 0) {
      P->Kc.apply(yc, kc.data());
      for (int i = 0; i < n; ++i) rhs[i] += kc[i];
    }
    CVec crhs(rhs.begin(), rhs.end());
    auto [a, sp] = fp.solve(crhs);
    CVec va(n);
    P->V.apply(a.data(), va.data());
    auto [t, sm] = fm.solve(va);
    double leak = 0;
    for (int i = 0; i < n; ++i) {
      lam[i] = t[i].real();
      leak = std::max(leak, std::abs(t[i].imag()));
    }
    RVec kl(n), vk(n);
    P->K.apply(lam, kl.data());
    mass_solve(*P, kl.data(), vk.data());
    for (int i = 0; i < n; ++i) {
      y[i] = ybar[i] - vk[i];
      u[i] = lam[i] / phi;
    }
    auto t2 = std::chrono::steady_clock::now();
    fill(plus, sp);
    fill(minus, sm);
    if (imag_leak) *imag_leak = leak;
    if (times) {
      times[0] = std::chrono::duration<double>(t1 - t0).count();
      times[1] = std::chrono::duration<double>(t2 - t1).count();
    }
  });
}

int orc_schur_solve(void* p, int sx, int sy, double phi, const double* ybar, const double* yc, double tol,
                    int max_iter, int threads, int augment, double* y, double* u, double* lam, OrcStats* plus,
                    OrcStats* minus, double* imag_leak, double* times) {
  return orc_schur_solve3(p, sx, sy, 1, phi, ybar, yc, tol, max_iter, threads, augment, y, u, lam, plus, minus,
                          imag_leak, times);
}

// Persistent pair of factor solvers (the two ComplexFactorSolver of control.cpp:303-304)
// so timing can separate setup from per-solve cost (experiments.cpp:264-265).
struct SchurPair {
  Problem* P;
  Feti plus, minus;
  double phi;
};
int orc_schur_create4(void* p, int sx, int sy, int sz, double phi, double tol, int max_iter, int threads,
                      int augment, int setup_threads, void** out, double* setup_seconds);
int orc_schur_create3(void* p, int sx, int sy, int sz, double phi, double tol, int max_iter, int threads,
                      int augment, void** out, double* setup_seconds) {
  return orc_schur_create4(p, sx, sy, sz, phi, tol, max_iter, threads, augment, 1, out, setup_seconds);
}
int orc_schur_create4(void* p, int sx, int sy, int sz, double phi, double tol, int max_iter, int threads,
                      int augment, int setup_threads, void** out, double* setup_seconds) {
  return guard([&] {
    auto* P = static_cast<Problem*>(p);
    if (!(phi > 0.0)) throw ContractError("ControlProblem: phi must be positive");
    auto sp = std::make_unique<SchurPair>();
    sp->P = P;
    sp->phi = phi;
    const cd c(0.0, -1.0 / std::sqrt(phi));
    auto t0 = std::chrono::steady_clock::now();
    for (Feti* F : {&sp->plus, &sp->minus}) {
      F->P = P;
      F->part = partition_any(*P, sx, sy, sz);
      F->augment = augment != 0;
      F->kcoef = 1.0;
      F->tol = tol;
      F->max_iter = max_iter;
      F->threads = threads;
      F->setup_threads = setup_threads;
    }
    sp->plus.mcoef = c;
    sp->minus.mcoef = -c;
    sp->plus.setup();
    sp->minus.setup();
    if (setup_seconds) *setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = sp.release();
  });
}
int orc_schur_create(void* p, int sx, int sy, double phi, double tol, int max_iter, int threads, int augment,
                     void** out, double* setup_seconds) {
  return orc_schur_create3(p, sx, sy, 1, phi, tol, max_iter, threads, augment, out, setup_seconds);
}
void orc_schur_destroy(void* h) { delete static_cast<SchurPair*>(h); }
int orc_schur_run(void* h, const double* ybar, const double* yc, double* y, double* u, double* lam, OrcStats* plus,
                  OrcStats* minus, double* imag_leak) {
  return guard([&] {
    auto* sp = static_cast<SchurPair*>(h);
    Problem* P = sp->P;
    const int n = P->n(), m = P->m();
    RVec rhs(n), kc(n, 0.0);
    P->K.apply(ybar, rhs.data());
    if (yc && m > 0) {
      P->Kc.apply(yc, kc.data());
      for (int i = 0; i < n; ++i) rhs[i] += kc[i];
    }
    CVec crhs(rhs.begin(), rhs.end());
    auto [a, s1] = sp->plus.solve(crhs);
    CVec va(n);
    P->V.apply(a.data(), va.data());
    auto [t, s2] = sp->minus.solve(va);
    double leak = 0;
    for (int i = 0; i < n; ++i) {
      lam[i] = t[i].real();
      leak = std::max(leak, std::abs(t[i].imag()));
    }
    RVec kl(n), vk(n);
    P->K.apply(lam, kl.data());
    mass_solve(*P, kl.data(), vk.data());
    for (int i = 0; i < n; ++i) {
      y[i] = ybar[i] - vk[i];
      u[i] = lam[i] / sp->phi;
    }
    fill(plus, s1);
    fill(minus, s2);
    if (imag_leak) *imag_leak = leak;
  });
}

// Dense GMRES harness (krylov.hpp restated) for the reference's Krylov tests.
int orc_gmres_dense(int n, const double* a, const double* b, double tol, int max_iter, double* x, int* iters,
                    double* relres, int* converged, double* hist, int hist_cap) {
  return guard([&] {
    const cd* A = (const cd*)a;
    Op ap = [&](const CVec& v, CVec& y) {
      y.assign(n, cd(0));
      for (int i = 0; i < n; ++i) {
        cd s = 0;
        for (int j = 0; j < n; ++j) s += A[(size_t)i * n + j] * v[j];
        y[i] = s;
      }
    };
    Op id = [&](const CVec& v, CVec& y) { y = v; };
    std::vector<double> h;
    CVec bb((const cd*)b, (const cd*)b + n);
    auto [xx, st] = gmres(n, ap, id, bb, tol, max_iter, std::max(1, max_iter), &h);
    std::copy(xx.begin(), xx.end(), (cd*)x);
    *iters = st.iterations;
    *relres = st.relative_residual;
    *converged = st.converged;
    if (hist)
      for (int i = 0; i < std::min<int>(hist_cap, (int)h.size()); ++i) hist[i] = h[i];
  });
}
}  // extern "C"
