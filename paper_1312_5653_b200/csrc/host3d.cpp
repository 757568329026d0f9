// host3d.cpp — see host3d.hpp.
#include "host3d.hpp"

#include <algorithm>
#include <cmath>
#include <random>

namespace fetigpu {

namespace {

// local node a of a hexahedron: the 2D counterclockwise order (mesh.cpp:31-34) of the
// bottom face, then the top face
const int kHx[8] = {0, 1, 1, 0, 0, 1, 1, 0};
const int kHy[8] = {0, 0, 1, 1, 0, 0, 1, 1};
const int kHz[8] = {0, 0, 0, 0, 1, 1, 1, 1};

// Heat: the Q1 hexahedron matrices are tensor products of the 1-D P1 ones (exact, the
// 2x2x2 Gauss rule of the 2D fem.cpp:62-81 extended integrates them exactly):
//   M = m (x) m (x) m,  K = k (x) m (x) m + m (x) k (x) m + m (x) m (x) k,
//   m = h/6 [[2,1],[1,2]],  k = 1/h [[1,-1],[-1,1]].
void heat_hex(double h, double ke[64], double me[64]) {
  const double m1[2][2] = {{h / 3.0, h / 6.0}, {h / 6.0, h / 3.0}};
  const double k1[2][2] = {{1.0 / h, -1.0 / h}, {-1.0 / h, 1.0 / h}};
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      const double mx = m1[kHx[a]][kHx[b]], my = m1[kHy[a]][kHy[b]], mz = m1[kHz[a]][kHz[b]];
      const double kx = k1[kHx[a]][kHx[b]], ky = k1[kHy[a]][kHy[b]], kz = k1[kHz[a]][kHz[b]];
      me[a * 8 + b] = mx * my * mz;
      ke[a * 8 + b] = kx * my * mz + mx * ky * mz + mx * my * kz;
    }
}

// Linear elasticity on the hexahedron (the 3D form of fem.cpp:92-117): 2x2x2 Gauss,
// Voigt strains (xx, yy, zz, xy, yz, zx), isotropic D; mass = heat mass (x) I_3.
void elastic_hex(double E, double nu, double h, double ke[576], double me[576]) {
  const double f = E / ((1.0 + nu) * (1.0 - 2.0 * nu));
  double D[6][6] = {};
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) D[p][q] = f * (p == q ? 1.0 - nu : nu);
  for (int p = 3; p < 6; ++p) D[p][p] = f * (1.0 - 2.0 * nu) / 2.0;
  const double g = 1.0 / std::sqrt(3.0);
  const double detj = h * h * h / 8.0, gs = 2.0 / h;
  std::fill(ke, ke + 576, 0.0);
  for (int q = 0; q < 8; ++q) {
    const double x = (q & 1) ? g : -g, y = (q & 2) ? g : -g, z = (q & 4) ? g : -g;
    double B[6][24] = {};
    for (int a = 0; a < 8; ++a) {
      const double sx = 2.0 * kHx[a] - 1.0, sy = 2.0 * kHy[a] - 1.0, sz = 2.0 * kHz[a] - 1.0;
      const double fx = 1.0 + sx * x, fy = 1.0 + sy * y, fz = 1.0 + sz * z;
      const double dx = gs * 0.125 * sx * fy * fz, dy = gs * 0.125 * sy * fx * fz, dz = gs * 0.125 * sz * fx * fy;
      B[0][3 * a] = dx;
      B[1][3 * a + 1] = dy;
      B[2][3 * a + 2] = dz;
      B[3][3 * a] = dy;
      B[3][3 * a + 1] = dx;
      B[4][3 * a + 1] = dz;
      B[4][3 * a + 2] = dy;
      B[5][3 * a] = dz;
      B[5][3 * a + 2] = dx;
    }
    for (int i = 0; i < 24; ++i)
      for (int j = i; j < 24; ++j) {
        double s = 0.0;
        for (int p = 0; p < 6; ++p)
          for (int r = 0; r < 6; ++r) s += B[p][i] * D[p][r] * B[r][j];
        ke[i * 24 + j] += detj * s;
      }
  }
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < i; ++j) ke[i * 24 + j] = ke[j * 24 + i];
  double kh[64], mh[64];
  heat_hex(h, kh, mh);
  std::fill(me, me + 576, 0.0);
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b)
      for (int c = 0; c < 3; ++c) me[(3 * a + c) * 24 + 3 * b + c] = mh[a * 8 + b];
}

std::pair<int, int> owner_range(int i, int e, int ns) {  // feti.cpp:13-17
  return {i == 0 ? 0 : (i - 1) / e, std::min(ns - 1, i / e)};
}

}  // namespace

Host3Problem build_problem3d(const fetigpu3d_desc& d) {
  if (d.n_x < 2 || d.n_y < 2 || d.n_z < 2) throw ContractError("build_box_mesh: need at least 2 elements per axis");
  if (d.len_x <= 0 || d.len_y <= 0 || d.len_z <= 0) throw ContractError("build_box_mesh: non-positive extent");
  const double hx = d.len_x / d.n_x, hy = d.len_y / d.n_y, hz = d.len_z / d.n_z;
  if (std::abs(hx - hy) > 1e-12 * std::max(hx, hy) || std::abs(hx - hz) > 1e-12 * std::max(hx, hz))
    throw ContractError("build_box_mesh: elements must be cubes");
  if (d.physics != 0 && d.physics != 1) throw ContractError("physics must be 0 (heat) or 1 (elasticity)");
  if ((long long)(d.n_x + 1) * (d.n_y + 1) * (d.n_z + 1) * 3 > (1LL << 31) - 1)
    throw ContractError("build_box_mesh: mesh too large");
  Host3Problem P;
  P.nx = d.n_x, P.ny = d.n_y, P.nz = d.n_z;
  P.lx = d.len_x, P.ly = d.len_y, P.lz = d.len_z;
  P.h = hx;
  P.physics = d.physics;
  P.dpn = d.physics == 0 ? 1 : 3;
  P.edofs = 8 * P.dpn;
  if (d.physics == 0) {
    heat_hex(P.h, P.ke, P.me);
  } else {
    if (!(d.poisson > 0.0 && d.poisson < 0.5))
      throw ContractError("Physics: poisson_ratio must lie strictly in (0, 0.5)");
    if (d.young <= 0.0) throw ContractError("Physics: young_modulus must be positive");
    P.young = d.young;
    P.poisson = d.poisson;
    elastic_hex(d.young, d.poisson, P.h, P.ke, P.me);
  }
  const int dpn = P.dpn;
  const long long nn = (long long)(P.nx + 1) * (P.ny + 1) * (P.nz + 1), nmd = nn * dpn;
  P.free_map.assign(nmd, -1);
  P.cons_map.assign(nmd, -1);
  for (int k = 0; k <= P.nz; ++k)
    for (int j = 0; j <= P.ny; ++j)
      for (int i = 0; i <= P.nx; ++i) {
        const int node = P.node_id(i, j, k);
        const bool cons = P.physics == 0
                              ? (i == 0 || i == P.nx || j == 0 || j == P.ny || k == 0 || k == P.nz)
                              : (i == 0);
        for (int c = 0; c < dpn; ++c) {
          const int md = node * dpn + c;
          if (cons) {
            P.cons_map[md] = (int)P.cons_dofs.size();
            P.cons_dofs.push_back(md);
          } else {
            P.free_map[md] = (int)P.free_dofs.size();
            P.free_dofs.push_back(md);
          }
        }
      }
  return P;
}

Host3Partition build_partition3d(const Host3Problem& P, int sx, int sy, int sz) {
  if (sx < 1 || sy < 1 || sz < 1 || sx * sy * sz < 2) throw ContractError("partition_structured: need at least two subdomains");
  if (P.nx % sx != 0 || P.ny % sy != 0 || P.nz % sz != 0)
    throw ContractError("partition_structured: subdomain grid must divide the element grid");
  const int ex = P.nx / sx, ey = P.ny / sy, ez = P.nz / sz;
  if (ex < 2 || ey < 2 || ez < 2) throw ContractError("partition_structured: H/h must be at least 2");
  const int dpn = P.dpn;
  Host3Partition H;
  H.sx = sx, H.sy = sy, H.sz = sz, H.ex = ex, H.ey = ey, H.ez = ez, H.dpn = dpn;
  H.S = sx * sy * sz;
  H.n_free = P.n();
  const int lx = ex + 1, ly = ey + 1, lz = ez + 1;
  H.nld = lx * ly * lz * dpn;
  const int nnx = P.nx + 1, nny = P.ny + 1, nnz = P.nz + 1;
  const long long nn = (long long)nnx * nny * nnz;
  // multiplicity and corner flag per mesh node
  std::vector<unsigned char> mult(nn), corner(nn);
  for (int k = 0; k < nnz; ++k) {
    auto [rlo, rhi] = owner_range(k, ez, sz);
    for (int j = 0; j < nny; ++j) {
      auto [qlo, qhi] = owner_range(j, ey, sy);
      for (int i = 0; i < nnx; ++i) {
        auto [plo, phi] = owner_range(i, ex, sx);
        const int node = P.node_id(i, j, k);
        const int m = (phi - plo + 1) * (qhi - qlo + 1) * (rhi - rlo + 1);
        mult[node] = (unsigned char)m;
        corner[node] = (i % ex == 0 && j % ey == 0 && k % ez == 0 && m >= 2 && P.free_map[node * dpn] >= 0) ? 1 : 0;
      }
    }
  }
  // global corner ids and first multiplier row of every (node, comp) (feti.cpp:69-81, pairwise)
  std::vector<int> corner_of(nn * dpn, -1), lambda0(nn * dpn, -1);
  for (long long node = 0; node < nn; ++node) {
    if (P.free_map[node * dpn] < 0) continue;
    if (corner[node]) {
      for (int c = 0; c < dpn; ++c) {
        corner_of[node * dpn + c] = H.n_corner++;
        H.corner_dof.push_back(P.free_map[node * dpn + c]);
      }
    } else if (mult[node] >= 2) {
      const int m = mult[node], pairs = m * (m - 1) / 2;
      H.MR = std::max(H.MR, m - 1);
      for (int c = 0; c < dpn; ++c) {
        lambda0[node * dpn + c] = H.n_lambda;
        H.n_lambda += pairs;
        for (int q = 0; q < pairs; ++q) H.lam_w.push_back(1.0 / m);
      }
    }
  }
  // pass 1: per-subdomain counts
  const int S = H.S;
  H.n_i.assign(S, 0);
  H.n_b.assign(S, 0);
  H.n_c.assign(S, 0);
  H.sub_i0.resize(S);
  H.sub_j0.resize(S);
  H.sub_k0.resize(S);
  for (int r = 0; r < sz; ++r)
    for (int q = 0; q < sy; ++q)
      for (int p = 0; p < sx; ++p) {
        const int s = (r * sy + q) * sx + p;
        H.sub_i0[s] = p * ex, H.sub_j0[s] = q * ey, H.sub_k0[s] = r * ez;
        for (int k = r * ez; k <= (r + 1) * ez; ++k)
          for (int j = q * ey; j <= (q + 1) * ey; ++j)
            for (int i = p * ex; i <= (p + 1) * ex; ++i) {
              const int node = P.node_id(i, j, k);
              if (P.free_map[node * dpn] < 0) continue;
              int& cnt = corner[node] ? H.n_c[s] : (mult[node] >= 2 ? H.n_b[s] : H.n_i[s]);
              cnt += dpn;
            }
      }
  for (int s = 0; s < S; ++s) {
    H.NI = std::max(H.NI, H.n_i[s]);
    H.NB = std::max(H.NB, H.n_b[s]);
    H.NC = std::max(H.NC, H.n_c[s]);
  }
  H.NI = std::max(32, (H.NI + 31) / 32 * 32);
  H.NB = std::max(H.NB, 1);
  H.NC = std::max(H.NC, 1);
  const int NI = H.NI, NB = H.NB, NC = H.NC, MR = H.MR;
  H.ldof.assign((size_t)S * H.nld, ldof_code(CAT_DIRICHLET, 0));
  H.idof.assign((size_t)S * NI, -1);
  H.bdof.assign((size_t)S * NB, -1);
  H.cglob.assign((size_t)S * NC, -1);
  H.brow.assign((size_t)S * NB * MR, -1);
  H.bsgn.assign((size_t)S * NB * MR, 0.0);
  H.bw.assign((size_t)S * NB, 0.0);
  H.lam_lo.assign(H.n_lambda, -1);
  H.lam_hi.assign(H.n_lambda, -1);
  H.corner_slots.assign((size_t)H.n_corner * 8, -1);
  H.xkind.assign(H.n_free, -1);
  H.xref.assign((size_t)H.n_free * 4, -1);
  H.xw.assign(H.n_free, 1.0);
  std::vector<int> corner_fill(H.n_corner, 0);
  // pass 2: tables
  std::vector<int> own;
  for (int s = 0; s < S; ++s) {
    int ni = 0, nb = 0, ncn = 0;
    const int i0 = H.sub_i0[s], j0 = H.sub_j0[s], k0 = H.sub_k0[s];
    for (int lk = 0; lk < lz; ++lk)
      for (int lj = 0; lj < ly; ++lj)
        for (int li = 0; li < lx; ++li) {
          const int i = i0 + li, j = j0 + lj, k = k0 + lk;
          const int node = P.node_id(i, j, k);
          const bool iface = !corner[node] && mult[node] >= 2;
          if (iface) {  // owners of the node, ascending subdomain id
            own.clear();
            auto [plo, phi] = owner_range(i, ex, sx);
            auto [qlo, qhi] = owner_range(j, ey, sy);
            auto [rlo, rhi] = owner_range(k, ez, sz);
            for (int r = rlo; r <= rhi; ++r)
              for (int q = qlo; q <= qhi; ++q)
                for (int p = plo; p <= phi; ++p) own.push_back((r * sy + q) * sx + p);
          }
          for (int c = 0; c < dpn; ++c) {
            const int md = node * dpn + c, f = P.free_map[md];
            const int l = ((lk * ly + lj) * lx + li) * dpn + c;
            if (f < 0) continue;
            if (corner[node]) {
              const int cid = corner_of[md];
              H.ldof[(size_t)s * H.nld + l] = ldof_code(CAT_CORNER, ncn);
              H.cglob[(size_t)s * NC + ncn] = cid;
              H.corner_slots[(size_t)cid * 8 + corner_fill[cid]++] = s * NC + ncn;
              H.xkind[f] = 2;
              H.xref[(size_t)f * 4] = cid;
              ++ncn;
            } else if (!iface) {
              H.ldof[(size_t)s * H.nld + l] = ldof_code(CAT_INTERIOR, ni);
              H.idof[(size_t)s * NI + ni] = f;
              H.xkind[f] = 0;
              H.xref[(size_t)f * 4] = s * NI + ni;
              ++ni;
            } else {
              const int kb = nb++;
              H.ldof[(size_t)s * H.nld + l] = ldof_code(CAT_BOUNDARY, kb);
              const size_t slot = (size_t)s * NB + kb;
              H.bdof[slot] = f;
              H.bw[slot] = 1.0 / mult[node];
              int row = lambda0[md], e = 0;
              for (size_t a = 0; a < own.size(); ++a)
                for (size_t b = a + 1; b < own.size(); ++b, ++row) {
                  if (own[a] != s && own[b] != s) continue;
                  H.brow[slot * MR + e] = row;
                  H.bsgn[slot * MR + e] = own[a] == s ? 1.0 : -1.0;
                  (own[a] == s ? H.lam_lo : H.lam_hi)[row] = (int)slot;
                  ++e;
                }
              H.xkind[f] = 1;
              H.xw[f] = 1.0 / mult[node];
              int* xr = &H.xref[(size_t)f * 4];
              int q = 0;
              while (xr[q] >= 0) ++q;
              xr[q] = (int)slot;
            }
          }
        }
  }
  // block half-bandwidth of A_ii and ELL widths of A_bi / A_ib: two dofs couple iff their
  // nodes lie within one element (|di|, |dj|, |dk| <= 1 inside the subdomain)
  for (int s = 0; s < S; ++s) {
    const int* ld = &H.ldof[(size_t)s * H.nld];
    for (int lk = 0; lk < lz; ++lk)
      for (int lj = 0; lj < ly; ++lj)
        for (int li = 0; li < lx; ++li)
          for (int c = 0; c < dpn; ++c) {
            const int code = ld[((lk * ly + lj) * lx + li) * dpn + c], cat = ldof_cat(code);
            if (cat != CAT_INTERIOR && cat != CAT_BOUNDARY) continue;
            int cnt = 0;
            for (int dk = -1; dk <= 1; ++dk)
              for (int dj = -1; dj <= 1; ++dj)
                for (int di = -1; di <= 1; ++di) {
                  const int ai = li + di, aj = lj + dj, ak = lk + dk;
                  if (ai < 0 || aj < 0 || ak < 0 || ai >= lx || aj >= ly || ak >= lz) continue;
                  for (int c2 = 0; c2 < dpn; ++c2) {
                    const int code2 = ld[((ak * ly + aj) * lx + ai) * dpn + c2], cat2 = ldof_cat(code2);
                    if (cat == CAT_INTERIOR && cat2 == CAT_INTERIOR) {
                      const int bi = ldof_idx(code) / 32, bj = ldof_idx(code2) / 32;
                      H.P = std::max(H.P, bi - bj);
                    } else if (cat == CAT_INTERIOR && cat2 == CAT_BOUNDARY) {
                      ++cnt;
                    } else if (cat == CAT_BOUNDARY && cat2 == CAT_INTERIOR) {
                      ++cnt;
                    }
                  }
                }
            if (cat == CAT_INTERIOR) H.MAXE_IB = std::max(H.MAXE_IB, cnt);
            else H.MAXE_BI = std::max(H.MAXE_BI, cnt);
          }
  }
  H.MAXE_BI = std::max(H.MAXE_BI, 1);
  H.MAXE_IB = std::max(H.MAXE_IB, 1);
  for (int r = 0; r < H.n_lambda; ++r)
    if (H.lam_lo[r] < 0 || H.lam_hi[r] < 0) throw NumericalError("partition3d: multiplier row without two owners");
  return H;
}

Host3Partition local_partition3d(const Host3Partition& G, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw ContractError("partition3d: bad rank/world");
  // rank r owns the subdomain-index range [r S/R, (r+1) S/R) of the z-outer, y, x ordering:
  // whole z-layers when R divides s_z, otherwise y-row blocks of a layer (config 5's 4x4x4
  // grid on 8 ranks: 8 subdomains = 2 y-rows of one z-layer per rank).  Dual vectors are
  // replicated and every jump is completed by one allreduce, so any split of the
  // subdomains is exact; contiguous ranges keep each rank's interface small.
  const int S = G.sx * G.sy * G.sz;
  if (S % world != 0) throw ContractError("partition3d: the subdomains (s_x s_y s_z) must divide evenly over the ranks");
  const int per = S / world, s0 = rank * per, s1 = s0 + per;
  Host3Partition L = G;
  L.S = per, L.s_first = s0, L.rank = rank, L.world = world;
  auto slice = [&](auto& v, const auto& src, size_t width) {
    v.assign(src.begin() + (size_t)s0 * width, src.begin() + (size_t)s1 * width);
  };
  slice(L.n_i, G.n_i, 1);
  slice(L.n_b, G.n_b, 1);
  slice(L.n_c, G.n_c, 1);
  slice(L.ldof, G.ldof, G.nld);
  slice(L.idof, G.idof, G.NI);
  slice(L.bdof, G.bdof, G.NB);
  slice(L.cglob, G.cglob, G.NC);
  slice(L.brow, G.brow, (size_t)G.NB * G.MR);
  slice(L.bsgn, G.bsgn, (size_t)G.NB * G.MR);
  slice(L.bw, G.bw, G.NB);
  slice(L.sub_i0, G.sub_i0, 1);
  slice(L.sub_j0, G.sub_j0, 1);
  slice(L.sub_k0, G.sub_k0, 1);
  const long long b0 = (long long)s0 * G.NB, b1 = (long long)s1 * G.NB;
  auto bslot = [&](int slot) { return (slot >= b0 && slot < b1) ? (int)(slot - b0) : -1; };
  for (int r = 0; r < G.n_lambda; ++r) L.lam_lo[r] = bslot(G.lam_lo[r]), L.lam_hi[r] = bslot(G.lam_hi[r]);
  const long long c0 = (long long)s0 * G.NC, c1 = (long long)s1 * G.NC;
  for (size_t q = 0; q < G.corner_slots.size(); ++q) {
    const int sl = G.corner_slots[q];
    L.corner_slots[q] = (sl >= c0 && sl < c1) ? (int)(sl - c0) : -1;
  }
  const long long i0 = (long long)s0 * G.NI, i1 = (long long)s1 * G.NI;
  for (int f = 0; f < G.n_free; ++f) {
    int* xr = &L.xref[(size_t)f * 4];
    const int* gr = &G.xref[(size_t)f * 4];
    if (G.xkind[f] == 0) {
      const bool mine = gr[0] >= i0 && gr[0] < i1;
      L.xkind[f] = mine ? 0 : -1;
      xr[0] = mine ? (int)(gr[0] - i0) : -1;
    } else if (G.xkind[f] == 1) {
      int q2 = 0;
      for (int q = 0; q < 4; ++q) xr[q] = -1;
      for (int q = 0; q < 4 && gr[q] >= 0; ++q)
        if (bslot(gr[q]) >= 0) xr[q2++] = bslot(gr[q]);
      L.xkind[f] = q2 > 0 ? 1 : -1;
    } else {
      L.xkind[f] = rank == 0 ? 2 : -1;  // corner values are replicated: one rank contributes
    }
  }
  return L;
}

void target_sine3d(const Host3Problem& P, uint64_t seed, int modes, int mmax, double* ybar) {
  if (modes < 0 || mmax < 1) throw ContractError("target_sine: need modes >= 0 and mmax >= 1");
  std::mt19937_64 rng(seed);
  std::vector<double> amp(modes);
  std::vector<int> kx(modes), ky(modes), kz(modes);
  const double two53 = 9007199254740992.0;
  for (int k = 0; k < modes; ++k) {
    const double u1 = (double)(rng() >> 11) / two53;
    const double u2 = (double)(rng() >> 11) / two53;
    amp[k] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
    kx[k] = 1 + (int)(rng() % (uint64_t)mmax);
    ky[k] = 1 + (int)(rng() % (uint64_t)mmax);
    kz[k] = 1 + (int)(rng() % (uint64_t)mmax);
  }
  const int nnx = P.nx + 1, nny = P.ny + 1;
  for (int f = 0; f < P.n(); ++f) {
    const int node = P.free_dofs[f] / P.dpn;
    const double x = (node % nnx) * P.h, y = ((node / nnx) % nny) * P.h, z = (node / (nnx * nny)) * P.h;
    double v = 0.0;
    for (int k = 0; k < modes; ++k)
      v += amp[k] * std::sin(kx[k] * M_PI * x) * std::sin(ky[k] * M_PI * y) * std::sin(kz[k] * M_PI * z);
    ybar[f] = v;
  }
}

}  // namespace fetigpu
