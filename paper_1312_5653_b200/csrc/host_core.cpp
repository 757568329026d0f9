// host_core.cpp — see host_core.hpp.
#include "host_core.hpp"

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <random>

namespace fetigpu {

namespace {

// Q1 reference element on [-1,1]^2, counterclockwise nodes (fem.cpp:15-34).
const double kXi[4] = {-1.0, 1.0, 1.0, -1.0};
const double kEta[4] = {-1.0, -1.0, 1.0, 1.0};
double shp(int a, double xi, double eta) { return 0.25 * (1.0 + kXi[a] * xi) * (1.0 + kEta[a] * eta); }
double dxi(int a, double eta) { return 0.25 * kXi[a] * (1.0 + kEta[a] * eta); }
double deta(int a, double xi) { return 0.25 * kEta[a] * (1.0 + kXi[a] * xi); }

void gauss_points(double xi[4], double eta[4]) {
  const double g = 1.0 / std::sqrt(3.0);
  const double px[4] = {-g, g, g, -g}, py[4] = {-g, -g, g, g};
  for (int q = 0; q < 4; ++q) xi[q] = px[q], eta[q] = py[q];
}

// 2x2 Gauss Q1 mass (fem.cpp:62-70) and stiffness (fem.cpp:72-81).
void heat_elements(double h, double ke[16], double me[16]) {
  double gx[4], gy[4];
  gauss_points(gx, gy);
  const double detj = h * h / 4.0;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      double m = 0.0, k = 0.0;
      for (int q = 0; q < 4; ++q) {
        m += shp(a, gx[q], gy[q]) * shp(b, gx[q], gy[q]) * detj;
        k += dxi(a, gy[q]) * dxi(b, gy[q]) + deta(a, gx[q]) * deta(b, gx[q]);
      }
      me[a * 4 + b] = m;
      ke[a * 4 + b] = k;
    }
}

// Plane strain (fem.cpp:83-117): interleaved (x, y) dofs per node.
void plane_strain_elements(double E, double nu, double h, double ke[64], double me[64]) {
  double ks[16], ms[16];
  heat_elements(h, ks, ms);
  std::fill(me, me + 64, 0.0);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      for (int c = 0; c < 2; ++c) me[(2 * a + c) * 8 + 2 * b + c] = ms[a * 4 + b];
  const double f = E / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double D[3][3] = {{f * (1 - nu), f * nu, 0}, {f * nu, f * (1 - nu), 0}, {0, 0, f * (1 - 2 * nu) / 2}};
  double gx[4], gy[4];
  gauss_points(gx, gy);
  std::fill(ke, ke + 64, 0.0);
  const double detj = h * h / 4.0, gs = 2.0 / h;
  for (int q = 0; q < 4; ++q) {
    double B[3][8] = {};
    for (int a = 0; a < 4; ++a) {
      const double dx = gs * dxi(a, gy[q]), dy = gs * deta(a, gx[q]);
      B[0][2 * a] = dx;
      B[1][2 * a + 1] = dy;
      B[2][2 * a] = dy;
      B[2][2 * a + 1] = dx;
    }
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double s = 0.0;
        for (int p = 0; p < 3; ++p)
          for (int r = 0; r < 3; ++r) s += B[p][i] * D[p][r] * B[r][j];
        ke[i * 8 + j] += detj * s;
      }
  }
}

std::pair<int, int> owner_range(int i, int e, int ns) {  // feti.cpp:13-17
  return {i == 0 ? 0 : (i - 1) / e, std::min(ns - 1, i / e)};
}

}  // namespace

HostProblem build_problem(const fetigpu_desc& d) {
  if (d.n_x < 2 || d.n_y < 2) throw ContractError("build_rectangle_mesh: need at least 2 elements per axis");
  if (d.len_x <= 0 || d.len_y <= 0) throw ContractError("build_rectangle_mesh: non-positive extent");
  const double hx = d.len_x / d.n_x, hy = d.len_y / d.n_y;
  if (std::abs(hx - hy) > 1e-12 * std::max(hx, hy))
    throw ContractError("build_rectangle_mesh: elements must be square (len_x/n_x == len_y/n_y)");
  if (d.physics != 0 && d.physics != 1) throw ContractError("physics must be 0 (heat) or 1 (plane strain)");
  HostProblem P;
  P.nx = d.n_x;
  P.ny = d.n_y;
  P.lx = d.len_x;
  P.ly = d.len_y;
  P.h = hx;
  P.physics = d.physics;
  P.dpn = d.physics == 0 ? 1 : 2;
  P.edofs = 4 * P.dpn;
  if (d.physics == 0) {
    double ks[16], ms[16];
    heat_elements(P.h, ks, ms);
    std::copy(ks, ks + 16, P.ke);
    std::copy(ms, ms + 16, P.me);
  } else {
    if (!(d.poisson > 0.0 && d.poisson < 0.5))
      throw ContractError("Physics: poisson_ratio must lie strictly in (0, 0.5)");
    if (d.young <= 0.0) throw ContractError("Physics: young_modulus must be positive");
    P.young = d.young;
    P.poisson = d.poisson;
    plane_strain_elements(d.young, d.poisson, P.h, P.ke, P.me);
  }
  const int nn = (P.nx + 1) * (P.ny + 1), nmd = nn * P.dpn;
  std::vector<char> cons(nmd, 0);
  for (int j = 0; j <= P.ny; ++j)
    for (int i = 0; i <= P.nx; ++i) {
      const int node = P.node_id(i, j);
      if (P.physics == 0) {
        if (i == 0 || i == P.nx || j == 0 || j == P.ny) cons[node] = 1;
      } else if (i == 0) {
        cons[2 * node] = cons[2 * node + 1] = 1;
      }
    }
  P.free_map.assign(nmd, -1);
  P.cons_map.assign(nmd, -1);
  for (int md = 0; md < nmd; ++md) {
    if (cons[md]) {
      P.cons_map[md] = (int)P.cons_dofs.size();
      P.cons_dofs.push_back(md);
    } else {
      P.free_map[md] = (int)P.free_dofs.size();
      P.free_dofs.push_back(md);
    }
  }
  return P;
}

HostPartition build_partition(const HostProblem& P, int sx, int sy, bool augment) {
  // contract checks of feti.cpp:36-41
  if (sx < 1 || sy < 1 || sx * sy < 2) throw ContractError("partition_structured: need at least two subdomains");
  if (P.nx % sx != 0 || P.ny % sy != 0)
    throw ContractError("partition_structured: subdomain grid must divide the element grid");
  const int ex = P.nx / sx, ey = P.ny / sy;
  if (ex < 2 || ey < 2) throw ContractError("partition_structured: H/h must be at least 2");
  const int dpn = P.dpn;
  HostPartition H;
  H.sx = sx;
  H.sy = sy;
  H.ex = ex;
  H.ey = ey;
  H.dpn = dpn;
  H.n_sub = sx * sy;
  H.n_free = P.n();
  H.nld = (ex + 1) * (ey + 1) * dpn;

  // multiplicity and corner flags per mesh node (feti.cpp:55-67)
  const int nn = (P.nx + 1) * (P.ny + 1);
  std::vector<int> mult(nn);
  std::vector<char> corner(nn);
  for (int j = 0; j <= P.ny; ++j) {
    const auto q = owner_range(j, ey, sy);
    for (int i = 0; i <= P.nx; ++i) {
      const auto p = owner_range(i, ex, sx);
      const int node = P.node_id(i, j);
      mult[node] = (p.second - p.first + 1) * (q.second - q.first + 1);
      corner[node] = (i % ex == 0) && (j % ey == 0) && mult[node] >= 2 && P.free_map[node * dpn] >= 0;
    }
  }
  // global corner and multiplier numbering ascending by (node, comp) (feti.cpp:69-81)
  std::vector<int> corner_of(nn * dpn, -1), lambda_of(nn * dpn, -1);
  for (int node = 0; node < nn; ++node) {
    if (P.free_map[node * dpn] < 0) continue;
    if (corner[node]) {
      for (int c = 0; c < dpn; ++c) corner_of[node * dpn + c] = H.n_corner++;
    } else if (mult[node] >= 2) {
      if (mult[node] != 2) throw NumericalError("partition_structured: unexpected interface multiplicity");
      for (int c = 0; c < dpn; ++c) lambda_of[node * dpn + c] = H.n_lambda++;
    }
  }

  // per-subdomain lists in the reference's local order (feti.cpp:90-130)
  struct Loc {
    std::vector<int> icode;  // local mesh dof -> code
    std::vector<int> idof, bdof, blam, cglob, cdof;
    std::vector<double> bsign;
  };
  std::vector<Loc> L(H.n_sub);
  for (int q = 0; q < sy; ++q)
    for (int p = 0; p < sx; ++p) {
      const int sid = q * sx + p;
      Loc& l = L[sid];
      l.icode.assign(H.nld, ldof_code(CAT_DIRICHLET, 0));
      for (int j = q * ey; j <= (q + 1) * ey; ++j)
        for (int i = p * ex; i <= (p + 1) * ex; ++i) {
          const int node = P.node_id(i, j);
          const int ln = (j - q * ey) * (ex + 1) + (i - p * ex);
          for (int c = 0; c < dpn; ++c) {
            const int md = node * dpn + c, f = P.free_map[md];
            if (f < 0) continue;
            int code;
            if (corner[node]) {
              code = ldof_code(CAT_CORNER, (int)l.cglob.size());
              l.cglob.push_back(corner_of[md]);
              l.cdof.push_back(f);
            } else if (lambda_of[md] >= 0) {
              code = ldof_code(CAT_BOUNDARY, (int)l.bdof.size());
              l.bdof.push_back(f);
              l.blam.push_back(lambda_of[md]);
              const auto po = owner_range(i, ex, sx);
              const auto qo = owner_range(j, ey, sy);
              l.bsign.push_back(sid == qo.first * sx + po.first ? 1.0 : -1.0);  // feti.cpp:117-121
            } else {
              code = ldof_code(CAT_INTERIOR, (int)l.idof.size());
              l.idof.push_back(f);
            }
            l.icode[ln * dpn + c] = code;
          }
        }
    }
  // interface edges (feti.cpp:132-167): vertical cuts (row q, cut p) then horizontal cuts;
  // free nodes strictly inside the segment, dpn multiplier rows per node
  struct EdgeRec {
    int lo, hi;
    bool vertical;
    std::vector<int> rows;
  };
  std::vector<EdgeRec> edges;
  auto add_edge = [&](int lo, int hi, bool vertical, const std::vector<int>& nodes) {
    if (nodes.empty()) return;
    EdgeRec e{lo, hi, vertical, {}};
    for (int node : nodes)
      for (int c = 0; c < dpn; ++c) e.rows.push_back(lambda_of[node * dpn + c]);
    edges.push_back(std::move(e));
  };
  for (int q = 0; q < sy; ++q)
    for (int p = 1; p < sx; ++p) {
      std::vector<int> nodes;
      for (int j = q * ey + 1; j < (q + 1) * ey; ++j)
        if (P.free_map[P.node_id(p * ex, j) * dpn] >= 0) nodes.push_back(P.node_id(p * ex, j));
      add_edge(q * sx + p - 1, q * sx + p, true, nodes);
    }
  for (int q = 1; q < sy; ++q)
    for (int p = 0; p < sx; ++p) {
      std::vector<int> nodes;
      for (int i = p * ex + 1; i < (p + 1) * ex; ++i)
        if (P.free_map[P.node_id(i, q * ey) * dpn] >= 0) nodes.push_back(P.node_id(i, q * ey));
      add_edge((q - 1) * sx + p, q * sx + p, false, nodes);
    }
  H.n_edges = (int)edges.size();
  // edge-RBM columns: the edge mean (scalar physics) or the two translations and the
  // in-plane rotation about the edge midpoint (plane strain), each normalised
  std::vector<std::vector<int>> sub_cols(H.n_sub);  // augmentation columns per subdomain
  if (augment) {
    H.col_ptr.push_back(0);
    for (int e = 0; e < (int)edges.size(); ++e) {
      const EdgeRec& ed = edges[e];
      const int nn = (int)ed.rows.size() / dpn;
      H.edge_col0.push_back((int)H.col_ptr.size() - 1);
      std::vector<std::pair<std::vector<int>, std::vector<double>>> cols;
      if (dpn == 1) {
        cols.push_back({ed.rows, std::vector<double>(nn, 1.0)});
      } else {
        std::vector<int> rx, ry, rr;
        std::vector<double> vr;
        for (int k = 0; k < nn; ++k) {
          rx.push_back(ed.rows[2 * k]);
          ry.push_back(ed.rows[2 * k + 1]);
          const double arm = (k - 0.5 * (nn - 1)) * P.h;
          rr.push_back(ed.vertical ? ed.rows[2 * k] : ed.rows[2 * k + 1]);
          vr.push_back(ed.vertical ? -arm : arm);
        }
        cols.push_back({rx, std::vector<double>(nn, 1.0)});
        cols.push_back({ry, std::vector<double>(nn, 1.0)});
        cols.push_back({rr, vr});
      }
      for (auto& c : cols) {
        double n2 = 0;
        for (double v : c.second) n2 += v * v;
        if (!(n2 > 0.0))
          throw NumericalError("build_edge_rbm_augmentation: dependent (zero) column on edge " + std::to_string(e) +
                               "; H/h too small for a rotation mode");
        const double inv = 1.0 / std::sqrt(n2);
        const int q = (int)H.col_ptr.size() - 1;
        for (size_t k = 0; k < c.first.size(); ++k) {
          H.col_rows.push_back(c.first[k]);
          H.col_vals.push_back(c.second[k] * inv);
        }
        H.col_ptr.push_back((int)H.col_rows.size());
        sub_cols[ed.lo].push_back(q);
        sub_cols[ed.hi].push_back(q);
      }
      H.edge_ncol.push_back((int)cols.size());
    }
    H.n_aug = (int)H.col_ptr.size() - 1;
    for (auto& v : sub_cols) std::sort(v.begin(), v.end());
  }
  H.n_coarse = H.n_corner + H.n_aug;

  const int S = H.n_sub;
  H.n_i.resize(S);
  H.n_b.resize(S);
  H.n_c.resize(S);
  for (int s = 0; s < S; ++s) {
    H.n_i[s] = (int)L[s].idof.size();
    H.n_b[s] = (int)L[s].bdof.size();
    H.n_c[s] = (int)L[s].cglob.size();
    H.NI = std::max(H.NI, H.n_i[s]);
    H.NB = std::max(H.NB, H.n_b[s]);
    H.NC = std::max(H.NC, H.n_c[s] + (int)sub_cols[s].size());
  }
  H.NI = std::max(H.NI, 1);
  H.NB = std::max(H.NB, 1);
  H.NC = std::max(H.NC, 1);
  H.ldof.resize((size_t)S * H.nld);
  H.idof.assign((size_t)S * H.NI, -1);
  H.bdof.assign((size_t)S * H.NB, -1);
  H.blam.assign((size_t)S * H.NB, -1);
  H.bsign.assign((size_t)S * H.NB, 0.0);
  H.cglob.assign((size_t)S * H.NC, -1);
  H.corner_dof.assign(H.n_corner, -1);
  H.lam_lo.assign(H.n_lambda, -1);
  H.lam_hi.assign(H.n_lambda, -1);
  H.corner_slots.assign((size_t)H.n_coarse * 4, -1);
  H.sub_i0.resize(S);
  H.sub_j0.resize(S);
  std::vector<int> ccount(H.n_coarse, 0);
  for (int s = 0; s < S; ++s) {
    const Loc& l = L[s];
    H.sub_i0[s] = (s % sx) * ex;
    H.sub_j0[s] = (s / sx) * ey;
    std::copy(l.icode.begin(), l.icode.end(), H.ldof.begin() + (size_t)s * H.nld);
    for (int k = 0; k < H.n_i[s]; ++k) H.idof[(size_t)s * H.NI + k] = l.idof[k];
    for (int k = 0; k < H.n_b[s]; ++k) {
      H.bdof[(size_t)s * H.NB + k] = l.bdof[k];
      H.blam[(size_t)s * H.NB + k] = l.blam[k];
      H.bsign[(size_t)s * H.NB + k] = l.bsign[k];
      int& slot = l.bsign[k] > 0 ? H.lam_lo[l.blam[k]] : H.lam_hi[l.blam[k]];
      if (slot != -1) throw NumericalError("partition: multiplier with two owners of one sign");
      slot = s * H.NB + k;
    }
    for (int k = 0; k < H.n_c[s]; ++k) {
      const int cg = l.cglob[k];
      H.cglob[(size_t)s * H.NC + k] = cg;
      H.corner_dof[cg] = l.cdof[k];
      if (ccount[cg] >= 4) throw NumericalError("partition: corner shared by more than 4 subdomains");
      H.corner_slots[(size_t)cg * 4 + ccount[cg]++] = s * H.NC + k;
    }
    // augmentation columns of the subdomain's edges after its corners; C^s^T entries on
    // the boundary rows with the subdomain's multiplier sign (feti.cpp:394-412)
    for (size_t a = 0; a < sub_cols[s].size(); ++a) {
      const int q = sub_cols[s][a], kc = H.n_c[s] + (int)a, cg = H.n_corner + q;
      H.cglob[(size_t)s * H.NC + kc] = cg;
      H.corner_slots[(size_t)cg * 4 + ccount[cg]++] = s * H.NC + kc;
      for (int e = H.col_ptr[q]; e < H.col_ptr[q + 1]; ++e) {
        const int row = H.col_rows[e];
        int kb = -1;
        for (int k = 0; k < H.n_b[s]; ++k)
          if (l.blam[k] == row) kb = k;
        if (kb < 0) throw NumericalError("augmentation: edge row not on the subdomain interface");
        H.aug_s.push_back(s);
        H.aug_kb.push_back(kb);
        H.aug_kc.push_back(kc);
        H.aug_val.push_back(l.bsign[kb] * H.col_vals[e]);
      }
    }
  }
  for (int r = 0; r < H.n_lambda; ++r)
    if (H.lam_lo[r] < 0 || H.lam_hi[r] < 0) throw NumericalError("partition: multiplier without two owners");

  // band half-width of A_ii (natural order) and the ELL widths, from element adjacency
  const int enl = 4;
  // per-row distinct-neighbour lists in flat scratch (at most 9 node neighbours x dpn),
  // reused across subdomains (no per-row allocations)
  const int KN = 9 * dpn;
  std::vector<int> bi_buf((size_t)H.NB * KN), ib_buf((size_t)H.NI * KN), bi_cnt(H.NB), ib_cnt(H.NI);
  auto add_unique = [KN](int* row, int& cnt, int v) {
    for (int k = 0; k < cnt; ++k)
      if (row[k] == v) return;
    if (cnt < KN) row[cnt++] = v;
  };
  // the widths depend on the local dof layout only: subdomains with an identical layout
  // (all interior ones, the edge classes, ...) are scanned once
  std::vector<std::pair<uint64_t, int>> seen;  // (hash of the layout, subdomain)
  for (int s = 0; s < S; ++s) {
    const int* code = &H.ldof[(size_t)s * H.nld];
    uint64_t hsh = 1469598103934665603ull;
    for (int k = 0; k < H.nld; ++k) hsh = (hsh ^ (uint64_t)(uint32_t)code[k]) * 1099511628211ull;
    bool dup = false;
    for (const auto& [h2, s2] : seen)
      if (h2 == hsh && std::equal(code, code + H.nld, &H.ldof[(size_t)s2 * H.nld])) dup = true;
    if (dup) continue;
    seen.push_back({hsh, s});
    std::fill(bi_cnt.begin(), bi_cnt.begin() + H.n_b[s], 0);
    std::fill(ib_cnt.begin(), ib_cnt.begin() + H.n_i[s], 0);
    for (int ey_ = 0; ey_ < ey; ++ey_)
      for (int ex_ = 0; ex_ < ex; ++ex_) {
        const int ln[enl] = {ey_ * (ex + 1) + ex_, ey_ * (ex + 1) + ex_ + 1, (ey_ + 1) * (ex + 1) + ex_ + 1,
                             (ey_ + 1) * (ex + 1) + ex_};
        for (int a = 0; a < enl; ++a)
          for (int ca = 0; ca < dpn; ++ca) {
            const int A = code[ln[a] * dpn + ca];
            for (int b = 0; b < enl; ++b)
              for (int cb = 0; cb < dpn; ++cb) {
                const int B = code[ln[b] * dpn + cb];
                if (ldof_cat(A) == CAT_INTERIOR && ldof_cat(B) == CAT_INTERIOR)
                  H.W = std::max(H.W, std::abs(ldof_idx(A) - ldof_idx(B)));
                if (ldof_cat(A) == CAT_BOUNDARY && ldof_cat(B) == CAT_INTERIOR)
                  add_unique(&bi_buf[(size_t)ldof_idx(A) * KN], bi_cnt[ldof_idx(A)], ldof_idx(B));
                if (ldof_cat(A) == CAT_INTERIOR && ldof_cat(B) == CAT_BOUNDARY)
                  add_unique(&ib_buf[(size_t)ldof_idx(A) * KN], ib_cnt[ldof_idx(A)], ldof_idx(B));
              }
          }
      }
    for (int k = 0; k < H.n_b[s]; ++k) H.MAXE_BI = std::max(H.MAXE_BI, bi_cnt[k]);
    for (int k = 0; k < H.n_i[s]; ++k) H.MAXE_IB = std::max(H.MAXE_IB, ib_cnt[k]);
  }
  H.MAXE_BI = std::max(H.MAXE_BI, 1);
  H.MAXE_IB = std::max(H.MAXE_IB, 1);
  // coarse band half-width in corner order
  for (int s = 0; s < S; ++s)
    for (int a = 0; a < H.n_c[s]; ++a)
      for (int b = 0; b < H.n_c[s]; ++b)
        H.WC = std::max(H.WC, std::abs(H.cglob[(size_t)s * H.NC + a] - H.cglob[(size_t)s * H.NC + b]));

  // primal assembly map (feti.cpp:699-708): interior -> 1 owner, boundary -> lo/hi, corner -> z
  H.xkind.assign(H.n_free, -1);
  H.xa.assign(H.n_free, -1);
  H.xb.assign(H.n_free, -1);
  for (int s = 0; s < S; ++s) {
    for (int k = 0; k < H.n_i[s]; ++k) {
      const int f = H.idof[(size_t)s * H.NI + k];
      H.xkind[f] = 0;
      H.xa[f] = s * H.NI + k;
    }
    for (int k = 0; k < H.n_b[s]; ++k) {
      const int f = H.bdof[(size_t)s * H.NB + k];
      const int r = H.blam[(size_t)s * H.NB + k];
      H.xkind[f] = 1;
      H.xa[f] = H.lam_lo[r];
      H.xb[f] = H.lam_hi[r];
    }
  }
  for (int c = 0; c < H.n_corner; ++c) {
    H.xkind[H.corner_dof[c]] = 2;
    H.xa[H.corner_dof[c]] = c;
  }
  for (int f = 0; f < H.n_free; ++f)
    if (H.xkind[f] < 0) throw NumericalError("partition: free dof owned by no subdomain");
  H.free_row.resize(H.n_free);
  for (int f = 0; f < H.n_free; ++f) H.free_row[f] = (P.free_dofs[f] / dpn) / (P.nx + 1);
  return H;
}

HostPartition build_rank_partition(const HostPartition& G, int rank, int world, RankPlan& plan) {
  if (world < 1 || rank < 0 || rank >= world) throw ContractError("rank partition: bad rank/world");
  if (G.sy % world != 0) throw ContractError("rank partition: subdomain rows must divide evenly over the ranks");
  const int sx = G.sx, rows = G.sy / world, NB = G.NB, NC = G.NC;
  plan = RankPlan{};
  plan.rank = rank;
  plan.world = world;
  plan.sub_first = rank * rows * sx;
  plan.n_sub_local = rows * sx;
  const int S = plan.n_sub_local, s0 = plan.sub_first;
  // phantoms: the lower neighbour row, then the upper one
  if (rank > 0)
    for (int p = 0; p < sx; ++p) plan.phantom_global.push_back(s0 - sx + p);
  if (rank < world - 1)
    for (int p = 0; p < sx; ++p) plan.phantom_global.push_back(s0 + S + p);
  plan.n_phantom = (int)plan.phantom_global.size();
  auto local_sub = [&](int sg) -> int {
    if (sg >= s0 && sg < s0 + S) return sg - s0;
    for (int p = 0; p < plan.n_phantom; ++p)
      if (plan.phantom_global[p] == sg) return S + p;
    return -1;
  };
  auto local_slot = [&](int gslot) -> int {
    const int ls = local_sub(gslot / NB);
    return ls < 0 ? -1 : ls * NB + gslot % NB;
  };
  auto is_local = [&](int gslot) { const int sg = gslot / NB; return sg >= s0 && sg < s0 + S; };
  // multiplier ranges: ghosts (bottom cut) then owned, contiguous in the global numbering
  int gmin = G.n_lambda, gmax = -1, omin = G.n_lambda, omax = -1;
  for (int r = 0; r < G.n_lambda; ++r) {
    if (is_local(G.lam_lo[r])) omin = std::min(omin, r), omax = std::max(omax, r), ++plan.n_owned;
    else if (is_local(G.lam_hi[r])) gmin = std::min(gmin, r), gmax = std::max(gmax, r), ++plan.n_ghost;
  }
  if (plan.n_owned > 0 && omax - omin + 1 != plan.n_owned) throw NumericalError("rank partition: owned rows not contiguous");
  if (plan.n_ghost > 0 && (gmax - gmin + 1 != plan.n_ghost || gmax + 1 != omin))
    throw NumericalError("rank partition: ghost rows not contiguous with the owned block");
  plan.lam_base = plan.n_ghost > 0 ? gmin : (plan.n_owned > 0 ? omin : 0);
  const int NL = plan.n_ghost + plan.n_owned;

  HostPartition L = G;  // copies scalars; per-subdomain arrays rebuilt below
  L.n_sub = S;
  L.n_lambda = NL;
  auto slice = [&](const auto& v, int width) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    return std::vector<T>(v.begin() + (size_t)s0 * width, v.begin() + (size_t)(s0 + S) * width);
  };
  L.ldof = slice(G.ldof, G.nld);
  L.idof = slice(G.idof, G.NI);
  L.bdof = slice(G.bdof, NB);
  L.bsign = slice(G.bsign, NB);
  L.n_i = slice(G.n_i, 1);
  L.n_b = slice(G.n_b, 1);
  L.n_c = slice(G.n_c, 1);
  L.sub_i0 = slice(G.sub_i0, 1);
  L.sub_j0 = slice(G.sub_j0, 1);
  L.blam = slice(G.blam, NB);
  for (int& r : L.blam)
    if (r >= 0) {
      r -= plan.lam_base;
      if (r < 0 || r >= NL) throw NumericalError("rank partition: interface dof outside the local multiplier range");
    }
  L.cglob.assign((size_t)(S + plan.n_phantom) * NC, -1);
  for (int ls = 0; ls < S + plan.n_phantom; ++ls) {
    const int sg = ls < S ? s0 + ls : plan.phantom_global[ls - S];
    for (int c = 0; c < NC; ++c) L.cglob[(size_t)ls * NC + c] = G.cglob[(size_t)sg * NC + c];
  }
  L.lam_lo.assign(NL, -1);
  L.lam_hi.assign(NL, -1);
  for (int r = 0; r < NL; ++r) {
    const int gr = plan.lam_base + r;
    L.lam_lo[r] = local_slot(G.lam_lo[gr]);
    L.lam_hi[r] = local_slot(G.lam_hi[gr]);
    if (L.lam_lo[r] < 0 || L.lam_hi[r] < 0) throw NumericalError("rank partition: multiplier owner outside the halo");
  }
  L.corner_slots.assign(G.corner_slots.size(), -1);  // local subdomains only (partial coarse sums)
  for (size_t q = 0; q < G.corner_slots.size(); ++q) {
    const int gs = G.corner_slots[q];
    if (gs >= 0 && (gs / NC) >= s0 && (gs / NC) < s0 + S) L.corner_slots[q] = (gs / NC - s0) * NC + gs % NC;
  }
  // top-cut rows: owned rows whose hi owner is an (upper) phantom
  for (int r = plan.n_ghost; r < NL; ++r)
    if (L.lam_hi[r] >= S * NB) ++plan.n_top_cut;
  for (int r = NL - plan.n_top_cut; r < NL; ++r)
    if (L.lam_hi[r] < S * NB) throw NumericalError("rank partition: top-cut rows not at the end of the owned block");
  // slot exchanges (canonical order = multiplier id)
  if (rank < world - 1) {
    plan.to_up.peer = rank + 1;
    for (int r = NL - plan.n_top_cut; r < NL; ++r) {
      plan.to_up.send_slots.push_back(L.lam_lo[r]);  // my side of the top cut
      plan.to_up.recv_slots.push_back(L.lam_hi[r]);  // the upper neighbour's side (phantom)
    }
  }
  if (rank > 0) {
    plan.to_down.peer = rank - 1;
    for (int r = 0; r < plan.n_ghost; ++r) {
      plan.to_down.send_slots.push_back(L.lam_hi[r]);  // my side of the bottom cut
      plan.to_down.recv_slots.push_back(L.lam_lo[r]);  // the lower neighbour's side (phantom)
    }
  }
  // owned free dofs: node rows (j0, j1] of this rank's band (contiguous in free-dof order)
  const int ey = G.ey;
  auto owned_range = [&](int rr, int& first, int& count) {
    const int j0 = rr * rows * ey, j1 = (rr + 1) * rows * ey;
    first = -1;
    count = 0;
    for (int f = 0; f < G.n_free; ++f) {
      const int j = G.free_row[f];
      const bool mine = (rr == 0 ? j >= 0 : j > j0) && j <= j1;
      if (mine) {
        if (first < 0) first = f;
        ++count;
      }
    }
    if (first < 0) first = 0;
  };
  plan.free_first_all.resize(world);
  plan.free_count_all.resize(world);
  for (int rr = 0; rr < world; ++rr) owned_range(rr, plan.free_first_all[rr], plan.free_count_all[rr]);
  plan.free_first = plan.free_first_all[rank];
  plan.free_count = plan.free_count_all[rank];
  L.xkind.assign(G.n_free, -1);
  L.xa.assign(G.n_free, -1);
  L.xb.assign(G.n_free, -1);
  for (int f = plan.free_first; f < plan.free_first + plan.free_count; ++f) {
    const int kind = G.xkind[f];
    L.xkind[f] = kind;
    if (kind == 0) {
      L.xa[f] = (G.xa[f] / G.NI - s0) * G.NI + G.xa[f] % G.NI;
      if (G.xa[f] / G.NI < s0 || G.xa[f] / G.NI >= s0 + S) throw NumericalError("rank partition: interior dof not local");
    } else if (kind == 1) {
      L.xa[f] = local_slot(G.xa[f]);
      L.xb[f] = local_slot(G.xb[f]);
      if (L.xa[f] < 0 || L.xb[f] < 0) throw NumericalError("rank partition: interface dof owner outside the halo");
    } else {
      L.xa[f] = G.xa[f];  // corner id (z is replicated)
    }
  }
  return L;
}

namespace {
double evaluate_target_thermal(double x1, double x2) {  // fem.cpp:194-202
  if (x1 <= 0.5 && x2 <= 0.5) {
    const double a = 2.0 * x1 - 1.0, b = 2.0 * x2 - 1.0;
    return a * a * b * b;
  }
  return 0.0;
}
}  // namespace

void target_thermal(const HostProblem& P, double* ybar, double* yc) {
  auto xy = [&](int md, double& x, double& y) {
    const int node = md / P.dpn;
    x = (node % (P.nx + 1)) * P.h;
    y = (node / (P.nx + 1)) * P.h;
  };
  double x, y;
  if (ybar)
    for (int f = 0; f < P.n(); ++f) xy(P.free_dofs[f], x, y), ybar[f] = evaluate_target_thermal(x, y);
  if (yc)
    for (int c = 0; c < P.m(); ++c) xy(P.cons_dofs[c], x, y), yc[c] = evaluate_target_thermal(x, y);
}

// BASELINE.json seeded target, recipe of SURVEY.md §8(d).  Independently restated in
// oracle/feti_oracle.cpp; tests/test_host.py checks the two agree bit for bit.
void bottom_pressure_load(const HostProblem& P, double pressure, double* f) {
  if (P.physics != 1) throw ContractError("bottom_pressure_load: elasticity physics required");
  std::fill(f, f + P.n(), 0.0);
  const double nodal = -pressure * P.h / 2.0;  // h/2 per end node of each bottom edge
  for (int i = 0; i < P.nx; ++i)
    for (int node : {P.node_id(i, 0), P.node_id(i + 1, 0)}) {
      const int fi = P.free_map[2 * node + 1];
      if (fi >= 0) f[fi] += nodal;
    }
}

void target_sine(const HostProblem& P, uint64_t seed, int modes, int mmax, double* ybar) {
  if (modes < 0 || mmax < 1) throw ContractError("target_sine: need modes >= 0 and mmax >= 1");
  std::mt19937_64 rng(seed);
  std::vector<double> amp(modes);
  std::vector<int> kx(modes), ky(modes);
  const double two53 = 9007199254740992.0;
  for (int k = 0; k < modes; ++k) {
    const double u1 = (double)(rng() >> 11) / two53;
    const double u2 = (double)(rng() >> 11) / two53;
    amp[k] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
    kx[k] = 1 + (int)(rng() % (uint64_t)mmax);
    ky[k] = 1 + (int)(rng() % (uint64_t)mmax);
  }
  for (int f = 0; f < P.n(); ++f) {
    const int node = P.free_dofs[f] / P.dpn;
    const double x = (node % (P.nx + 1)) * P.h, y = (node / (P.nx + 1)) * P.h;
    double v = 0.0;
    for (int k = 0; k < modes; ++k) v += amp[k] * std::sin(kx[k] * M_PI * x) * std::sin(ky[k] * M_PI * y);
    ybar[f] = v;
  }
}

}  // namespace fetigpu
