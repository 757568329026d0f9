// host3d.hpp — C++ host side of the 3D extension (BASELINE.json configs 4-5: trilinear Q1
// hexahedra, heat with whole-boundary Dirichlet, linear elasticity clamped on x = 0).
//
// The reference is 2D only; the 3D rules are the natural extension of
// its 2D ones and are restated identically by the oracle (oracle/feti_oracle.cpp
// partition_structured3d):
//   mesh / free-dof order   mesh.cpp:7-36, fem.cpp:133-150 extruded in z (x fastest)
//   corners                 feti.cpp:55-65: free subdomain-grid vertices, multiplicity >= 2
//   multipliers             feti.cpp:69-81, 117-121 applied pairwise: a non-corner dof shared
//                           by s_1 < .. < s_m gets one row per pair (s_a, s_b), +1 on s_a;
//                           rows ascend by (node, component, pair)
//   Dirichlet scaling       W = 1/m per row (feti.cpp:602, 626 hard-code 1/2 = 1/m in 2D)
//   r-dof load weights      1/m (feti.cpp:505)
// Everything here is O(n) integer bookkeeping run once per context.
#pragma once

#include <cstdint>
#include <vector>

#include "fetigpu.h"
#include "host_core.hpp"

namespace fetigpu {

struct Host3Problem {
  int nx = 0, ny = 0, nz = 0, dpn = 1, physics = 0, edofs = 8;
  double h = 0, lx = 1, ly = 1, lz = 1, young = 0, poisson = 0;
  std::vector<int> free_map, cons_map, free_dofs, cons_dofs;
  double ke[576] = {}, me[576] = {};  // row-major edofs x edofs, dof = dpn * local node + comp
  int n() const { return (int)free_dofs.size(); }
  int m() const { return (int)cons_dofs.size(); }
  int node_id(int i, int j, int k) const { return (k * (ny + 1) + j) * (nx + 1) + i; }
};

// Flattened 3D partition in the layout the device wants (per-subdomain slabs padded to
// NI / NB / NC; jump entries padded to MR rows per interface dof).
struct Host3Partition {
  int sx = 0, sy = 0, sz = 0, ex = 0, ey = 0, ez = 0, dpn = 1;
  int S = 0, n_free = 0, n_corner = 0, n_lambda = 0;
  int nld = 0;        // local mesh dofs per subdomain (ex+1)(ey+1)(ez+1) dpn
  int NI = 0;         // max interior dofs, rounded up to a multiple of 32 (block rows of A_ii)
  int NB = 0, NC = 0; // max interface / corner dofs
  int MR = 1;         // max multiplier rows per interface dof of one subdomain
  int P = 0;          // block half-bandwidth of A_ii in 32-row blocks (natural order)
  int MAXE_BI = 0, MAXE_IB = 0;  // ELL widths of A_bi rows / A_ib rows
  std::vector<int> n_i, n_b, n_c;
  std::vector<int> ldof;            // [S][nld] category/index code (ldof_code of host_core.hpp)
  std::vector<int> idof, bdof;      // [S][NI] / [S][NB] global free dof (-1 pad)
  std::vector<int> cglob;           // [S][NC] global corner id (-1 pad)
  std::vector<int> brow;            // [S][NB][MR] multiplier rows of interface dof k (-1 pad)
  std::vector<double> bsgn;         // [S][NB][MR] +1 / -1 (0 pad)
  std::vector<double> bw;           // [S][NB] load weight 1/mult
  std::vector<int> lam_lo, lam_hi;  // [n_lambda] flat slot s*NB+k of the +1 / -1 owner
  std::vector<double> lam_w;        // [n_lambda] Dirichlet scaling 1/mult
  std::vector<int> corner_dof;      // [n_corner] global free dof
  std::vector<int> corner_slots;    // [n_corner][8] flat slot s*NC+k, ascending s (-1 pad)
  std::vector<int> xref;            // [n_free][4]: primal assembly refs (see xkind)
  std::vector<int> xkind;           // [n_free] 0 interior (xref[0] = s*NI+k), 1 interface (up to 4
                                    // slots s*NB+k, -1 pad), 2 corner (xref[0] = corner id)
  std::vector<double> xw;           // [n_free] weight of interface slots (1/mult)
  std::vector<int> sub_i0, sub_j0, sub_k0;  // element origin of each subdomain
  // sharded view (local_partition3d): global id of local subdomain 0, rank, world
  int s_first = 0, rank = 0, world = 1;
};

Host3Problem build_problem3d(const fetigpu3d_desc& d);
Host3Partition build_partition3d(const Host3Problem& P, int sx, int sy, int sz);
// Multi-GPU view: rank r of R owns the subdomain ids [r S/R, (r+1) S/R) of
// the z-outer ordering — whole z-layers when R divides s_z, else y-row blocks of a layer.  Per-subdomain tables are
// sliced; multiplier rows stay global (dual vectors are replicated on every rank) with the
// slot of a non-local owner set to -1, so every jump gather yields this rank's partial sum
// and one allreduce completes it (each row has exactly two owners: the sum is exact).
// Corner slots / primal refs keep local slots only; corner values are assembled by rank 0.
Host3Partition local_partition3d(const Host3Partition& G, int rank, int world);
// seeded sine-mode target of configs 4-5: a_k (Box-Muller), l_k, m_k, n_k =
// 1 + rng() % mmax; the same scalar field for every component (2D plane strain convention)
void target_sine3d(const Host3Problem& P, uint64_t seed, int modes, int mmax, double* ybar);

}  // namespace fetigpu
