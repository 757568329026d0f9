// host_core.hpp — C++ host side of the B200 FETI-DP(H) path: structured mesh,
// free-dof numbering, Q1 element matrices, the reference partition rules and the
// flattened per-subdomain index tables the device kernels consume.
//
// Restates (not copies) the reference host logic:
//   build_rectangle_mesh      mesh.cpp:7-36
//   element matrices          fem.cpp:62-117
//   free/constrained numbering fem.cpp:133-150
//   partition_structured      feti.cpp:34-169  (corner rule, lambda numbering, signs)
// Everything here is O(n) integer bookkeeping run once per context.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fetigpu.h"

namespace fetigpu {

struct ContractError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Local-dof category codes of the per-subdomain table (ldof).
enum : int { CAT_DIRICHLET = 0, CAT_CORNER = 1, CAT_INTERIOR = 2, CAT_BOUNDARY = 3 };
inline int ldof_code(int cat, int idx) { return (cat << 24) | idx; }
inline int ldof_cat(int code) { return code >> 24; }
inline int ldof_idx(int code) { return code & 0xFFFFFF; }

struct HostProblem {
  int nx = 0, ny = 0, dpn = 1, physics = 0, edofs = 4;
  double h = 0, lx = 1, ly = 1, young = 0, poisson = 0;
  std::vector<int> free_map, cons_map;  // mesh dof -> free / constrained index, -1 otherwise
  std::vector<int> free_dofs, cons_dofs;
  double ke[64] = {}, me[64] = {};       // element matrices, row-major edofs x edofs
  int n() const { return (int)free_dofs.size(); }
  int m() const { return (int)cons_dofs.size(); }
  int node_id(int i, int j) const { return j * (nx + 1) + i; }
};

// Flattened partition in the layout the device wants.  Per-subdomain arrays are
// padded to the maxima (NI, NB, NC) so subdomain s owns a fixed-stride slab.
struct HostPartition {
  int sx = 0, sy = 0, ex = 0, ey = 0, dpn = 1;
  int n_sub = 0, n_free = 0, n_corner = 0, n_lambda = 0, n_edges = 0;
  int nld = 0;             // local mesh dofs per subdomain: (ex+1)(ey+1) dpn
  int NI = 0, NB = 0, NC = 0;
  int W = 0;               // max half-bandwidth of A_ii in natural order
  int WC = 0;              // half-bandwidth of the coarse matrix in corner order
  int MAXE_BI = 0, MAXE_IB = 0;  // ELL widths of A_bi (per b row) and A_ib (per i row)
  std::vector<int> n_i, n_b, n_c;        // per subdomain counts
  std::vector<int> ldof;                 // [S][nld] category/index codes
  std::vector<int> idof;                 // [S][NI] global free dof of interior k (-1 pad)
  std::vector<int> bdof;                 // [S][NB] global free dof of boundary k
  std::vector<int> blam;                 // [S][NB] multiplier row of boundary k (-1 pad)
  std::vector<double> bsign;             // [S][NB] +1 / -1 (0 pad)
  std::vector<int> cglob;                // [S][NC] global corner id (-1 pad)
  std::vector<int> corner_dof;           // [n_corner] global free dof of corner c
  std::vector<int> lam_lo, lam_hi;       // [n_lambda] flat slot s*NB+k of the +1 / -1 owner
  std::vector<int> corner_slots;         // [n_coarse][4] flat slot s*NC+k, ascending s, -1 pad
  // edge-RBM augmentation (augment = true; feti.cpp:171-242, 394-454).  The coarse unknowns
  // are [corner dofs | augmentation columns]; a subdomain's local coarse list is its corners
  // followed by the columns of its edges (ascending column id), so NC counts both.
  int n_coarse = 0, n_aug = 0;
  std::vector<int> aug_s, aug_kb, aug_kc;   // entries of C^s^T: subdomain, boundary index, local col
  std::vector<double> aug_val;              //   value sign * q (A_bc-like, A_ic part zero)
  std::vector<int> col_ptr, col_rows;       // [n_aug+1] / rows of column q (ascending by column)
  std::vector<double> col_vals;
  std::vector<int> edge_col0, edge_ncol;    // columns of edge e: [edge_col0[e], + edge_ncol[e])
  std::vector<int> xkind, xa, xb;        // [n_free] primal assembly map (0 int, 1 bnd, 2 corner)
  std::vector<int> free_row;             // [n_free] mesh node row j of each free dof
  // element-local structure: sub origin (node) for subdomain s
  std::vector<int> sub_i0, sub_j0;
};

// thread-local message returned by fetigpu_last_error (fetigpu.cu)
void set_last_error(const std::string& msg);

HostProblem build_problem(const fetigpu_desc& d);
HostPartition build_partition(const HostProblem& P, int sx, int sy, bool augment = false);

// ---------------------------------------------------------------------------------------
// Multi-GPU sharding.  Rank r of R owns the subdomain rows
// [r sy/R, (r+1) sy/R) (contiguous subdomain ids).  Its local view is a HostPartition over
// the local subdomains whose slot space is extended by "phantom" subdomains (the
// neighbour rows across each cut line), so every slot-indexed gather of the single-GPU
// kernels works unchanged.  Multipliers are numbered locally as
//   [ghost rows of the bottom cut (owned by r-1)] [owned rows, incl. the top cut]
// which is a contiguous range of the global numbering (multipliers ascend by node id).
struct SlotExchange {  // one direction of a neighbour exchange of per-dof slot values
  int peer = -1;
  std::vector<int> send_slots;  // local slots packed in canonical (multiplier id) order
  std::vector<int> recv_slots;  // phantom slots unpacked in the same order
};
struct RankPlan {
  int rank = 0, world = 1;
  int sub_first = 0, n_sub_local = 0, n_phantom = 0;
  int lam_base = 0;     // global id of local multiplier 0
  int n_ghost = 0;      // ghost rows [0, n_ghost) (bottom cut)
  int n_owned = 0;      // owned rows [n_ghost, n_ghost + n_owned)
  int n_top_cut = 0;    // last n_top_cut owned rows sit on the top cut (sent up as ghosts)
  int free_first = 0, free_count = 0;  // owned free dofs (x assembly)
  std::vector<int> free_first_all, free_count_all;  // per rank (all-gather of x)
  SlotExchange to_up, to_down;  // slot values sent to rank r+1 / r-1
  std::vector<int> phantom_global;  // global subdomain id of each phantom
};

// Local view for rank `rank` of `world` and its exchange plan (throws ContractError when
// the subdomain rows do not divide evenly).
HostPartition build_rank_partition(const HostPartition& G, int rank, int world, RankPlan& plan);

void target_thermal(const HostProblem& P, double* ybar, double* yc);
// consistent traction of a constant downward pressure on the bottom edge (fem.cpp:222-238)
void bottom_pressure_load(const HostProblem& P, double pressure, double* f);
void target_sine(const HostProblem& P, uint64_t seed, int modes, int mmax, double* ybar);

}  // namespace fetigpu
