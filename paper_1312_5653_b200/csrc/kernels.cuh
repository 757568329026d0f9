// kernels.cuh — FETI-DP(H) device kernels other than the banded ones (band.cuh).
//
// Layout (all complex = double2, per-subdomain slabs padded to NI / NB / NC):
//   bi_idx/bi_val [S][NB][EBI]   A_bi as ELL rows (interior column, value)
//   ib_idx/ib_val [S][NI][EIB]   A_ib as ELL rows (boundary column, value)
//   Sbb, Sinv     [S][NB][NB]    Dirichlet Schur complement S_bb = A_bb - A_bi A_ii^-1 A_ib
//                                and its inverse S_bb^-1 = (A_rr^-1)_bb
//   Aic [S][NI][NC], Abc [S][NB][NC], Acc [S][NC][NC]   corner couplings
//   cpl_i [S][NI][NC], cpl_b [S][NB][NC]                coupling = A_rr^-1 A_rc (feti.cpp:432)
// A_rr is never formed: with r = [interior | boundary],
//   A_rr^-1 t = [ y_i - A_ii^-1 A_ib u_b ; u_b ],  y_i = A_ii^-1 t_i,  u_b = S_bb^-1 (t_b - A_bi y_i),
// an exact block LDL^T of A_rr (banded interior factor + dense boundary Schur factor).
#pragma once

#include "common.cuh"

namespace fetigpu {

constexpr int MAX_EDOFS = 8;
constexpr int MAXE = 24;  // ELL capacity checked on the host

__constant__ double2 c_Ae[MAX_EDOFS * MAX_EDOFS];  // Ae = kc*Ke + mc*Me (feti.cpp:264-265)
__constant__ double c_Ke[MAX_EDOFS * MAX_EDOFS];
__constant__ double c_Me[MAX_EDOFS * MAX_EDOFS];

struct SubLayout {
  int S, nld, ex, ey, dpn, NI, NB, NC, W, EBI, EIB;
};

// ------------------------------------------------------------------ K1 block assembly
// One thread per (subdomain, local mesh dof a).  The thread owns row a of every block it
// belongs to, visits the <= 4 elements around its node in ascending element id (the
// reference's sub.elements order, feti.cpp:305) and accumulates deterministically.
__global__ void k_assemble(SubLayout L, const int* __restrict__ ldof, double2* __restrict__ colband,
                           int* __restrict__ bi_idx, double2* __restrict__ bi_val, int* __restrict__ ib_idx,
                           double2* __restrict__ ib_val, double2* __restrict__ Sbb, double2* __restrict__ Aic,
                           double2* __restrict__ Abc, double2* __restrict__ Acc) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)L.S * L.nld) return;
  const int s = (int)(gid / L.nld), a = (int)(gid % L.nld);
  const int* code = ldof + (size_t)s * L.nld;
  const int ca = code[a];
  const int cat_a = ca >> 24, ia = ca & 0xFFFFFF;
  if (cat_a == 0) return;
  const int dpn = L.dpn, ed = 4 * dpn, LD = L.W + 1;
  const int node = a / dpn, comp = a % dpn;
  const int lx = node % (L.ex + 1), ly = node / (L.ex + 1);
  int eidx[MAXE];
  double2 evals[MAXE];
  int ecount = 0;
  for (int ey_ = ly - 1; ey_ <= ly; ++ey_) {
    if (ey_ < 0 || ey_ >= L.ey) continue;
    for (int ex_ = lx - 1; ex_ <= lx; ++ex_) {
      if (ex_ < 0 || ex_ >= L.ex) continue;
      const int en[4] = {ey_ * (L.ex + 1) + ex_, ey_ * (L.ex + 1) + ex_ + 1, (ey_ + 1) * (L.ex + 1) + ex_ + 1,
                         (ey_ + 1) * (L.ex + 1) + ex_};
      int alpha = 0;
      for (int q = 0; q < 4; ++q)
        if (en[q] == node) alpha = q;
      const int ra = dpn * alpha + comp;
      for (int b = 0; b < 4; ++b)
        for (int cb = 0; cb < dpn; ++cb) {
          const int code_b = code[en[b] * dpn + cb];
          const int cat_b = code_b >> 24, ib = code_b & 0xFFFFFF;
          if (cat_b == 0) continue;
          const double2 v = c_Ae[ra * ed + dpn * b + cb];
          if (cat_a == 2) {  // interior row
            if (cat_b == 2) {
              if (ib <= ia) {
                double2& t = colband[((size_t)s * L.NI + ib) * LD + (ia - ib)];
                t = cadd(t, v);
              }
            } else if (cat_b == 3) {
              int e = 0;
              while (e < ecount && eidx[e] != ib) ++e;
              if (e == ecount) {
                eidx[ecount] = ib;
                evals[ecount++] = v;
              } else {
                evals[e] = cadd(evals[e], v);
              }
            } else {  // corner
              double2& t = Aic[((size_t)s * L.NI + ia) * L.NC + ib];
              t = cadd(t, v);
            }
          } else if (cat_a == 3) {  // boundary row
            if (cat_b == 2) {
              int e = 0;
              while (e < ecount && eidx[e] != ib) ++e;
              if (e == ecount) {
                eidx[ecount] = ib;
                evals[ecount++] = v;
              } else {
                evals[e] = cadd(evals[e], v);
              }
            } else if (cat_b == 3) {
              double2& t = Sbb[((size_t)s * L.NB + ia) * L.NB + ib];
              t = cadd(t, v);
            } else {
              double2& t = Abc[((size_t)s * L.NB + ia) * L.NC + ib];
              t = cadd(t, v);
            }
          } else {  // corner row: only the corner-corner block is needed (symmetry)
            if (cat_b == 1) {
              double2& t = Acc[((size_t)s * L.NC + ia) * L.NC + ib];
              t = cadd(t, v);
            }
          }
        }
    }
  }
  if (cat_a == 2) {
    for (int e = 0; e < L.EIB; ++e) {
      ib_idx[((size_t)s * L.NI + ia) * L.EIB + e] = e < ecount ? eidx[e] : -1;
      ib_val[((size_t)s * L.NI + ia) * L.EIB + e] = e < ecount ? evals[e] : cz();
    }
  } else if (cat_a == 3) {
    for (int e = 0; e < L.EBI; ++e) {
      bi_idx[((size_t)s * L.NB + ia) * L.EBI + e] = e < ecount ? eidx[e] : -1;
      bi_val[((size_t)s * L.NB + ia) * L.EBI + e] = e < ecount ? evals[e] : cz();
    }
  }
}

// identity rows/cols for padding: colband rows >= n_i, Sbb rows/cols >= n_b
__global__ void k_pad_identity(SubLayout L, const int* __restrict__ n_i, const int* __restrict__ n_b,
                               double2* __restrict__ colband, double2* __restrict__ Sbb) {
  const int s = blockIdx.x;
  const int LD = L.W + 1;
  for (int i = n_i[s] + threadIdx.x; i < L.NI; i += blockDim.x)
    colband[((size_t)s * L.NI + i) * LD] = make_double2(1.0, 0.0);
  for (int i = n_b[s] + threadIdx.x; i < L.NB; i += blockDim.x)
    Sbb[((size_t)s * L.NB + i) * L.NB + i] = make_double2(1.0, 0.0);
}

// Y[s][b][i] = A_ib(i, b) (RHS-major, one RHS per boundary dof); Y pre-zeroed
__global__ void k_build_aib_rhs(SubLayout L, const int* __restrict__ bi_idx, const double2* __restrict__ bi_val,
                                double2* __restrict__ Y) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)L.S * L.NB * L.EBI) return;
  const int e = (int)(gid % L.EBI);
  const long long sb = gid / L.EBI;
  const int i = bi_idx[sb * L.EBI + e];
  if (i >= 0) Y[sb * L.NI + i] = bi_val[sb * L.EBI + e];
}

// Yc[s][c][i] = A_ic(i, c)
__global__ void k_build_aic_rhs(SubLayout L, const double2* __restrict__ Aic, double2* __restrict__ Yc) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)L.S * L.NI * L.NC) return;
  const int c = (int)(gid % L.NC);
  const long long si = gid / L.NC;
  const int s = (int)(si / L.NI), i = (int)(si % L.NI);
  Yc[((size_t)s * L.NC + c) * L.NI + i] = Aic[gid];
}

// S_bb(b1, b2) -= sum_e A_bi(b1, e) Y[b2][e]   (the Schur complement of feti.cpp:611-617)
__global__ void k_schur_bb(SubLayout L, const int* __restrict__ bi_idx, const double2* __restrict__ bi_val,
                           const double2* __restrict__ Y, double2* __restrict__ Sbb) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)L.S * L.NB * L.NB) return;
  const int b2 = (int)(gid % L.NB);
  const long long sb1 = gid / L.NB;
  const int s = (int)(sb1 / L.NB);
  const double2* yrow = Y + ((size_t)s * L.NB + b2) * L.NI;
  double2 acc = Sbb[gid];
  for (int e = 0; e < L.EBI; ++e) {
    const int i = bi_idx[sb1 * L.EBI + e];
    if (i >= 0) acc = cfms(bi_val[sb1 * L.EBI + e], yrow[i], acc);
  }
  Sbb[gid] = acc;
}

// In-place Gauss-Jordan inverse (no pivoting: S_bb has an SPD real part) of the n x n
// matrices A[s] (row stride n).  One CTA per matrix; status[s] = 1 + failing pivot.
__global__ void __launch_bounds__(256) k_gauss_jordan(double2* __restrict__ A, int n, int* __restrict__ status) {
  extern __shared__ double2 gj_sh[];
  double2* rowk = gj_sh;
  double2* colk = gj_sh + n;
  const int s = blockIdx.x, tid = threadIdx.x;
  double2* M = A + (size_t)s * n * n;
  int bad = 0;
  for (int k = 0; k < n; ++k) {
    for (int j = tid; j < n; j += blockDim.x) {
      rowk[j] = M[(size_t)k * n + j];
      colk[j] = M[(size_t)j * n + k];
    }
    __syncthreads();
    const double2 p = rowk[k];
    const double2 pinv = crecip(p);
    if (tid == 0 && bad == 0) {
      const double a2 = cabs2(p);
      if (!(a2 > 0.0) || !isfinite(a2)) bad = k + 1;
    }
    for (int idx = tid; idx < n * n; idx += blockDim.x) {
      const int i = idx / n, j = idx % n;
      double2 v;
      if (i == k)
        v = (j == k) ? pinv : cmul(rowk[j], pinv);
      else if (j == k)
        v = cmul(make_double2(-colk[i].x, -colk[i].y), pinv);
      else
        v = cfms(cmul(colk[i], pinv), rowk[j], M[idx]);
      M[idx] = v;
    }
    __syncthreads();
  }
  if (tid == 0) status[s] = bad;
}

// coupling_b = S_bb^-1 (A_bc - A_bi Yc),  Yc = A_ii^-1 A_ic.  One CTA per subdomain.
__global__ void k_coupling_b(SubLayout L, const double2* __restrict__ Sinv, const double2* __restrict__ Abc,
                             const int* __restrict__ bi_idx, const double2* __restrict__ bi_val,
                             const double2* __restrict__ Yc, double2* __restrict__ cpl_b) {
  extern __shared__ double2 q_sh[];  // [NB][NC]
  const int s = blockIdx.x;
  for (int idx = threadIdx.x; idx < L.NB * L.NC; idx += blockDim.x) {
    const int b = idx / L.NC, c = idx % L.NC;
    double2 acc = Abc[(size_t)s * L.NB * L.NC + idx];
    const size_t sb = (size_t)s * L.NB + b;
    for (int e = 0; e < L.EBI; ++e) {
      const int i = bi_idx[sb * L.EBI + e];
      if (i >= 0) acc = cfms(bi_val[sb * L.EBI + e], Yc[((size_t)s * L.NC + c) * L.NI + i], acc);
    }
    q_sh[idx] = acc;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < L.NB * L.NC; idx += blockDim.x) {
    const int b = idx / L.NC, c = idx % L.NC;
    const double2* srow = Sinv + ((size_t)s * L.NB + b) * L.NB;
    double2 acc = cz();
    for (int k = 0; k < L.NB; ++k) acc = cfma(srow[k], q_sh[k * L.NC + c], acc);
    cpl_b[(size_t)s * L.NB * L.NC + idx] = acc;
  }
}

// coupling_i = Yc - Y coupling_b   (Y = A_ii^-1 A_ib, RHS-major)
__global__ void k_coupling_i(SubLayout L, const double2* __restrict__ Yc, const double2* __restrict__ Y,
                             const double2* __restrict__ cpl_b, double2* __restrict__ cpl_i) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)L.S * L.NI) return;
  const int s = (int)(gid / L.NI), i = (int)(gid % L.NI);
  double2 acc[8];
  for (int c = 0; c < L.NC; ++c) acc[c] = Yc[((size_t)s * L.NC + c) * L.NI + i];
  for (int b = 0; b < L.NB; ++b) {
    const double2 y = Y[((size_t)s * L.NB + b) * L.NI + i];
    for (int c = 0; c < L.NC; ++c) acc[c] = cfms(y, cpl_b[((size_t)s * L.NB + b) * L.NC + c], acc[c]);
  }
  for (int c = 0; c < L.NC; ++c) cpl_i[((size_t)s * L.NI + i) * L.NC + c] = acc[c];
}

// contrib[s] = A_rc^T coupling (transpose, not adjoint: feti.cpp:433). One warp per entry.
__global__ void k_coarse_contrib(SubLayout L, const double2* __restrict__ Aic, const double2* __restrict__ Abc,
                                 const double2* __restrict__ cpl_i, const double2* __restrict__ cpl_b,
                                 double2* __restrict__ contrib) {
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int e = warp; e < L.NC * L.NC; e += nw) {
    const int a = e / L.NC, b = e % L.NC;
    double2 acc = cz();
    for (int i = lane; i < L.NI; i += 32)
      acc = cfma(Aic[((size_t)s * L.NI + i) * L.NC + a], cpl_i[((size_t)s * L.NI + i) * L.NC + b], acc);
    for (int k = lane; k < L.NB; k += 32)
      acc = cfma(Abc[((size_t)s * L.NB + k) * L.NC + a], cpl_b[((size_t)s * L.NB + k) * L.NC + b], acc);
    acc = warp_sum2(acc);
    if (lane == 0) contrib[((size_t)s * L.NC + a) * L.NC + b] = acc;
  }
}

// Coarse band assembly (feti.cpp:440-454), one thread per coarse row r, subdomains in
// ascending order, "+= A_cc then -= contrib" per subdomain as the reference does.
__global__ void k_coarse_assemble(int nc, int WC, int NC, const int* __restrict__ corner_slots,
                                  const int* __restrict__ cglob, const double2* __restrict__ Acc,
                                  const double2* __restrict__ contrib, double2* __restrict__ cband) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nc) return;
  const int LDC = WC + 1;
  for (int q = 0; q < 4; ++q) {
    const int slot = corner_slots[r * 4 + q];
    if (slot < 0) continue;
    const int s = slot / NC, ka = slot % NC;
    for (int kb = 0; kb < NC; ++kb) {
      const int col = cglob[(size_t)s * NC + kb];
      if (col < 0 || col > r) continue;
      double2& t = cband[(size_t)col * LDC + (r - col)];
      t = cadd(t, Acc[((size_t)s * NC + ka) * NC + kb]);
    }
    for (int kb = 0; kb < NC; ++kb) {
      const int col = cglob[(size_t)s * NC + kb];
      if (col < 0 || col > r) continue;
      double2& t = cband[(size_t)col * LDC + (r - col)];
      t = csub(t, contrib[((size_t)s * NC + ka) * NC + kb]);
    }
  }
}

// symmetric equilibration 1/sqrt|diag| (feti.cpp:460-467)
__global__ void k_coarse_scale(int nc, int WC, double2* __restrict__ cband, double* __restrict__ scale) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nc) return;
  const double d = sqrt(cabs2(cband[(size_t)r * (WC + 1)]));
  scale[r] = d > 0.0 ? 1.0 / sqrt(d) : 1.0;
}
__global__ void k_coarse_apply_scale(int nc, int WC, double2* __restrict__ cband, const double* __restrict__ scale) {
  const int col = blockIdx.x;
  for (int k = threadIdx.x; k <= WC; k += blockDim.x) {
    if (col + k >= nc) continue;
    double2& t = cband[(size_t)col * (WC + 1) + k];
    t = cscale(t, scale[col] * scale[col + k]);
  }
}
// X[c][r] = delta_rc (identity RHS block, RHS-major)
__global__ void k_identity(int n, double2* __restrict__ X) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)n * n) return;
  X[gid] = (gid / n == gid % n) ? make_double2(1.0, 0.0) : cz();
}
// Cinv[c][r] = scale_c X[c][r] scale_r  (C^-1 = D (DCD)^-1 D)
__global__ void k_scale_inverse(int n, double2* __restrict__ X, const double* __restrict__ scale) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)n * n) return;
  X[gid] = cscale(X[gid], scale[gid / n] * scale[gid % n]);
}

// --------------------------------------------------------------- per-iteration kernels
// K5/K6 local operator apply, one CTA per subdomain:
//   in_b[k] = alpha * sign_k * lam[row_k]            (B^T scatter, feti.cpp:588-589 / 609-610)
//   out_b   = M_s in_b                               (M = S_bb: Dirichlet; M = S_bb^-1: dual)
//   gcp[c]  = sum_k cpl_b[k][c] in_b[k]              (= A_rc^T A_rr^-1 t, optional)
// M rows are streamed once, 16 B per lane per load, 2 rows in flight per warp.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_bnd_gemv(int NB, int NC, const double2* __restrict__ M, const int* __restrict__ blam,
               const double* __restrict__ bsign, const double2* __restrict__ lam, double alpha,
               double2* __restrict__ out_b, const double2* __restrict__ cpl_b, double2* __restrict__ gcp) {
  extern __shared__ double2 in_sh[];
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < NB; k += blockDim.x) {
    const int r = blam[(size_t)s * NB + k];
    in_sh[k] = r >= 0 ? cscale(lam[r], alpha * bsign[(size_t)s * NB + k]) : cz();
  }
  __syncthreads();
  const double2* Ms = M + (size_t)s * NB * NB;
  int row = warp;
  for (; row + WARPS < NB; row += 2 * WARPS) {
    const double2* r0 = Ms + (size_t)row * NB;
    const double2* r1 = Ms + (size_t)(row + WARPS) * NB;
    double2 a0 = cz(), a1 = cz();
    for (int k = lane; k < NB; k += 32) {
      const double2 m0 = __ldcs(r0 + k), m1 = __ldcs(r1 + k);
      const double2 v = in_sh[k];
      a0 = cfma(m0, v, a0);
      a1 = cfma(m1, v, a1);
    }
    a0 = warp_sum2(a0);
    a1 = warp_sum2(a1);
    if (lane == 0) {
      out_b[(size_t)s * NB + row] = a0;
      out_b[(size_t)s * NB + row + WARPS] = a1;
    }
  }
  for (; row < NB; row += WARPS) {
    const double2* r0 = Ms + (size_t)row * NB;
    double2 a0 = cz();
    for (int k = lane; k < NB; k += 32) a0 = cfma(__ldcs(r0 + k), in_sh[k], a0);
    a0 = warp_sum2(a0);
    if (lane == 0) out_b[(size_t)s * NB + row] = a0;
  }
  if (gcp != nullptr) {
    for (int c = warp; c < NC; c += WARPS) {
      double2 acc = cz();
      for (int k = lane; k < NB; k += 32) acc = cfma(cpl_b[((size_t)s * NB + k) * NC + c], in_sh[k], acc);
      acc = warp_sum2(acc);
      if (lane == 0) gcp[(size_t)s * NC + c] = acc;
    }
  }
}

// Dirichlet tail: out[r] = (w_lo - w_hi) / 2   (feti.cpp:620-626, signs +1 / -1)
__global__ void k_lam_gather_pre(int nl, const int* __restrict__ lo, const int* __restrict__ hi,
                                 const double2* __restrict__ wb, double2* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nl) return;
  out[r] = cscale(csub(wb[lo[r]], wb[hi[r]]), 0.5);
}

// g[c] = fc[c] - sum_slots gcp[slot]   (feti.cpp:523-538, subdomains ascending)
__global__ void k_coarse_rhs(int nc, const int* __restrict__ corner_slots, const double2* __restrict__ gcp,
                             const double2* __restrict__ fc, double2* __restrict__ g) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double2 acc = fc ? fc[c] : cz();
  for (int q = 0; q < 4; ++q) {
    const int slot = corner_slots[c * 4 + q];
    if (slot >= 0) acc = csub(acc, gcp[slot]);
  }
  g[c] = acc;
}

// z = C^-1 g  (dense explicit coarse inverse, K4), one warp per row, g staged in smem
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_coarse_gemv(int nc, const double2* __restrict__ Cinv, const double2* __restrict__ g, double2* __restrict__ z) {
  extern __shared__ double2 g_sh[];
  for (int k = threadIdx.x; k < nc; k += blockDim.x) g_sh[k] = g[k];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int row = blockIdx.x * WARPS + warp; row < nc; row += gridDim.x * WARPS) {
    const double2* cr = Cinv + (size_t)row * nc;
    double2 a = cz();
    for (int k = lane; k < nc; k += 32) a = cfma(cr[k], g_sh[k], a);
    a = warp_sum2(a);
    if (lane == 0) z[row] = a;
  }
}

// Dual tail: u_b = u1_b - cpl_b z_loc ; out[r] = -(u_lo - u_hi)   (feti.cpp:542-555, 593)
__global__ void k_lam_gather_dual(int nl, int NB, int NC, const int* __restrict__ lo, const int* __restrict__ hi,
                                  const double2* __restrict__ u1b, const double2* __restrict__ cpl_b,
                                  const int* __restrict__ cglob, const double2* __restrict__ z,
                                  double2* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nl) return;
  double2 u[2];
  const int slots[2] = {lo[r], hi[r]};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int slot = slots[q];
    const int s = slot / NB;
    double2 acc = cz();
    for (int c = 0; c < NC; ++c) {
      const int cg = cglob[(size_t)s * NC + c];
      if (cg >= 0) acc = cfma(cpl_b[(size_t)slot * NC + c], z[cg], acc);
    }
    u[q] = csub(u1b[slot], acc);
  }
  const double2 d = csub(u[0], u[1]);
  out[r] = make_double2(-d.x, -d.y);
}

// ------------------------------------------------------------------ eliminate pieces
// split_rhs (feti.cpp:493-510): f_i = rhs[idof], f_b = rhs[bdof] / 2 (w = 1/mult = 1/2)
__global__ void k_split_rhs(SubLayout L, const int* __restrict__ idof, const int* __restrict__ bdof,
                            const double2* __restrict__ rhs, double2* __restrict__ fi, double2* __restrict__ fb) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long ni = (long long)L.S * L.NI, nb = (long long)L.S * L.NB;
  if (gid < ni) {
    const int f = idof[gid];
    fi[gid] = f >= 0 ? rhs[f] : cz();
  } else if (gid < ni + nb) {
    const long long k = gid - ni;
    const int f = bdof[k];
    fb[k] = f >= 0 ? cscale(rhs[f], 0.5) : cz();
  }
}
__global__ void k_gather_corner(int nc, const int* __restrict__ corner_dof, const double2* __restrict__ rhs,
                                double2* __restrict__ fc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc) fc[c] = rhs[corner_dof[c]];
}
// t_b = f_b - sign * lam[row]  (feti.cpp:690-696)
__global__ void k_recover_tb(int nsb, const int* __restrict__ blam, const double* __restrict__ bsign,
                             const double2* __restrict__ fb, const double2* __restrict__ lam,
                             double2* __restrict__ tb) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nsb) return;
  const int r = blam[k];
  tb[k] = r >= 0 ? cfms(make_double2(bsign[k], 0.0), lam[r], fb[k]) : cz();
}

// u1_b = S_bb^-1 (t_b - A_bi y_i) and gcp_b[c] = sum_k A_bc(k,c) u1_b[k]; one CTA per subdomain
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_elim_b(SubLayout L, const double2* __restrict__ Sinv, const double2* __restrict__ tb,
             const int* __restrict__ bi_idx, const double2* __restrict__ bi_val, const double2* __restrict__ yi,
             double2* __restrict__ u1b) {
  extern __shared__ double2 q_sh2[];
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < L.NB; k += blockDim.x) {
    const size_t sb = (size_t)s * L.NB + k;
    double2 acc = tb[sb];
    for (int e = 0; e < L.EBI; ++e) {
      const int i = bi_idx[sb * L.EBI + e];
      if (i >= 0) acc = cfms(bi_val[sb * L.EBI + e], yi[(size_t)s * L.NI + i], acc);
    }
    q_sh2[k] = acc;
  }
  __syncthreads();
  for (int row = warp; row < L.NB; row += WARPS) {
    const double2* r0 = Sinv + ((size_t)s * L.NB + row) * L.NB;
    double2 a = cz();
    for (int k = lane; k < L.NB; k += 32) a = cfma(r0[k], q_sh2[k], a);
    a = warp_sum2(a);
    if (lane == 0) u1b[(size_t)s * L.NB + row] = a;
  }
}
// r_i = A_ib u1_b
__global__ void k_ib_apply(SubLayout L, const int* __restrict__ ib_idx, const double2* __restrict__ ib_val,
                           const double2* __restrict__ u1b, double2* __restrict__ ri) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)L.S * L.NI) return;
  const int s = (int)(gid / L.NI);
  double2 acc = cz();
  for (int e = 0; e < L.EIB; ++e) {
    const int b = ib_idx[gid * L.EIB + e];
    if (b >= 0) acc = cfma(ib_val[gid * L.EIB + e], u1b[(size_t)s * L.NB + b], acc);
  }
  ri[gid] = acc;
}
// u1_i = y_i - ri (ri already A_ii^-1 A_ib u1_b); gcp[c] = A_ic^T u1_i + A_bc^T u1_b
__global__ void k_elim_i_gcp(SubLayout L, const double2* __restrict__ yi, double2* __restrict__ ri,
                             const double2* __restrict__ u1b, const double2* __restrict__ Aic,
                             const double2* __restrict__ Abc, double2* __restrict__ gcp) {
  __shared__ double2 red[8][32];
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 acc[8];
  for (int c = 0; c < 8; ++c) acc[c] = cz();
  for (int i = threadIdx.x; i < L.NI; i += blockDim.x) {
    const size_t si = (size_t)s * L.NI + i;
    const double2 u = csub(yi[si], ri[si]);
    ri[si] = u;  // ri now holds u1_i
    for (int c = 0; c < L.NC; ++c) acc[c] = cfma(Aic[si * L.NC + c], u, acc[c]);
  }
  for (int k = threadIdx.x; k < L.NB; k += blockDim.x) {
    const size_t sb = (size_t)s * L.NB + k;
    for (int c = 0; c < L.NC; ++c) acc[c] = cfma(Abc[sb * L.NC + c], u1b[sb], acc[c]);
  }
  for (int c = 0; c < L.NC; ++c) {
    const double2 v = warp_sum2(acc[c]);
    if (lane == 0) red[c][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < L.NC) {
    double2 t = cz();
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = cadd(t, red[threadIdx.x][w]);
    gcp[(size_t)s * L.NC + threadIdx.x] = t;
  }
}
// u = u1 - coupling z_loc (feti.cpp:542-555), interior and boundary slabs
__global__ void k_elim_final(SubLayout L, const int* __restrict__ cglob, const double2* __restrict__ z,
                             const double2* __restrict__ cpl_i, const double2* __restrict__ cpl_b,
                             double2* __restrict__ ui, double2* __restrict__ ub) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long ni = (long long)L.S * L.NI, nb = (long long)L.S * L.NB;
  if (gid >= ni + nb) return;
  const bool interior = gid < ni;
  const long long k = interior ? gid : gid - ni;
  const int s = (int)(k / (interior ? L.NI : L.NB));
  const double2* cp = (interior ? cpl_i : cpl_b) + k * L.NC;
  double2 acc = cz();
  for (int c = 0; c < L.NC; ++c) {
    const int cg = cglob[(size_t)s * L.NC + c];
    if (cg >= 0) acc = cfma(cp[c], z[cg], acc);
  }
  double2* u = interior ? ui : ub;
  u[k] = csub(u[k], acc);
}
// d[r] = u_lo - u_hi (gather_jump, feti.cpp:560-569)
__global__ void k_jump(int nl, const int* __restrict__ lo, const int* __restrict__ hi, const double2* __restrict__ ub,
                       double2* __restrict__ d) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nl) d[r] = csub(ub[lo[r]], ub[hi[r]]);
}
// primal assembly (feti.cpp:699-708)
__global__ void k_assemble_x(int n, const int* __restrict__ kind, const int* __restrict__ xa,
                             const int* __restrict__ xb, const double2* __restrict__ ui,
                             const double2* __restrict__ ub, const double2* __restrict__ z, double2* __restrict__ x) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const int k = kind[f];
  double2 v;
  if (k == 0)
    v = ui[xa[f]];
  else if (k == 1)
    v = cadd(cscale(ub[xa[f]], 0.5), cscale(ub[xb[f]], 0.5));
  else
    v = z[xa[f]];
  x[f] = v;
}

// ------------------------------------------------------------------ GMRES (K7)
// Partial Hermitian dots of w against nv basis vectors (+ |w|^2 when with_norm):
// part[i][blk] = sum_{chunk} conj(V_i) w.  w chunk staged in shared memory.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_mdot(int n, int chunk, const double2* __restrict__ V, size_t ldv, int nv, const double2* __restrict__ w,
           int with_norm, double2* __restrict__ part) {
  extern __shared__ double2 w_sh[];
  const int b = blockIdx.x, lo = b * chunk, len = min(chunk, n - lo);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < len; k += blockDim.x) w_sh[k] = w[lo + k];
  __syncthreads();
  const int nout = nv + (with_norm ? 1 : 0);
  for (int i = warp; i < nout; i += WARPS) {
    double2 acc = cz();
    if (i < nv) {
      const double2* v = V + (size_t)i * ldv + lo;
      for (int k = lane; k < len; k += 32) acc = cfma_conj(v[k], w_sh[k], acc);
    } else {
      for (int k = lane; k < len; k += 32) acc.x += cabs2(w_sh[k]);
    }
    acc = warp_sum2(acc);
    if (lane == 0) part[(size_t)i * gridDim.x + b] = acc;
  }
}
// w -= sum_i h_i V_i on the block's chunk, then partial dots again (CGS2 second pass)
// or |w|^2 only (final pass).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_mupdate(int n, int chunk, const double2* __restrict__ V, size_t ldv, int nv, const double2* __restrict__ h,
              double2* __restrict__ w, int dots, double2* __restrict__ part) {
  extern __shared__ double2 w_sh[];
  const int b = blockIdx.x, lo = b * chunk, len = min(chunk, n - lo);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double2 h_sh[1024];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) h_sh[i] = h[i];
  __syncthreads();
  for (int k = threadIdx.x; k < len; k += blockDim.x) {
    double2 acc = w[lo + k];
    for (int i = 0; i < nv; ++i) acc = cfms(h_sh[i], V[(size_t)i * ldv + lo + k], acc);
    w[lo + k] = acc;
    w_sh[k] = acc;
  }
  __syncthreads();
  const int nout = dots ? nv + 1 : 1;
  for (int i = warp; i < nout; i += WARPS) {
    double2 acc = cz();
    if (dots && i < nv) {
      const double2* v = V + (size_t)i * ldv + lo;
      for (int k = lane; k < len; k += 32) acc = cfma_conj(v[k], w_sh[k], acc);
    } else {
      for (int k = lane; k < len; k += 32) acc.x += cabs2(w_sh[k]);
    }
    acc = warp_sum2(acc);
    if (lane == 0) part[(size_t)i * gridDim.x + b] = acc;
  }
}
// out[i] = sum_b part[i][b] (fixed order => deterministic), optional accumulate into acc
__global__ void k_reduce_parts(int nout, int nblk, const double2* __restrict__ part, double2* __restrict__ out) {
  const int i = blockIdx.x;
  const int lane = threadIdx.x;
  double2 acc = cz();
  for (int b = lane; b < nblk; b += 32) acc = cadd(acc, part[(size_t)i * nblk + b]);
  acc = warp_sum2(acc);
  if (lane == 0) out[i] = acc;
}
// y = alpha * x (complex scalar from device memory: y = x / sqrt(re(*nrm2)))
__global__ void k_normalize(int n, const double2* __restrict__ x, const double2* __restrict__ nrm2,
                            double2* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double inv = 1.0 / sqrt(nrm2->x);
  y[k] = cscale(x[k], inv);
}
__global__ void k_scale_copy(int n, const double2* __restrict__ x, double s, double2* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = cscale(x[k], s);
}
// t = sum_i y_i V_i
__global__ void k_combine(int n, const double2* __restrict__ V, size_t ldv, int nv, const double2* __restrict__ y,
                          double2* __restrict__ t) {
  __shared__ double2 y_sh[1024];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) y_sh[i] = y[i];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double2 acc = cz();
  for (int i = 0; i < nv; ++i) acc = cfma(y_sh[i], V[(size_t)i * ldv + k], acc);
  t[k] = acc;
}
// y = a - b ;  y = a + b
__global__ void k_sub(int n, const double2* a, const double2* b, double2* y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = csub(a[k], b[k]);
}
__global__ void k_add_inplace(int n, double2* __restrict__ y, const double2* __restrict__ b) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = cadd(y[k], b[k]);
}
__global__ void k_conj(int n, const double2* x, double2* y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = cconj(x[k]);
}
// block-partial |x|^2 and max|x| (abs) -> part2[blk] = (sum, max)
__global__ void k_norm_max_part(int n, const double2* __restrict__ x, double2* __restrict__ part) {
  __shared__ double ssum[32], smax[32];
  double s = 0.0, m = 0.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const double a2 = cabs2(x[k]);
    s += a2;
    m = fmax(m, sqrt(a2));
  }
  s = warp_sum(s);
  m = warp_max(m);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) ssum[warp] = s, smax[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tm = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ts += ssum[w], tm = fmax(tm, smax[w]);
    part[blockIdx.x] = make_double2(ts, tm);
  }
}
__global__ void k_norm_max_final(int nblk, const double2* __restrict__ part, double2* __restrict__ out) {
  double s = 0.0, m = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 32) s += part[b].x, m = fmax(m, part[b].y);
  s = warp_sum(s);
  m = warp_max(m);
  if (threadIdx.x == 0) *out = make_double2(s, m);
}

// ------------------------------------------------------------------ global operators (K8)
// y = kc K x + mc V x (+ K_c xc) matrix-free over the Q1 elements around each free dof.
// Real or complex vectors (T = double or double2); coefficients complex.
struct MeshLayout {
  int nx, ny, dpn;
};
template <typename T>
__device__ __forceinline__ double2 as_c(T v);
template <>
__device__ __forceinline__ double2 as_c<double>(double v) {
  return make_double2(v, 0.0);
}
template <>
__device__ __forceinline__ double2 as_c<double2>(double2 v) {
  return v;
}
template <typename T>
__device__ __forceinline__ void store_c(T* p, double2 v);
template <>
__device__ __forceinline__ void store_c<double>(double* p, double2 v) {
  *p = v.x;
}
template <>
__device__ __forceinline__ void store_c<double2>(double2* p, double2 v) {
  *p = v;
}
template <typename T>
__global__ void k_apply_global(MeshLayout M, int n, const int* __restrict__ free_dofs, const int* __restrict__ free_map,
                               const int* __restrict__ cons_map, const T* __restrict__ x, const double* __restrict__ xc,
                               double2 kc, double2 mc, T* __restrict__ y) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const int dpn = M.dpn, ed = 4 * dpn;
  const int md = free_dofs[f];
  const int node = md / dpn, comp = md % dpn;
  const int i = node % (M.nx + 1), j = node / (M.nx + 1);
  double2 acc = cz();
  for (int ej = j - 1; ej <= j; ++ej) {
    if (ej < 0 || ej >= M.ny) continue;
    for (int ei = i - 1; ei <= i; ++ei) {
      if (ei < 0 || ei >= M.nx) continue;
      const int en[4] = {ej * (M.nx + 1) + ei, ej * (M.nx + 1) + ei + 1, (ej + 1) * (M.nx + 1) + ei + 1,
                         (ej + 1) * (M.nx + 1) + ei};
      int alpha = 0;
      for (int q = 0; q < 4; ++q)
        if (en[q] == node) alpha = q;
      const int ra = dpn * alpha + comp;
      for (int b = 0; b < 4; ++b)
        for (int cb = 0; cb < dpn; ++cb) {
          const int mdb = en[b] * dpn + cb;
          const double kv = c_Ke[ra * ed + dpn * b + cb], mv = c_Me[ra * ed + dpn * b + cb];
          const int fb = free_map[mdb];
          if (fb >= 0) {
            const double2 xv = as_c<T>(x[fb]);
            const double2 coef = make_double2(kc.x * kv + mc.x * mv, kc.y * kv + mc.y * mv);
            acc = cfma(coef, xv, acc);
          } else if (xc != nullptr) {
            const int cb2 = cons_map[mdb];
            acc = cfma(make_double2(kv, 0.0), make_double2(xc[cb2], 0.0), acc);
          }
        }
    }
  }
  store_c<T>(y + f, acc);
}

// Kronecker mass solve V^-1 = (M_y ⊗ M_x ⊗ I_dpn)^-1 with pre-factored 1-D tridiagonal
// Thomas coefficients (SPD, no pivoting).  Pass along x (lines = rows), then along y.
// cp[i] = c'_i, dinv[i] = 1 / (b_i - a_i c'_{i-1}); off-diagonals are the constant 'off'.
__global__ void k_tridiag_x(int nlines, int len, int dpn, const double* __restrict__ cp,
                            const double* __restrict__ dinv, double off, double* __restrict__ v) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nlines * dpn) return;
  const int line = t / dpn, comp = t % dpn;
  double* p = v + (size_t)line * len * dpn + comp;
  double prev = 0.0;
  for (int i = 0; i < len; ++i) {
    const double d = (p[(size_t)i * dpn] - off * prev) * dinv[i];
    p[(size_t)i * dpn] = d;
    prev = d;
  }
  for (int i = len - 2; i >= 0; --i) p[(size_t)i * dpn] -= cp[i] * p[(size_t)(i + 1) * dpn];
}
__global__ void k_tridiag_y(int nlines_y, int stride, const double* __restrict__ cp, const double* __restrict__ dinv,
                            double off, double* __restrict__ v, int len) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // t indexes (x position, comp)
  if (t >= stride) return;
  double prev = 0.0;
  for (int j = 0; j < len; ++j) {
    const double d = (v[(size_t)j * stride + t] - off * prev) * dinv[j];
    v[(size_t)j * stride + t] = d;
    prev = d;
  }
  for (int j = len - 2; j >= 0; --j) v[(size_t)j * stride + t] -= cp[j] * v[(size_t)(j + 1) * stride + t];
  (void)nlines_y;
}
// y = ybar - v ; u = lam / phi ; lam = Re t ; leak partial
__global__ void k_realify(int n, const double2* __restrict__ t, double* __restrict__ lam) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) lam[k] = t[k].x;
}
__global__ void k_recover_yu(int n, const double* __restrict__ ybar, const double* __restrict__ vk,
                             const double* __restrict__ lam, double inv_phi, double* __restrict__ y,
                             double* __restrict__ u) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  y[k] = ybar[k] - vk[k];
  u[k] = lam[k] * inv_phi;
}
__global__ void k_real_to_complex(int n, const double* __restrict__ x, double2* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = make_double2(x[k], 0.0);
}
// max |Im t| partials
__global__ void k_imag_max_part(int n, const double2* __restrict__ t, double* __restrict__ part) {
  __shared__ double sm[32];
  double m = 0.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) m = fmax(m, fabs(t[k].y));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t2 = fmax(t2, sm[w]);
    part[blockIdx.x] = t2;
  }
}

}  // namespace fetigpu
