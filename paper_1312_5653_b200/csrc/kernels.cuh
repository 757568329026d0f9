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

// Element matrices travel by value in the kernel parameter space (constant bank), so
// several contexts (different meshes / phi, or emulated ranks) can coexist in a process.
struct ElemAe {
  double2 v[MAX_EDOFS * MAX_EDOFS];  // Ae = kc*Ke + mc*Me (feti.cpp:264-265)
};
struct ElemKM {
  double k[MAX_EDOFS * MAX_EDOFS], m[MAX_EDOFS * MAX_EDOFS];
};

struct SubLayout {
  int S, nld, ex, ey, dpn, NI, NB, NC, W, EBI, EIB;
};

// ------------------------------------------------------------------ K1 block assembly
// One thread per (subdomain, local mesh dof a).  The thread owns row a of every block it
// belongs to, visits the <= 4 elements around its node in ascending element id (the
// reference's sub.elements order, feti.cpp:305) and accumulates deterministically.
__global__ void k_assemble(SubLayout L, ElemAe Ae, const int* __restrict__ ldof, double2* __restrict__ colband,
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
          const double2 v = Ae.v[ra * ed + dpn * b + cb];
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

// S_bb^-1 of every subdomain by the symmetric sweep operator, the whole packed lower
// triangle resident in shared memory (n(n+1)/2 complex: 124 KB at n = 124).  S_bb is
// complex symmetric (A = A^T; real part SPD), so Gauss-Jordan without pivoting keeps the
// symmetric form when row and column k are both scaled by 1/d:
//   d = a_kk;  a_ij -= a_ik a_kj / d (i, j != k);  a_ik = a_ik / d;  a_kk = -1/d
// and sweeping every k yields -A^-1 (Goodnight 1979).  Reads S (dense [S][n][n]), writes the
// dense symmetric inverse; status[s] = 1-based index of a zero / non-finite pivot.
__global__ void __launch_bounds__(256) k_sym_sweep_inverse(const double2* __restrict__ S, double2* __restrict__ Sinv,
                                                           int n, int* __restrict__ status) {
  extern __shared__ double2 sw_sh[];
  double2* a = sw_sh;                               // packed lower: (i, j <= i) at i(i+1)/2 + j
  double2* col = sw_sh + (size_t)n * (n + 1) / 2;   // column k of the current step
  __shared__ double2 dinv_sh;
  const int s = blockIdx.x, tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;           // 8 row groups x 32 columns
  const double2* M = S + (size_t)s * n * n;
  for (int i = ty; i < n; i += 8)
    for (int j = tx; j <= i; j += 32) a[i * (i + 1) / 2 + j] = M[(size_t)i * n + j];
  int bad = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    for (int i = tid; i < n; i += 256) col[i] = i >= k ? a[i * (i + 1) / 2 + k] : a[k * (k + 1) / 2 + i];
    __syncthreads();
    const double2 d = col[k];
    if (tid == 0) {
      const double a2 = cabs2(d);
      if (bad == 0 && (!(a2 > 0.0) || !isfinite(a2))) bad = k + 1;
      dinv_sh = crecip(d);
    }
    __syncthreads();
    const double2 dinv = dinv_sh;
    for (int i = ty; i < n; i += 8) {
      const double2 ci = col[i];
      const double2 cid = cmul(ci, dinv);
      for (int j = tx; j <= i; j += 32) {
        double2& e = a[i * (i + 1) / 2 + j];
        if (i == k && j == k) e = make_double2(-dinv.x, -dinv.y);
        else if (i == k) e = cmul(col[j], dinv);
        else if (j == k) e = cid;
        else e = cfms(cid, col[j], e);
      }
    }
    __syncthreads();
  }
  double2* O = Sinv + (size_t)s * n * n;  // A^-1 = -(swept matrix)
  for (int i = ty; i < n; i += 8)
    for (int j = tx; j <= i; j += 32) {
      const double2 v = a[i * (i + 1) / 2 + j];
      const double2 m = make_double2(-v.x, -v.y);
      O[(size_t)i * n + j] = m;
      O[(size_t)j * n + i] = m;
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
  for (int c0 = 0; c0 < L.NC; c0 += 8) {  // columns in chunks of 8
    const int nc = min(8, L.NC - c0);
    double2 acc[8];
    for (int c = 0; c < nc; ++c) acc[c] = Yc[((size_t)s * L.NC + c0 + c) * L.NI + i];
    for (int b = 0; b < L.NB; ++b) {
      const double2 y = Y[((size_t)s * L.NB + b) * L.NI + i];
      for (int c = 0; c < nc; ++c) acc[c] = cfms(y, cpl_b[((size_t)s * L.NB + b) * L.NC + c0 + c], acc[c]);
    }
    for (int c = 0; c < nc; ++c) cpl_i[((size_t)s * L.NI + i) * L.NC + c0 + c] = acc[c];
  }
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

// ---- dense coarse path (edge-RBM augmentation: the coarse matrix is indefinite and not
// banded in corner order).  Assembly, equilibration and an in-place Gauss-Jordan inverse
// with partial pivoting (the pivot sequence of the reference's PartialPivLU, feti.cpp:468).
__global__ void k_coarse_assemble_dense(int nc, int NC, const int* __restrict__ slots, const int* __restrict__ cglob,
                                        const double2* __restrict__ Acc, const double2* __restrict__ contrib,
                                        double2* __restrict__ C) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nc) return;
  for (int q = 0; q < 4; ++q) {
    const int slot = slots[r * 4 + q];
    if (slot < 0) continue;
    const int s = slot / NC, ka = slot % NC;
    for (int kb = 0; kb < NC; ++kb) {
      const int col = cglob[(size_t)s * NC + kb];
      if (col >= 0) C[(size_t)r * nc + col] = cadd(C[(size_t)r * nc + col], Acc[((size_t)s * NC + ka) * NC + kb]);
    }
    for (int kb = 0; kb < NC; ++kb) {
      const int col = cglob[(size_t)s * NC + kb];
      if (col >= 0) C[(size_t)r * nc + col] = csub(C[(size_t)r * nc + col], contrib[((size_t)s * NC + ka) * NC + kb]);
    }
  }
}
__global__ void k_dense_diag_scale(int nc, const double2* __restrict__ C, double* __restrict__ scale) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const double d = sqrt(cabs2(C[(size_t)i * nc + i]));
  scale[i] = d > 0.0 ? 1.0 / sqrt(d) : 1.0;
}
__global__ void k_dense_apply_scale(int nc, double2* __restrict__ C, const double* __restrict__ scale) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)nc * nc) return;
  C[e] = cscale(C[e], scale[e / nc] * scale[e % nc]);
}
// Gauss-Jordan step k, part 1 (one block): pivot row p = argmax_{i>=k} |A(i,k)| (smallest
// index on ties), swap rows k and p, scale row k by 1/A(k,k) (A(k,k) <- 1/A(k,k)), stash
// column k for the update.  pivabs[k] = |pivot| (the reference's U_kk check).
__global__ void __launch_bounds__(1024) k_gj_pivot(int n, int k, double2* __restrict__ A, int* __restrict__ piv,
                                                   double* __restrict__ pivabs, double2* __restrict__ fcol) {
  __shared__ double wb[32];
  __shared__ int wi[32];
  __shared__ int p_sh;
  __shared__ double2 dinv_sh;
  double best = -1.0;
  int bidx = n;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double a = cabs2(A[(size_t)i * n + k]);
    if (a > best) best = a, bidx = i;
  }
  for (int m = 16; m > 0; m >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, m);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, m);
    if (ob > best || (ob == best && oi < bidx)) best = ob, bidx = oi;
  }
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = best, wi[threadIdx.x >> 5] = bidx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = -1.0;
    int bi = n;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      if (wb[w] > b || (wb[w] == b && wi[w] < bi)) b = wb[w], bi = wi[w];
    p_sh = bi < n ? bi : k;
    piv[k] = p_sh;
  }
  __syncthreads();
  const int p = p_sh;
  if (p != k)
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double2 t = A[(size_t)k * n + j];
      A[(size_t)k * n + j] = A[(size_t)p * n + j];
      A[(size_t)p * n + j] = t;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double2 d = A[(size_t)k * n + k];
    pivabs[k] = sqrt(cabs2(d));
    dinv_sh = crecip(d);
  }
  __syncthreads();
  const double2 dinv = dinv_sh;
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    A[(size_t)k * n + j] = j == k ? dinv : cmul(A[(size_t)k * n + j], dinv);
  for (int i = threadIdx.x; i < n; i += blockDim.x) fcol[i] = i == k ? cz() : A[(size_t)i * n + k];
}
// part 2: rows i != k: A(i,j) -= f_i A(k,j) (j != k), A(i,k) = -f_i / pivot
__global__ void k_gj_update(int n, int k, double2* __restrict__ A, const double2* __restrict__ fcol) {
  const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || i == k) return;
  const double2 f = fcol[i], pk = A[(size_t)k * n + j];
  double2& a = A[(size_t)i * n + j];
  a = j == k ? make_double2(-(f.x * pk.x - f.y * pk.y), -(f.x * pk.y + f.y * pk.x)) : cfms(f, pk, a);
}
// undo the row interchanges as column interchanges, last pivot first (one thread per row)
__global__ void k_gj_unpermute(int n, double2* __restrict__ A, const int* __restrict__ piv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2* row = A + (size_t)i * n;
  for (int k = n - 1; k >= 0; --k) {
    const int p = piv[k];
    if (p != k) {
      const double2 t = row[k];
      row[k] = row[p];
      row[p] = t;
    }
  }
}
// signed C^s^T entries of the augmentation columns into the A_bc-like coupling rhs
__global__ void k_add_aug(int cnt, int NB, int NC, const int* __restrict__ s_, const int* __restrict__ kb,
                          const int* __restrict__ kc, const double* __restrict__ val, double2* __restrict__ Abc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cnt) return;
  double2& t = Abc[((size_t)s_[e] * NB + kb[e]) * NC + kc[e]];
  t.x += val[e];
}
// v -= Q Q^T v edge by edge (feti.cpp:572-578): one warp per edge, its columns in order
// (plane strain: tx, ty, rot — rot overlaps one translation), edges are disjoint.
__global__ void k_project_aug(int n_edges, const int* __restrict__ edge_col0, const int* __restrict__ edge_ncol,
                              const int* __restrict__ col_ptr, const int* __restrict__ rows,
                              const double* __restrict__ vals, double2* __restrict__ v) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (e >= n_edges) return;
  for (int c = edge_col0[e]; c < edge_col0[e] + edge_ncol[e]; ++c) {
    double2 coef = cz();
    for (int q = col_ptr[c] + lane; q < col_ptr[c + 1]; q += 32) coef = cadd(coef, cscale(v[rows[q]], vals[q]));
    coef = warp_sum2(coef);
    __syncwarp();
    for (int q = col_ptr[c] + lane; q < col_ptr[c + 1]; q += 32) v[rows[q]] = csub(v[rows[q]], cscale(coef, vals[q]));
    __syncwarp();
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
// selected columns of the identity (X[r n + rows[r]] = 1, X zeroed) and the matching
// rescale X[r][j] *= scale[rows[r]] scale[j]: rows `rows` of the equilibrated C^-1
__global__ void k_select_identity(int nr, int n, const int* __restrict__ rows, double2* __restrict__ X) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nr) X[(size_t)r * n + rows[r]] = make_double2(1.0, 0.0);
}
__global__ void k_scale_inverse_rows(int nr, int n, const int* __restrict__ rows, double2* __restrict__ X,
                                     const double* __restrict__ scale) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)nr * n) return;
  X[gid] = cscale(X[gid], scale[rows[gid / n]] * scale[gid % n]);
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
               double2* __restrict__ out_b, const double2* __restrict__ cpl_b, double2* __restrict__ gcp,
               const int* __restrict__ jsel = nullptr, size_t jstride = 0) {
  extern __shared__ double2 in_sh[];
  const int s = blockIdx.x;
  if (jsel != nullptr) lam += (size_t)(*jsel) * jstride;  // GMRES basis column V_j
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

// ------------------------------------------------------------------ packed symmetric GEMV
// S_bb and S_bb^-1 are complex symmetric (A_rr = A_rr^T).  They are stored as the lower
// triangle of 32x32 tiles (NT = ceil(NB/32) tiles per dimension), "diagonal-major":
//   off-diagonal tile (I, J), J < I :  O[c][l] = M[32I + l][32J + (l+c) mod 32],  c = 0..31
//   diagonal tile (I, I)             :  D[c][l] = M[32I + l][32I + (l+c) mod 32],  c = 0..16
// so at step c lane l streams entry (l, l+c): coalesced 512 B per warp-load, the row
// product accumulates in the lane, and the transposed product is carried in a register
// rotated by one lane per step (no per-row reductions).  Bytes per subdomain:
// NT*17*512 + NT(NT-1)/2*16384 (133 KB at NB = 124 vs 246 KB dense).
__host__ __device__ constexpr int sym_tile_entries(int NT) { return NT * 17 * 32 + NT * (NT - 1) / 2 * 1024; }

// ---- sharded path: cut-line halo of per-dof slot values -------------
// buf[i * width + c] = val[slots[i] * width + c]
__global__ void k_pack_slots(int n, int width, const int* __restrict__ slots, const double2* __restrict__ val,
                             double2* __restrict__ buf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * width) return;
  const int i = t / width, c = t % width;
  buf[t] = val[(size_t)slots[i] * width + c];
}
// val[slots[i] * width + c] = buf[i * width + c]
__global__ void k_unpack_slots(int n, int width, const int* __restrict__ slots, const double2* __restrict__ buf,
                               double2* __restrict__ val) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * width) return;
  const int i = t / width, c = t % width;
  val[(size_t)slots[i] * width + c] = buf[t];
}

// pack[s] <- full[s] (row-major NB x NB); entries outside NB are zero
__global__ void k_pack_sym(int S, int NB, int NT, const double2* __restrict__ full, double2* __restrict__ pack) {
  const int per = sym_tile_entries(NT);
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)S * per) return;
  const int s = (int)(gid / per);
  int e = (int)(gid % per);
  int r, c;
  const int ndiag = NT * 17 * 32;
  if (e < ndiag) {
    const int I = e / (17 * 32);
    e %= 17 * 32;
    const int cc = e / 32, l = e % 32;
    r = 32 * I + l;
    c = 32 * I + ((l + cc) & 31);
  } else {
    e -= ndiag;
    const int t = e / 1024;
    e %= 1024;
    int I = 1;
    while ((I + 1) * I / 2 <= t) ++I;
    const int J = t - I * (I - 1) / 2;
    const int cc = e / 32, l = e % 32;
    r = 32 * I + l;
    c = 32 * J + ((l + cc) & 31);
  }
  pack[gid] = (r < NB && c < NB) ? full[((size_t)s * NB + r) * NB + c] : cz();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// optional kernel-span instrumentation (FETIGPU_STEP_TIMES=1): span[(it * 3 + kid) * 2 + {0,1}]
// = earliest CTA start / latest CTA end of kernel kid (0 precond, 1 dual, 2 tail) of Arnoldi
// step `it` (read from the GMRES state)
__device__ __forceinline__ void span_mark(unsigned long long* span, const int* it_ptr, int kid, int end) {
  if (span == nullptr || threadIdx.x != 0) return;
  unsigned long long* p = span + ((size_t)(*it_ptr) * 3 + kid) * 2 + end;
  if (end) atomicMax(p, gtimer());
  else atomicMin(p, gtimer());
}

__global__ void k_span_init(int count, unsigned long long* span) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) span[i] = (i & 1) ? 0ULL : ~0ULL;
}

struct SymGemvArgs {
  int NB, NT, NC, NI, EBI;
  const double2* pack;  // [S][sym_tile_entries(NT)]
  // inputs
  int mode;                       // 0: in = alpha sign lam[blam]; 1: in = alpha sign (wb_lo - wb_hi)/2; 2: in = tb - A_bi yi
  const int* blam;
  const double* bsign;
  const double2* lam;
  const int* jsel;                // mode 0: lam += (*jsel) * jstride (GMRES basis column)
  size_t jstride;
  double2* zout;                  // mode 1, optional: zout[(*jsel) jstride + r] = (wb_lo - wb_hi)/2
                                  // (the preconditioned basis column Z_j = M^-1 V_j, written
                                  // by the CTA owning the row's +1 slot)
  double alpha;
  const int* lam_lo;
  const int* lam_hi;
  const double2* wb;
  const double2* tb;
  const int* bi_idx;
  const double2* bi_val;
  const double2* yi;
  // outputs
  double2* out;                   // [S][NB]
  const double2* cpl_b;           // optional: gcp = cpl_b^T in
  double2* gcp;
  // optional, with gcp: the last CTA assembles the coarse rhs g = fc - sum gcp (feti.cpp:523-538)
  unsigned int* g_counter;
  int nc;
  const int* corner_slots;
  const double2* fc;
  double2* g;
  unsigned long long* span;  // FETIGPU_STEP_TIMES (Arnoldi-step GEMVs only)
  const int* it_ptr;
  // unrolled WHILE body: a step after the cycle stopped (cont == 0) returns at once
  const int* cont_ptr;
  // MODE 2 coarse rhs: the nonzeros of A_ic per (subdomain, corner), AE per corner
  int AE;
  const int* aic_idx;
  const double2* aic_val;
};


// The per-subdomain packed symmetric GEMV (one CTA = one subdomain), shared by k_sym_gemv
// and k_sym_gemv_giv (the preconditioner GEMV with the previous step's Givens folded in).
// Solve-constant index operands of the input-vector gather (B^T scatter) of entry
// k = threadIdx.x, loaded BEFORE griddepcontrol.wait so that only the data-dependent loads
// (one round trip) remain after it: multiplier row, its sign, and (mode 1) the row's two slots.
// Used by k_sym_gemv_aside (+0.4 % there; no gain in the plain GEMVs, whose CTAs only become
// resident when the producer kernel's CTAs exit, and their register budget is full).
struct SymPre {
  int r, lo, hi;
  double sg;
};
template <int MODE>
__device__ __forceinline__ SymPre sym_pre_load(const SymGemvArgs& a, int s) {
  SymPre p{-1, 0, 0, 0.0};
  const int k = threadIdx.x;
  if (MODE != 2 && k < a.NB) {
    const size_t sb = (size_t)s * a.NB + k;
    p.r = a.blam[sb];
    p.sg = a.bsign[sb];
    if (MODE == 1 && p.r >= 0) {
      p.lo = a.lam_lo[p.r];
      p.hi = a.lam_hi[p.r];
    }
  }
  return p;
}
// EARLY (dual GEMV of the Arnoldi step with the coarse solve beside it, k_sym_gemv_aside):
// gcp = cpl_b^T x is formed right after the input vector -- from coupling entries `cp` the
// warp loaded before griddepcontrol.wait (warp c = local corner c, lane l = rows l + 32 q) --
// and stored at once (plain stores over the all-ones sentinel the tail left there: the value
// is its own ready flag, no fence stalls the warp), so the coarse CTAs of the same launch can
// start while this CTA streams its operator.  Same summation order as the epilogue form.
template <int MODE, int SYM_BATCH, int WARPS, bool EARLY = false>
__device__ __forceinline__ void sym_gemv_run(const SymGemvArgs& a, const SymPre* pre = nullptr,
                                             const double2* cp = nullptr) {
  // dynamic smem: x (32 NT) | row partials (ntiles x 32) | column partials (noff x 32)
  extern __shared__ double2 sg_sh[];
  const int NB = a.NB, NT = a.NT;
  const int noff = NT * (NT - 1) / 2, ntiles = noff + NT;
  double2* x_sh = sg_sh;
  double2 (*part_row)[32] = reinterpret_cast<double2 (*)[32]>(sg_sh + 32 * NT);
  double2 (*part_col)[32] = reinterpret_cast<double2 (*)[32]>(sg_sh + 32 * NT + 32 * ntiles);
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  span_mark(a.span, a.it_ptr, MODE, 0);
  // ---- input vector (B^T scatter) ----
  const double2* lam = a.lam;
  if (MODE == 0 && a.jsel != nullptr) lam += (size_t)(*a.jsel) * a.jstride;
  for (int k = threadIdx.x; k < 32 * NT; k += blockDim.x) {
    double2 v = cz();
    if (k < NB) {
      const size_t sb = (size_t)s * NB + k;
      if (MODE == 2) {
        v = a.tb[sb];
        for (int e = 0; e < a.EBI; ++e) {
          const int i = a.bi_idx[sb * a.EBI + e];
          if (i >= 0) v = cfms(a.bi_val[sb * a.EBI + e], a.yi[(size_t)s * a.NI + i], v);
        }
      } else {
        int r, lo = 0, hi = 0;
        double sg;
        if (pre != nullptr && k == (int)threadIdx.x) {
          r = pre->r;
          lo = pre->lo;
          hi = pre->hi;
          sg = pre->sg;
        } else {
          r = a.blam[sb];
          sg = a.bsign[sb];
          if (MODE == 1 && r >= 0) {
            lo = a.lam_lo[r];
            hi = a.lam_hi[r];
          }
        }
        if (r >= 0) {
          double2 z;
          if (MODE == 0)
            z = lam[r];
          else {
            z = cscale(csub(a.wb[lo], a.wb[hi]), 0.5);
            if (a.zout != nullptr && lo == (int)sb) a.zout[(size_t)(*a.jsel) * a.jstride + r] = z;
          }
          v = cscale(z, a.alpha * sg);
        }
      }
    }
    x_sh[k] = v;
  }
  __syncthreads();
  if (EARLY) {
    if (warp < a.NC) {
      double2 acc = cz();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < NB) acc = cfma(cp[q], x_sh[lane + 32 * q], acc);
      acc = warp_sum2(acc);
      if (lane == 0) __stcg(a.gcp + (size_t)s * a.NC + warp, acc);
    }
  }
  // ---- tiles: off-diagonal first (t < noff), then diagonal.  A diagonal tile streams half
  // the bytes of an off-diagonal one, so two diagonal tiles form one work item
  // (NT = 4, 8 warps: one item each; 4 warps: two items each).
  const double2* P = a.pack + (size_t)s * sym_tile_entries(NT);
  const bool paired = true;
  for (int item = warp; item < (paired ? noff + (NT + 1) / 2 : ntiles); item += WARPS)
  for (int half = 0; half < ((paired && item >= noff) ? 2 : 1); ++half) {
    const int t = (paired && item >= noff) ? noff + 2 * (item - noff) + half : item;
    if (t >= ntiles) break;
    double2 yr = cz(), yc = cz();
    if (t < noff) {
      int I = 1;
      while ((I + 1) * I / 2 <= t) ++I;
      const int J = t - I * (I - 1) / 2;
      const double2* O = P + NT * 17 * 32 + (size_t)t * 1024;
      const double2 xi = x_sh[32 * I + lane];
      // explicit SYM_BATCH-row load batches: all loads of a batch are in flight together
#pragma unroll
      for (int cb = 0; cb < 32; cb += SYM_BATCH) {
        double2 m[SYM_BATCH];
#pragma unroll
        for (int u = 0; u < SYM_BATCH; ++u) m[u] = __ldcs(O + (cb + u) * 32 + lane);
#pragma unroll
        for (int u = 0; u < SYM_BATCH; ++u) {
          const int c = cb + u;
          yr = cfma(m[u], x_sh[32 * J + ((lane + c) & 31)], yr);
          yc = cfma(m[u], xi, yc);
          yc = shfl2(yc, (lane + 1) & 31);  // carry column (l+c+1) into lane l
        }
      }
      // after 32 rotations lane l holds column l
      part_row[t][lane] = yr;
      part_col[t][lane] = yc;
    } else {
      const int I = t - noff;
      const double2* D = P + (size_t)I * 17 * 32;
      const double2 xi = x_sh[32 * I + lane];
#pragma unroll
      for (int cb = 0; cb < 16; cb += SYM_BATCH) {
        double2 m[SYM_BATCH];
#pragma unroll
        for (int u = 0; u < SYM_BATCH; ++u) m[u] = __ldcs(D + (cb + u) * 32 + lane);
#pragma unroll
        for (int u = 0; u < SYM_BATCH; ++u) {
          const int c = cb + u;
          if (c == 0) {
            yr = cmul(m[u], xi);  // diagonal entry
          } else {  // c = 1..15: row + transposed; carry for the transposed part as above
            yr = cfma(m[u], x_sh[32 * I + ((lane + c) & 31)], yr);
            yc = shfl2(yc, (lane + 1) & 31);
            yc = cfma(m[u], xi, yc);
          }
        }
      }
      // yc in lane l now holds column (l + 15); c = 16 covers both (l, l+16) and (l+16, l)
      {
        const double2 m = __ldcs(D + 16 * 32 + lane);
        yr = cfma(m, x_sh[32 * I + ((lane + 16) & 31)], yr);
      }
      yc = shfl2(yc, (lane + 17) & 31);  // lane l <- column l
      part_row[t][lane] = cadd(yr, yc);
    }
  }
  __syncthreads();
  // ---- deterministic combination: y_I = sum_J<I rows(I,J) + diag(I) + sum_{I'>I} cols(I',I) ----
  for (int k = threadIdx.x; k < NB; k += blockDim.x) {
    const int I = k >> 5, l = k & 31;
    double2 acc = part_row[noff + I][l];
    for (int J = 0; J < I; ++J) acc = cadd(acc, part_row[I * (I - 1) / 2 + J][l]);
    for (int I2 = I + 1; I2 < NT; ++I2) acc = cadd(acc, part_col[I2 * (I2 - 1) / 2 + I][l]);
    a.out[(size_t)s * NB + k] = acc;
  }
  if (!EARLY && a.gcp != nullptr) {
    for (int c = warp; c < a.NC; c += WARPS) {
      double2 acc = cz();
      for (int k = lane; k < NB; k += 32) acc = cfma(a.cpl_b[((size_t)s * NB + k) * a.NC + c], x_sh[k], acc);
      // eliminate (MODE 2): coupling^T t = cpl_b^T (t_b - A_bi y_i) + A_ic^T y_i
      if (MODE == 2 && a.aic_idx != nullptr && lane < a.AE) {
        const size_t e = ((size_t)s * a.NC + c) * a.AE + lane;
        const int i = a.aic_idx[e];
        if (i >= 0) acc = cfma(a.aic_val[e], a.yi[(size_t)s * a.NI + i], acc);
      }
      acc = warp_sum2(acc);
      if (lane == 0) a.gcp[(size_t)s * a.NC + c] = acc;
    }
    if (a.g_counter != nullptr) {
      __shared__ bool is_last;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) is_last = atomicAdd(a.g_counter, 1u) == gridDim.x - 1;
      __syncthreads();
      if (is_last) {
        __threadfence();
        for (int c = threadIdx.x; c < a.nc; c += blockDim.x) {
          double2 acc = a.fc ? a.fc[c] : cz();
          for (int q = 0; q < 4; ++q) {
            const int slot = a.corner_slots[c * 4 + q];
            if (slot >= 0) acc = csub(acc, __ldcg(a.gcp + slot));
          }
          a.g[c] = acc;
        }
        if (threadIdx.x == 0) *a.g_counter = 0u;
      }
    }
  }
  if (a.span != nullptr) {
    __syncthreads();
    span_mark(a.span, a.it_ptr, MODE, 1);
  }
}

template <int MODE, int SYM_BATCH, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, (WARPS == 8 ? 4 : 8)) k_sym_gemv(SymGemvArgs a) {
  pdl_trigger();
#ifndef FETIGPU_GEMV_PF_ROWS
#define FETIGPU_GEMV_PF_ROWS 8
#endif
#ifndef FETIGPU_GEMV_PF_MODES
#define FETIGPU_GEMV_PF_MODES 3
#endif
#ifndef FETIGPU_GEMV_PF_ROWS_ASIDE
#define FETIGPU_GEMV_PF_ROWS_ASIDE 8
#endif
  if ((FETIGPU_GEMV_PF_MODES >> MODE) & 1) {
    // the operator is solve-constant: warm L1 with the first rows of this warp's first
    // off-diagonal tile while the producer kernel drains (CTAs that become resident early)
    const int NT = a.NT, noff = NT * (NT - 1) / 2, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < noff) {
      const double2* O = a.pack + (size_t)blockIdx.x * sym_tile_entries(NT) + NT * 17 * 32 + (size_t)warp * 1024;
#pragma unroll
      for (int u = 0; u < FETIGPU_GEMV_PF_ROWS; ++u) prefetch_l1(O + u * 32 + lane);
    }
  }
  pdl_wait();
  if (a.cont_ptr != nullptr && *a.cont_ptr == 0) return;
  sym_gemv_run<MODE, SYM_BATCH, WARPS>(a);
}

// debugging aid (FETIGPU_WATCHDOG): progress marker between graph body kernels
__global__ void k_mark(unsigned int* progress, unsigned int v) {
  if (threadIdx.x == 0) atomicExch(progress, v);
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
                             const double2* __restrict__ fc, double2* __restrict__ g,
                             const int* __restrict__ cont_ptr = nullptr) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  if (cont_ptr != nullptr && *cont_ptr == 0) return;  // a step after the cycle stopped
  double2 acc = fc ? fc[c] : cz();
  for (int q = 0; q < 4; ++q) {
    const int slot = corner_slots[c * 4 + q];
    if (slot >= 0) acc = csub(acc, gcp[slot]);
  }
  g[c] = acc;
}

// z = C^-1 g  (dense explicit coarse inverse, K4), one row per block of THREADS threads
// (rows != nullptr, sharded: Cinv holds only the rows C^-1[rows[b], :] and z is written at
// rows[b]):
// each thread takes a strided set of columns (a few loads, all independent), then a block
// reduction in fixed order.  Latency-bound kernel (C^-1 stays in L2), so the parallelism
// comes from the number of warps, not from per-thread batching (ptxas serialises those).
template <int THREADS>
__global__ void __launch_bounds__(THREADS)
    k_coarse_gemv(int nc, const double2* __restrict__ Cinv, const double2* __restrict__ g, double2* __restrict__ z,
                  const int* __restrict__ rows = nullptr, const int* __restrict__ cont_ptr = nullptr) {
  constexpr int WARPS = THREADS / 32;
  __shared__ double2 red[WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  pdl_wait();
  if (cont_ptr != nullptr && *cont_ptr == 0) return;  // a step after the cycle stopped
  const int row = blockIdx.x;
  const double2* cr = Cinv + (size_t)row * nc;
  double2 a = cz();
  for (int k = threadIdx.x; k < nc; k += THREADS) a = cfma(__ldg(cr + k), __ldg(g + k), a);
  a = warp_sum2(a);
  if (lane == 0) red[warp] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = red[0];
#pragma unroll
    for (int q = 1; q < WARPS; ++q) t = cadd(t, red[q]);
    z[rows != nullptr ? rows[row] : row] = t;
  }
}

// ---- large coarse spaces: z = C^-1 g with C^-1 complex symmetric, packed in the 32 x 32
// tile format of k_pack_sym (4 diagonal tiles' 17 rows + lower off-diagonal tiles): half the
// bytes of the dense row-major GEMV.  Kernel 1: one warp per tile (row and transposed
// partials, as k_sym_gemv); kernel 2: fixed-order combination per 32-row block.
__global__ void __launch_bounds__(128) k_big_sym_gemv(int nc, int NT, const double2* __restrict__ pack,
                                                      const double2* __restrict__ x, double2* __restrict__ part_row,
                                                      double2* __restrict__ part_col,
                                                      const int* __restrict__ cont_ptr = nullptr) {
  __shared__ double2 xs[4][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int noff = NT * (NT - 1) / 2, items = noff + NT;
  const int t = blockIdx.x * 4 + warp;
  pdl_trigger();
  pdl_wait();
  if (cont_ptr != nullptr && *cont_ptr == 0) return;  // a step after the cycle stopped
  if (t >= items) return;
  double2* xI = xs[warp][0];
  double2* xJ = xs[warp][1];
  if (t < noff) {
    int I = 1;
    while ((I + 1) * I / 2 <= t) ++I;
    const int J = t - I * (I - 1) / 2;
    xI[lane] = 32 * I + lane < nc ? x[32 * I + lane] : cz();
    xJ[lane] = 32 * J + lane < nc ? x[32 * J + lane] : cz();
    __syncwarp();
    const double2* O = pack + (size_t)NT * 17 * 32 + (size_t)t * 1024;
    const double2 xi = xI[lane];
    double2 yr = cz(), yc = cz();
#pragma unroll
    for (int cb = 0; cb < 32; cb += 8) {
      double2 m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m[u] = __ldcs(O + (cb + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = cb + u;
        yr = cfma(m[u], xJ[(lane + c) & 31], yr);
        yc = cfma(m[u], xi, yc);
        yc = shfl2(yc, (lane + 1) & 31);
      }
    }
    part_row[(size_t)t * 32 + lane] = yr;
    part_col[(size_t)t * 32 + lane] = yc;
  } else {
    const int I = t - noff;
    xI[lane] = 32 * I + lane < nc ? x[32 * I + lane] : cz();
    __syncwarp();
    const double2* D = pack + (size_t)I * 17 * 32;
    const double2 xi = xI[lane];
    double2 yr = cz(), yc = cz();
#pragma unroll
    for (int cb = 0; cb < 16; cb += 8) {
      double2 m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m[u] = __ldcs(D + (cb + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = cb + u;
        if (c == 0) {
          yr = cmul(m[u], xi);
        } else {
          yr = cfma(m[u], xI[(lane + c) & 31], yr);
          yc = shfl2(yc, (lane + 1) & 31);
          yc = cfma(m[u], xi, yc);
        }
      }
    }
    yr = cfma(__ldcs(D + 16 * 32 + lane), xI[(lane + 16) & 31], yr);
    yc = shfl2(yc, (lane + 17) & 31);
    part_row[(size_t)t * 32 + lane] = cadd(yr, yc);
  }
}
// y_I = diag(I) + sum_{J<I} rows(I,J) + sum_{I'>I} cols(I',I): one CTA per row block I, 8
// warps over the partial tiles (fixed assignment and order), then the 8 sums in order
__global__ void __launch_bounds__(256) k_big_sym_reduce(int nc, int NT, const double2* __restrict__ part_row,
                                                        const double2* __restrict__ part_col, double2* __restrict__ z,
                                                        const int* __restrict__ cont_ptr = nullptr) {
  __shared__ double2 red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, I = blockIdx.x;
  const int noff = NT * (NT - 1) / 2;
  pdl_trigger();
  pdl_wait();
  if (cont_ptr != nullptr && *cont_ptr == 0) return;  // a step after the cycle stopped
  double2 acc = cz();
  for (int J = warp; J < I; J += 8) acc = cadd(acc, part_row[((size_t)I * (I - 1) / 2 + J) * 32 + lane]);
  for (int I2 = I + 1 + warp; I2 < NT; I2 += 8) acc = cadd(acc, part_col[((size_t)I2 * (I2 - 1) / 2 + I) * 32 + lane]);
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    double2 t = part_row[((size_t)noff + I) * 32 + lane];
#pragma unroll
    for (int q = 0; q < 8; ++q) t = cadd(t, red[q][lane]);
    if (32 * I + lane < nc) z[32 * I + lane] = t;
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

// u1_b = S_bb^-1 (t_b - A_bi y_i); one CTA per subdomain
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
// gcp[s][c] = (A_rc^T A_rr^-1 t)_c = sum_i cpl_i(i,c) t_i + sum_k cpl_b(k,c) t_b   (feti.cpp:530;
// equal to A_rc^T u1 because A_rr^-1 is symmetric).  One CTA per subdomain.
// Nonzeros of A_ic column-wise per (subdomain, corner): the sparse term A_ic^T y_i of the
// eliminate-phase coarse rhs.  status[0] = 1 if a column has more than AE nonzeros.
__global__ void k_compact_aic(SubLayout L, int AE, const double2* __restrict__ Aic, int* __restrict__ idx,
                              double2* __restrict__ val, int* __restrict__ status) {
  const int sc = blockIdx.x * blockDim.x + threadIdx.x;
  if (sc >= L.S * L.NC) return;
  const int s = sc / L.NC, c = sc % L.NC;
  int e = 0;
  for (int i = 0; i < L.NI; ++i) {
    const double2 v = Aic[((size_t)s * L.NI + i) * L.NC + c];
    if (v.x != 0.0 || v.y != 0.0) {
      if (e < AE) {
        idx[(size_t)sc * AE + e] = i;
        val[(size_t)sc * AE + e] = v;
      }
      ++e;
    }
  }
  if (e > AE) atomicExch(status, 1);
  for (; e < AE; ++e) {
    idx[(size_t)sc * AE + e] = -1;
    val[(size_t)sc * AE + e] = cz();
  }
}

// Compact table of the coupled interior rows (an A_ib entry or a nonzero A_ic entry), built
// on the device in three passes with a fixed order (ascending row): per-1024-row block
// counts, one block scanning the counts, then the per-block local scan + row copy.
__device__ __forceinline__ bool ri_coupled(size_t g, int E, int NC, const int* __restrict__ idx,
                                           const double2* __restrict__ aic) {
  bool any = false;
  for (int e = 0; e < E; ++e) any = any || idx[g * E + e] >= 0;
  for (int c = 0; c < NC; ++c) any = any || aic[g * NC + c].x != 0.0 || aic[g * NC + c].y != 0.0;
  return any;
}
__global__ void __launch_bounds__(1024) k_ri_count(long long rows, int E, int NC, const int* __restrict__ idx,
                                                   const double2* __restrict__ aic, int* __restrict__ bcount) {
  __shared__ int wsum[32];
  const long long g = (long long)blockIdx.x * 1024 + threadIdx.x;
  const int f = g < rows && ri_coupled((size_t)g, E, NC, idx, aic) ? 1 : 0;
  const int c = __popc(__ballot_sync(0xffffffffu, f));
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = wsum[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) bcount[blockIdx.x] = v;
  }
}
// exclusive scan of nb block counts (one block, sequential over chunks of 1024); total at [nb]
__global__ void __launch_bounds__(1024) k_ri_scan(int nb, int* __restrict__ bcount) {
  __shared__ int sh[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? bcount[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
      const int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nb) bcount[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) bcount[nb] = carry;
}
__global__ void __launch_bounds__(1024) k_ri_compact(long long rows, int E, int NC, const int* __restrict__ idx,
                                                     const double2* __restrict__ val, const double2* __restrict__ aic,
                                                     const int* __restrict__ boff, int* __restrict__ map,
                                                     int* __restrict__ cidx, double2* __restrict__ cval,
                                                     double2* __restrict__ caic) {
  __shared__ int wsum[32];
  const long long g = (long long)blockIdx.x * 1024 + threadIdx.x;
  const int f = g < rows && ri_coupled((size_t)g, E, NC, idx, aic) ? 1 : 0;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 32 warp counts
    const int v = wsum[lane];
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    wsum[lane] = x - v;
  }
  __syncthreads();
  if (g >= rows) return;
  if (!f) {
    map[g] = -1;
    return;
  }
  const int q = boff[blockIdx.x] + wsum[warp] + __popc(bal & ((1u << lane) - 1u));
  map[g] = q;
  for (int e = 0; e < E; ++e) {
    cidx[(size_t)q * E + e] = idx[(size_t)g * E + e];
    cval[(size_t)q * E + e] = val[(size_t)g * E + e];
  }
  for (int c = 0; c < NC; ++c) caic[(size_t)q * NC + c] = aic[(size_t)g * NC + c];
}

__global__ void k_gcp_full(SubLayout L, const double2* __restrict__ cpl_i, const double2* __restrict__ cpl_b,
                           const double2* __restrict__ ti, const double2* __restrict__ tb, double2* __restrict__ gcp) {
  __shared__ double2 red[8][32];
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = cz();
  for (int i = threadIdx.x; i < L.NI; i += blockDim.x) {
    const size_t si = (size_t)s * L.NI + i;
    const double2 t = ti[si];
    for (int c = 0; c < L.NC; ++c) acc[c] = cfma(cpl_i[si * L.NC + c], t, acc[c]);
  }
  for (int k = threadIdx.x; k < L.NB; k += blockDim.x) {
    const size_t sb = (size_t)s * L.NB + k;
    const double2 t = tb[sb];
    for (int c = 0; c < L.NC; ++c) acc[c] = cfma(cpl_b[sb * L.NC + c], t, acc[c]);
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
// u_b = u1_b - cpl_b z_loc  (feti.cpp:542-555, boundary rows)
// u_b = (u1_b [+ add]) - cpl_b z   (feti.cpp:542-548; `add`: the first elimination's part of u1_b
// when the final elimination is assembled by linearity)
__global__ void k_ub_correct(SubLayout L, const int* __restrict__ cglob, const double2* __restrict__ z,
                             const double2* __restrict__ cpl_b, double2* __restrict__ ub,
                             const double2* __restrict__ add = nullptr) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (long long)L.S * L.NB) return;
  const int s = (int)(k / L.NB);
  double2 acc = cz();
  for (int c = 0; c < L.NC; ++c) {
    const int cg = cglob[(size_t)s * L.NC + c];
    if (cg >= 0) acc = cfma(cpl_b[k * L.NC + c], z[cg], acc);
  }
  const double2 u = add != nullptr ? cadd(ub[k], add[k]) : ub[k];
  ub[k] = csub(u, acc);
}
// r_i = A_ib u_b + A_ic z_loc  (rhs of the interior harmonic extension)
__global__ void k_ri_rhs(SubLayout L, const int* __restrict__ ib_idx, const double2* __restrict__ ib_val,
                         const double2* __restrict__ Aic, const int* __restrict__ cglob, const double2* __restrict__ z,
                         const double2* __restrict__ ub, double2* __restrict__ ri) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)L.S * L.NI) return;
  const int s = (int)(gid / L.NI);
  double2 acc = cz();
  for (int e = 0; e < L.EIB; ++e) {
    const int b = ib_idx[gid * L.EIB + e];
    if (b >= 0) acc = cfma(ib_val[gid * L.EIB + e], ub[(size_t)s * L.NB + b], acc);
  }
  for (int c = 0; c < L.NC; ++c) {
    const int cg = cglob[(size_t)s * L.NC + c];
    if (cg >= 0) acc = cfma(Aic[gid * L.NC + c], z[cg], acc);
  }
  ri[gid] = acc;
}
// same on the compacted coupled rows: map[gid] = row of the compact tables or -1 (no
// interface / corner coupling: r_i = 0, ~87 % of the interior rows at config 2)
__global__ void k_ri_rhs_compact(long long cnt, int EIB, int NC, int NI, int NB, const int* __restrict__ map,
                                 const int* __restrict__ cidx, const double2* __restrict__ cval,
                                 const double2* __restrict__ caic, const int* __restrict__ cglob,
                                 const double2* __restrict__ z, const double2* __restrict__ ub,
                                 double2* __restrict__ ri) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= cnt) return;
  const int q = map[gid];
  double2 acc = cz();
  if (q >= 0) {
    const int s = (int)(gid / NI);
    for (int e = 0; e < EIB; ++e) {
      const int b = cidx[(size_t)q * EIB + e];
      if (b >= 0) acc = cfma(cval[(size_t)q * EIB + e], ub[(size_t)s * NB + b], acc);
    }
    for (int c = 0; c < NC; ++c) {
      const int cg = cglob[(size_t)s * NC + c];
      if (cg >= 0) acc = cfma(caic[(size_t)q * NC + c], z[cg], acc);
    }
  }
  ri[gid] = acc;
}
// u_i = y_i - A_ii^-1 r_i   (r_i already solved in place)
__global__ void k_ui_final(long long cnt, const double2* __restrict__ yi, double2* __restrict__ ri) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < cnt) ri[k] = csub(yi[k], ri[k]);
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
                             const double2* __restrict__ ub, const double2* __restrict__ z, double2* __restrict__ x,
                             const double2* __restrict__ yi = nullptr) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const int k = kind[f];
  if (k < 0) return;  // owned by another rank (sharded path)
  double2 v;
  if (k == 0)  // yi given: ui holds A_ii^-1 r_i and u_i = y_i - A_ii^-1 r_i is formed here
    v = yi != nullptr ? csub(yi[xa[f]], ui[xa[f]]) : ui[xa[f]];
  else if (k == 1)
    v = cadd(cscale(ub[xa[f]], 0.5), cscale(ub[xb[f]], 0.5));
  else
    v = z[xa[f]];
  x[f] = v;
}

// ------------------------------------------------------------------ GMRES (K7)
// Device-resident Arnoldi state.  One Arnoldi step (krylov.hpp:150-188) is a fixed kernel
// sequence that reads j from here, so it can run eagerly or inside a CUDA-graph
// conditional WHILE node with no host round trip per step.
struct GmresState {
  int j;           // current column
  int iterations;  // Arnoldi steps so far (SolveStats::iterations)
  int k;           // columns completed this cycle
  int cont;        // 1 while the cycle continues
  int status;      // 1 = NaN/Inf breakdown (krylov.hpp:165-166)
  int max_iter;
  int m;           // restart length (= max_iter: unrestarted, feti.cpp:684)
  int jcol;        // basis column of the next preconditioner GEMV (split-Givens graph path)
  double tol, bnorm, inv_hnext, est;
};

// Hessenberg column update, Givens rotations and both stopping tests of one Arnoldi
// step (krylov.hpp:164-188), run by one warp.  R is the rotated Hessenberg, packed by
// columns (column j at R + j(j+1)/2).  The rotation operands are staged in shared
// memory and the sequential rotation chain runs on lane 0.  In graph mode it drives the
// WHILE node.  h1 = [V^H w0, |w0|^2], h2 = [V^H w1, |w1|^2] (CGS2 passes).
struct GivensArgs {
  GmresState* st;
  const double2* h1;
  const double2* h2;
  double2* R;
  double* gcos;
  double2* gsin;
  double2* g;
  int in_graph;
  cudaGraphConditionalHandle handle;
};
template <bool SMEM>
__device__ __forceinline__ double2 ldh(const double2* p) {
  if constexpr (SMEM) return *p;
  else return __ldcg(p);
}
// hnext = |w1 - V h2| = sqrt(|w1|^2 - sum_{i<=j} |h2_i|^2) (V orthonormal; h2 round-off sized)
// and the finiteness of h1 + h2, one warp; every caller gets bit-identical results.
template <bool SMEM>
__device__ __forceinline__ double warp_hnext(const double2* h1, const double2* h2, int j, bool& finite) {
  const int lane = threadIdx.x & 31;
  bool fin = true;
  double s2 = 0.0;
  for (int i = lane; i <= j; i += 32) {
    const double2 h2i = ldh<SMEM>(h2 + i);
    const double2 v = cadd(ldh<SMEM>(h1 + i), h2i);
    fin = fin && isfinite(v.x) && isfinite(v.y);
    s2 += cabs2(h2i);
  }
  fin = __all_sync(0xffffffffu, fin);
  s2 = warp_sum(s2);
  const double hnext = sqrt(fmax(0.0, ldh<SMEM>(h2 + j + 1).x - s2));
  finite = fin && isfinite(hnext);
  return hnext;
}
// Operands of a Givens step that are known before the Arnoldi step's reductions (the fused
// tail loads them at its start, off the critical path): the state scalars, g_j and, when
// j <= 256, the previous rotations already staged in sc / ss.
struct GivensPre {
  int j, iterations, max_iter, m;
  double tol, bnorm;
  double2 gj;
  int staged;
};
// block 0, warp 0 of the fused tail: fill GivensPre and the rotation staging
__device__ __forceinline__ void givens_prefetch(const GivensArgs& a, GivensPre* pre, double* sc, double2* ss) {
  const int lane = threadIdx.x & 31;
  const GmresState* st = a.st;
  const int j = st->j;
  const bool staged = j <= 256;
  if (staged)
    for (int q = lane; q < j; q += 32) {
      sc[q] = a.gcos[q];
      ss[q] = a.gsin[q];
    }
  if (lane == 0) {
    pre->j = j;
    pre->iterations = st->iterations;
    pre->max_iter = st->max_iter;
    pre->m = st->m;
    pre->tol = st->tol;
    pre->bnorm = st->bnorm;
    pre->gj = a.g[j];
    pre->staged = staged ? 1 : 0;
  }
}
template <bool SMEM = false>
__device__ void givens_warp(const GivensArgs& a, double* sc, double2* ss, double2* sh, const double2* h1 = nullptr,
                            const double2* h2 = nullptr, const GivensPre* pre = nullptr) {
  constexpr int CHK = 256;
  const int lane = threadIdx.x & 31;
  if (h1 == nullptr) h1 = a.h1;
  if (h2 == nullptr) h2 = a.h2;
  GmresState* st = a.st;
  const int j = pre ? pre->j : st->j;
  double2* col = a.R + (size_t)j * (j + 1) / 2;
  bool finite;
  const double hnext = warp_hnext<SMEM>(h1, h2, j, finite);
  const double wpre = sqrt(ldh<SMEM>(h1 + j + 1).x);
  if (!finite) {
    if (lane == 0) {
      st->status = 1;
      st->cont = 0;
      if (a.in_graph) cudaGraphSetConditional(a.handle, 0u);
    }
    return;
  }
  // previous rotations (krylov.hpp:169-173): carry = rotated entry i, t2 = original entry i+1
  double2 carry = cadd(ldh<SMEM>(h1), ldh<SMEM>(h2));
  for (int base = 0; base < j; base += CHK) {
    const int cnt = min(CHK, j - base);
    const bool have = pre != nullptr && pre->staged;  // (staged only when j <= CHK)
    for (int q = lane; q < cnt; q += 32) {
      if (!have) {
        sc[q] = a.gcos[base + q];
        ss[q] = a.gsin[base + q];
      }
      sh[q] = cadd(ldh<SMEM>(h1 + base + q + 1), ldh<SMEM>(h2 + base + q + 1));
    }
    __syncwarp();
    if (lane == 0) {
      for (int q = 0; q < cnt; ++q) {
        const double c = sc[q];
        const double2 s = ss[q], t1 = carry, t2 = sh[q];
        col[base + q] = cfma(s, t2, cscale(t1, c));
        carry = cfms(cconj(s), t1, cscale(t2, c));
      }
    }
    __syncwarp();
  }
  if (lane != 0) return;
  // make_givens (krylov.hpp:66-83) on (carry = rotated col[j], hnext)
  const double2 x = carry;
  const double a1 = sqrt(cabs2(x)), a2 = hnext;
  double c;
  double2 s;
  if (a2 == 0.0) {
    c = 1.0;
    s = cz();
  } else if (a1 == 0.0) {
    c = 0.0;
    s = make_double2(1.0, 0.0);
  } else {
    const double t = hypot(a1, a2);
    c = a1 / t;
    s = cscale(make_double2(x.x / a1, x.y / a1), a2 / t);  // (h1/|h1|) conj(h2)/t, h2 real
  }
  a.gcos[j] = c;
  a.gsin[j] = s;
  col[j] = cfma(s, make_double2(hnext, 0.0), cscale(x, c));
  const double2 gj = pre ? pre->gj : a.g[j];
  const double2 gj1 = cmul(make_double2(-s.x, s.y), gj);  // -conj(s) g_j
  a.g[j + 1] = gj1;
  a.g[j] = cscale(gj, c);
  const int iters = (pre ? pre->iterations : st->iterations) + 1;
  st->iterations = iters;
  st->k = j + 1;
  const double est = sqrt(cabs2(gj1));
  st->est = est;
  const bool happy = hnext <= 1e-14 * fmax(wpre, 1e-300);
  const double tol = pre ? pre->tol : st->tol, bnorm = pre ? pre->bnorm : st->bnorm;
  const int max_iter = pre ? pre->max_iter : st->max_iter, m = pre ? pre->m : st->m;
  const int cont = !(happy || est <= tol * bnorm) && iters < max_iter && (j + 1) < m;
  if (cont) {
    st->inv_hnext = 1.0 / hnext;
    st->j = j + 1;
  }
  st->cont = cont;
  if (a.in_graph) cudaGraphSetConditional(a.handle, cont ? 1u : 0u);
}

__global__ void __launch_bounds__(32) k_givens(GivensArgs a) {
  __shared__ double sc[256];
  __shared__ double2 ss[256], sh[256];
  if (a.st->cont == 0) return;  // a step launched past the end of the cycle (sharded loop)
  givens_warp(a, sc, ss, sh);
}
// split-Givens graph path: the Givens step of the last step of an unrolled body, skipped
// once the cycle stopped (the tail of that step returned at once and published nothing)
__global__ void __launch_bounds__(32) k_givens_step(GivensArgs a) {
  __shared__ double sc[256];
  __shared__ double2 ss[256], sh[256];
  pdl_trigger();
  pdl_wait();  // (launched with programmatic serialization after the tail)
  if (a.st->cont == 0) {
    if (a.in_graph && threadIdx.x == 0) cudaGraphSetConditional(a.handle, 0u);
    return;
  }
  givens_warp(a, sc, ss, sh);
}
// Preconditioner GEMV of Arnoldi step j+1 with the Givens step of step j folded in as one
// extra CTA (blockIdx.x == gridDim.x - 1): the rotation chain runs concurrently with the
// operator stream instead of ending the previous tail on the critical path.  The GEMV CTAs
// take their basis column from st->jcol (published by the tail) and may run once past the
// end of a stopped cycle (harmless: the dual GEMV and tail of that step return at once).
template <int SYM_BATCH, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, (WARPS == 8 ? 4 : 8)) k_sym_gemv_giv(SymGemvArgs a, GivensArgs ga) {
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x == gridDim.x - 1) {
    extern __shared__ double2 sg_sh[];  // >= 640 entries (host)
    if (threadIdx.x < 32) {
      if (ga.st->cont == 0) {
        if (ga.in_graph && threadIdx.x == 0) cudaGraphSetConditional(ga.handle, 0u);
      } else {
        givens_warp(ga, reinterpret_cast<double*>(sg_sh), sg_sh + 128, sg_sh + 384);
      }
    }
    return;
  }
  if (a.cont_ptr != nullptr && *a.cont_ptr == 0) return;
  sym_gemv_run<0, SYM_BATCH, WARPS>(a);
}

// One classical Gram-Schmidt pass on the block's chunk of w:
//   w chunk = fused dual-operator tail (gather) or loaded; optional w -= sum_i h_in[i] V_i;
//   partial sums of conj(V_i) w and/or |w|^2, reduced by the last block to finish (fixed
//   order => deterministic); optionally the last block then runs the Givens step.
// nv = st->j + 1.  mode 0: dots + norm (out[0..nv]) ; 1: dots ; 2: norm only.
struct CgsArgs {
  int n, chunk, mode;
  const double2* V;
  size_t ldv;
  GmresState* st;
  const double2* h_in;
  double2* w;
  double2* part;
  double2* out;
  unsigned int* counter;
  // fused dual tail (feti.cpp:542-555, 593): w[r] = -((u1_lo - cpl z)_lo - (u1_hi - cpl z)_hi)
  int gather;
  int NB, NC;
  const int *lam_lo, *lam_hi, *cglob;
  const double2 *u1b, *cpl_b, *z;
  // fused Givens (pass 2)
  int givens;
  GivensArgs ga;
};
// sum_{lo <= i < hi} h[i] V_i[r], loads issued in batches of 8 (fixed summation order)
__device__ __forceinline__ double2 sum_vh(const double2* __restrict__ h, const double2* __restrict__ V, size_t ldv,
                                          int r, int lo, int hi) {
  constexpr int VB = 8;
  double2 acc = cz();
  int i = lo;
  for (; i + VB <= hi; i += VB) {
    double2 v[VB];
#pragma unroll
    for (int u = 0; u < VB; ++u) v[u] = V[(size_t)(i + u) * ldv + r];
#pragma unroll
    for (int u = 0; u < VB; ++u) acc = cfma(__ldg(h + i + u), v[u], acc);
  }
  for (; i < hi; ++i) acc = cfma(__ldg(h + i), V[(size_t)i * ldv + r], acc);
  return acc;
}

// w[r] = -(u_lo - u_hi), u_slot = u1_b[slot] - cpl_b[slot] z_loc: the dual-operator tail of
// multiplier row r (feti.cpp:542-555, 593).  z_l2: read z through L2 (written in this kernel).
template <typename A>
__device__ __forceinline__ double2 dual_tail_row(const A& a, int r, bool z_l2) {
  const int slots[2] = {a.lam_lo[r], a.lam_hi[r]};
  double2 u[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int slot = slots[q], s = slot / a.NB;
    double2 cz_ = cz();
    for (int c = 0; c < a.NC; ++c) {
      const int cg = a.cglob[(size_t)s * a.NC + c];
      if (cg >= 0) cz_ = cfma(a.cpl_b[(size_t)slot * a.NC + c], z_l2 ? __ldcg(a.z + cg) : a.z[cg], cz_);
    }
    u[q] = csub(a.u1b[slot], cz_);
  }
  const double2 d = csub(u[0], u[1]);
  return make_double2(-d.x, -d.y);
}

// One classical Gram-Schmidt pass over ROWS multiplier rows per block (THREADS / ROWS
// thread groups):
//   phase A  w[r] = fused dual-operator tail (gather) or loaded; optional w -= sum_i h_in[i] V_i
//            (each group sums a contiguous range of basis vectors, combined in fixed order);
//   phase B  one warp per basis vector: block partials of conj(V_i) w over the block's rows
//            (and |w|^2), so each lane keeps ROWS/32 independent loads in flight;
//   the last block reduces the partials in a fixed order (deterministic) and optionally runs
//   the Givens step.  nv = st->j + 1.  mode 0: dots + norm (out[0..nv]); 1: dots; 2: norm.
template <int THREADS, int ROWS>
__global__ void __launch_bounds__(THREADS) k_cgs_pass(CgsArgs a) {
  constexpr int WARPS = THREADS / 32, GROUPS = THREADS / ROWS, LPR = ROWS / 32;
  static_assert(THREADS % ROWS == 0 && ROWS % 32 == 0, "block shape");
  __shared__ double2 w_sh[ROWS];
  __shared__ double2 acc_sh[GROUPS][ROWS];
  __shared__ double2 stage[640];  // Givens staging (cos 256 doubles | sin 256 | h 256)
  __shared__ bool is_last;
  pdl_trigger();
  pdl_wait();
  const int nv = a.st->j + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = threadIdx.x % ROWS, grp = threadIdx.x / ROWS;
  const int row0 = blockIdx.x * ROWS, r = row0 + lr;
  const bool act = r < a.n;
  if (a.h_in != nullptr) {
    const int per = (nv + GROUPS - 1) / GROUPS;
    const int lo = min(nv, grp * per), hi = min(nv, lo + per);
    acc_sh[grp][lr] = act ? sum_vh(a.h_in, a.V, a.ldv, r, lo, hi) : cz();
    __syncthreads();
  }
  if (grp == 0) {
    double2 w = cz();
    if (act) {
      if (a.gather) {
        w = dual_tail_row(a, r, false);
      } else {
        w = a.w[r];
      }
      if (a.h_in != nullptr) {
#pragma unroll
        for (int g = 0; g < GROUPS; ++g) w = csub(w, acc_sh[g][lr]);
      }
      if (a.gather || a.h_in != nullptr) a.w[r] = w;
    }
    w_sh[lr] = w;
  }
  __syncthreads();
  const int ndots = (a.mode == 2) ? 0 : nv;
  const int nout = ndots + (a.mode == 1 ? 0 : 1);
  for (int i = warp; i < nout; i += WARPS) {
    double2 acc = cz();
    if (i < ndots) {
      const double2* v = a.V + (size_t)i * a.ldv + row0;
      double2 x[LPR];
      // clamped addresses keep the loads unpredicated (all in flight); w_sh is 0 past n
#pragma unroll
      for (int u = 0; u < LPR; ++u) x[u] = v[min(lane + 32 * u, a.n - 1 - row0)];
#pragma unroll
      for (int u = 0; u < LPR; ++u) acc = cfma_conj(x[u], w_sh[lane + 32 * u], acc);
    } else {
#pragma unroll
      for (int u = 0; u < LPR; ++u) acc.x += cabs2(w_sh[lane + 32 * u]);
    }
    acc = warp_sum2(acc);
    if (lane == 0) a.part[(size_t)i * gridDim.x + blockIdx.x] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // grid reduction: SEGS threads per output, strided over the block partials, then shuffles
  constexpr int SEGS = 16, PER = THREADS / SEGS;
  const int G = gridDim.x, seg = threadIdx.x % SEGS;
  for (int i0 = 0; i0 < nout; i0 += PER) {
    const int i = i0 + threadIdx.x / SEGS;
    double2 t = cz();
    if (i < nout) {
      const double2* pp = a.part + (size_t)i * G;
#pragma unroll 8
      for (int bb = seg; bb < G; bb += SEGS) t = cadd(t, __ldcg(pp + bb));
    }
#pragma unroll
    for (int m = SEGS / 2; m > 0; m >>= 1) t = cadd(t, shfl_xor2(t, m));
    if (seg == 0 && i < nout) a.out[i] = t;
  }
  if (threadIdx.x == 0) *a.counter = 0u;
  if (a.givens) {
    __threadfence_block();
    __syncthreads();
    if (warp == 0) givens_warp(a.ga, reinterpret_cast<double*>(stage), stage + 128, stage + 384);
  }
}

// Augmented Arnoldi step, scalar physics (one column per edge, rows = the edge's multiplier
// rows): w = P F z in one pass, one warp per edge — the dual-operator tail gathered per row
// (dual_tail_row), the edge coefficient q^T w reduced in the warp, w -= coef q, stored.
struct EdgeGatherArgs {
  int n_edges, NB, NC;
  const int *col_ptr, *col_rows;
  const double* col_vals;
  const int *lam_lo, *lam_hi, *cglob;
  const double2 *u1b, *cpl_b, *z;
  double2* w;
  const int* cont_ptr;  // graph-captured step: a launch after the cycle stopped returns at once
};
__global__ void k_gather_project_edges(EdgeGatherArgs a) {
  constexpr int MAXR = 4;  // up to 128 rows per edge
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (e >= a.n_edges) return;
  if (a.cont_ptr != nullptr && *a.cont_ptr == 0) return;
  const int q0 = a.col_ptr[e], len = a.col_ptr[e + 1] - q0;
  double2 w[MAXR];
  double qv[MAXR];
  double2 coef = cz();
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    const int k = lane + 32 * t;
    w[t] = cz();
    qv[t] = 0.0;
    if (k < len) {
      qv[t] = a.col_vals[q0 + k];
      w[t] = dual_tail_row(a, a.col_rows[q0 + k], false);
      coef = cadd(coef, cscale(w[t], qv[t]));
    }
  }
  coef = warp_sum2(coef);
#pragma unroll
  for (int t = 0; t < MAXR; ++t) {
    const int k = lane + 32 * t;
    if (k < len) a.w[a.col_rows[q0 + k]] = csub(w[t], cscale(coef, qv[t]));
  }
}

// Row-block x vector-group combination: ROWS rows per block, GROUPS thread groups each
// summing a contiguous range of the nv basis vectors (all loads of a group in flight at
// once), combined in fixed order by group 0.  Returns true on group-0 threads of live rows.
template <int ROWS, int GROUPS>
__device__ __forceinline__ bool combine_rows(const double2* __restrict__ h, const double2* __restrict__ V, size_t ldv,
                                             int n, int nv, int& r, double2& sum) {
  __shared__ double2 acc_sh[GROUPS][ROWS];
  const int lr = threadIdx.x % ROWS, grp = threadIdx.x / ROWS;
  r = blockIdx.x * ROWS + lr;
  const int per = (nv + GROUPS - 1) / GROUPS;
  const int lo = min(nv, grp * per), hi = min(nv, lo + per);
  acc_sh[grp][lr] = r < n ? sum_vh(h, V, ldv, r, lo, hi) : cz();
  __syncthreads();
  if (grp != 0 || r >= n) return false;
  sum = acc_sh[0][lr];
#pragma unroll
  for (int g = 1; g < GROUPS; ++g) sum = cadd(sum, acc_sh[g][lr]);
  return true;
}

// V_{j+1} = (w - V h2) / h_{j+1,j}: the second CGS update fused with the normalisation
// (only while the cycle continues; st->j already advanced, so V_0..V_{j-1} are read).
template <int ROWS, int GROUPS>
__global__ void __launch_bounds__(ROWS* GROUPS)
    k_update_normalize(int n, const GmresState* __restrict__ st, const double2* __restrict__ h2,
                       const double2* __restrict__ w, double2* __restrict__ V, size_t ldv) {
  pdl_trigger();
  pdl_wait();
  if (!st->cont) return;
  const int nv = st->j;
  int r;
  double2 sum;
  if (combine_rows<ROWS, GROUPS>(h2, V, ldv, n, nv, r, sum))
    V[(size_t)nv * ldv + r] = cscale(csub(w[r], sum), st->inv_hnext);
}

// y = R^-1 g (krylov.hpp:191-196), one warp.  When the packed triangle fits (k <= BS_KMAX)
// it is staged in shared memory first (all loads in flight; static 48 KB cap), so the k-row recurrence runs
// on shared-memory latencies instead of one global round trip per row.
constexpr int BS_KMAX = 72;
__global__ void __launch_bounds__(32) k_backsub(const GmresState* __restrict__ st, const double2* __restrict__ R,
                                                const double2* __restrict__ g, double2* __restrict__ y) {
  __shared__ double2 rs[BS_KMAX * (BS_KMAX + 1) / 2];
  __shared__ double2 ys[BS_KMAX], gs[BS_KMAX];
  const int k = st->k, lane = threadIdx.x;
  if (k <= BS_KMAX) {
    const int tot = k * (k + 1) / 2;
    for (int e = lane; e < tot; e += 32) rs[e] = R[e];
    for (int e = lane; e < k; e += 32) gs[e] = g[e];  // (no global load inside the recurrence)
    __syncwarp();
    for (int i = k - 1; i >= 0; --i) {
      double2 acc = cz();
      for (int j2 = i + 1 + lane; j2 < k; j2 += 32) acc = cfma(rs[j2 * (j2 + 1) / 2 + i], ys[j2], acc);
      acc = warp_sum2(acc);
      if (lane == 0) ys[i] = cmul(csub(gs[i], acc), crecip(rs[i * (i + 1) / 2 + i]));
      __syncwarp();
    }
    for (int i = lane; i < k; i += 32) y[i] = ys[i];
    return;
  }
  for (int i = k - 1; i >= 0; --i) {
    double2 acc = cz();
    for (int j2 = i + 1 + lane; j2 < k; j2 += 32) acc = cfma(R[(size_t)j2 * (j2 + 1) / 2 + i], y[j2], acc);
    acc = warp_sum2(acc);
    if (lane == 0) {
      const double2 num = csub(g[i], acc);
      y[i] = cmul(num, crecip(R[(size_t)i * (i + 1) / 2 + i]));
    }
    __syncwarp();
  }
}

// first GMRES cycle without a host round trip: |b| from the statistics slot (sum of squares)
__global__ void k_scale_by_norm(int n, const double2* __restrict__ x, const double2* __restrict__ nrm2,
                                double2* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const double s2 = nrm2->x;
  if (k < n) y[k] = s2 > 0.0 ? cscale(x[k], 1.0 / sqrt(s2)) : cz();
}
// Start of a device-driven first GMRES cycle in ONE launch: x = 0, r = b, best iterate = 0,
// V_0 = b / |b| (|b|^2 in *nrm2, the expression of k_scale_by_norm), the cycle state (init with
// bnorm and cont from |b|, as k_gmres_init), g_0 = |b|, and -- with the coarse solve beside the
// dual GEMV -- its done-counter cleared and the coarse partials at the all-ones sentinel.
__global__ void k_gmres_start(int n, const double2* __restrict__ b, const double2* __restrict__ nrm2,
                              double2* __restrict__ x, double2* __restrict__ r, double2* __restrict__ best,
                              double2* __restrict__ V0, GmresState init, GmresState* __restrict__ st,
                              double2* __restrict__ g, double2* __restrict__ gcp, int n_gcp,
                              unsigned int* __restrict__ aside_ctr) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const double s2 = nrm2->x;
  if (k < n) {
    const double2 bb = b[k];
    x[k] = cz();
    best[k] = cz();
    r[k] = bb;
    V0[k] = s2 > 0.0 ? cscale(bb, 1.0 / sqrt(s2)) : cz();
  }
  if (gcp != nullptr && k < n_gcp) {
    const double ones = __longlong_as_double(-1LL);
    gcp[k] = make_double2(ones, ones);
  }
  if (k == 0) {
    const double bn = sqrt(s2);
    init.bnorm = bn;
    init.cont = bn > 0.0 ? 1 : 0;  // zero rhs: the (fused) step kernels all return at once
    *st = init;
    g[0] = make_double2(bn, 0.0);
    if (aside_ctr != nullptr) aside_ctr[0] = aside_ctr[1] = 0u;
  }
}
__global__ void k_gmres_init(GmresState* __restrict__ st, const double2* __restrict__ nrm2, double2* __restrict__ g) {
  if (threadIdx.x != 0) return;
  const double bn = sqrt(nrm2->x);
  st->bnorm = bn;
  st->cont = bn > 0.0 ? 1 : 0;  // zero rhs: the (fused) step kernels all return at once
  g[0] = make_double2(bn, 0.0);
}
__global__ void k_scale_copy(int n, const double2* __restrict__ x, double s, double2* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = cscale(x[k], s);
}
// t = sum_i y_i V_i
template <int ROWS, int GROUPS>
__global__ void __launch_bounds__(ROWS* GROUPS) k_combine(int n, const double2* __restrict__ V, size_t ldv,
                                                          const GmresState* __restrict__ st,
                                                          const double2* __restrict__ y, double2* __restrict__ t) {
  int r;
  double2 sum;
  if (combine_rows<ROWS, GROUPS>(y, V, ldv, n, st->k, r, sum)) t[r] = sum;
}
// ---------------------------------------------------------------------------------------
// Fused Arnoldi tail (one GPU): coarse solve z = C^-1 g (unless it ran beside the dual GEMV:
// ASIDE), CGS pass 1 (dual-operator tail gathered per row, h1 = V^H w, |w|^2), CGS pass 2
// (w -= V h1, h2 = V^H w, |w|^2), Givens and V_{j+1} = (w - V h2) / h_{j+1,j}, in ONE launch.
// The data dependences are grid barriers (grid_sync_plain) after which every block reduces
// the block partials in block order (deterministic, identical in all blocks).  Each thread
// keeps its multiplier row(s) of w in registers across the phases and re-reads its V rows from
// L1.  All blocks are co-resident by construction (cooperative launch, probed at setup); a
// barrier that does not complete within ~2 s traps instead of hanging.
// k_arnoldi_tail: one row per thread; k_arnoldi_tail_mr: up to RPT rows per thread.
struct ArnoldiTailArgs {
  int n;        // multiplier rows
  int rows_pb;  // rows per block (<= THREADS; k_arnoldi_tail_mr: <= THREADS RPT)
  double2* V;
  size_t ldv;
  GmresState* st;
  double2* part;
  double2 *h1, *h2;
  unsigned int* bar;  // [0] arrivals, [1] generation
  int hcap, vcap;  // h staging capacity (>= nv + 1), basis columns allocated
  // coarse
  int nc, coarse_rb;  // rb: coarse rows per block per round (1, 2, 4 or 8)
  const double2* Cinv;
  const double2* gcp;        // per-(subdomain, corner) coarse contributions of the dual GEMV
  const int* corner_slots;   // [nc][4]
  double2* z;
  // dual tail gather
  int NB, NC;
  const int *lam_lo, *lam_hi, *cglob;
  const double2 *u1b, *cpl_b;
  GivensArgs ga;
  // split_givens: the Givens step runs as its own kernel on a side branch of the graph,
  // concurrently with the next preconditioner GEMV; the tail only publishes h1/h2 and the
  // next basis column index (st->jcol)
  int split_givens;
  unsigned long long* tstamp;  // optional phase timestamps (block 0), 8 per Arnoldi step
  unsigned long long* span;    // FETIGPU_STEP_TIMES
  // coarse solve beside the dual GEMV (k_sym_gemv_aside): ctr[1] == aside_nx when z is
  // already there; the tail resets both counters for the next step.  nullptr: off.
  unsigned int* aside_ctr;
  unsigned int aside_nx;
  int n_gcp;                // entries of gcp (n_sub * NC)
  // bulk L2 prefetch of the head of every subdomain's preconditioner operator (the first
  // off-diagonal tile: what the next launch's CTAs stream first): pf_count slices of pf_bytes
  // at pf_base + s pf_stride, issued at the tail's start while HBM is idle.  16 KB per
  // subdomain shortens the next GEMV's ramp by ~2 us; more only slows the tail's own L2 loads.
  const char* pf_base;
  size_t pf_stride;
  unsigned int pf_bytes;
  int pf_count;
  int wg;                   // entries of the w / g staging region: max(THREADS, nc)
  int hcs;                  // dot-vector entries that use shared memory (<= kTailHcs; test hook: smaller)
  double2* hbuf;            // [grid][2][hcap] dot vectors of long cycles (nv + 1 > kTailHcs)
  const double2* w_in;      // k_arnoldi_tail_mr, optional: w already formed (augmented: projected)
  const double2* zpart;     // [nc][aside_nx] partial coarse solutions
  const int* blk_corners;   // [grid][kTailCorners] corners the block's rows touch (-1 pad)
};
constexpr int kTailHcs = 128;      // dot-vector entries kept in shared memory
constexpr int kTailCorners = 128;  // corners a tail block's rows may touch (4 threads each)


__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned int atom_add_release_u32(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------------------
// Dual GEMV of the Arnoldi step with the coarse solve beside it.  The launch is the dual
// GEMV's n_sub CTAs plus 4 ca.ng coarse CTAs (blockIdx >= n_sub), all resident in one wave
// (the host sizes ng from the occupancy of this kernel).  Every GEMV CTA stores its coarse
// partials gcp = cpl_b^T t right after forming its input vector (sym_gemv_run EARLY) over
// the all-ones sentinel the tail left there; a value whose two words both differ from the
// sentinel is complete, so the value is its own ready flag and no fence stalls the GEMV.
// The coarse CTAs work in groups of four: group q owns the corners c in [q cpg, (q+1) cpg),
// each of its CTAs polls the (up to 4) partials of those corners, forms g_c = -sum gcp
// (feti.cpp:523-538, the order of k_coarse_rhs) and writes one quarter of the columns of the
// group's share of the coarse solve z = C^-1 g (feti.cpp:483-490),
//   zpart[j][q] = sum_{c in slice q} C^-1[c][j] g_c        (C^-1 symmetric: row c = column c)
// while the GEMV CTAs stream S_bb^-1 -- no coarse CTA waits for another one -- then counts
// itself on ctr[1].  The fused tail finds ctr[1] == 4 ng, sums the ng partials of the corners
// its rows touch (fixed order) and skips its own coarse phase and the grid barrier after it.
// The poll is one-directional (GEMV CTAs never wait) and bounded: a coarse CTA that does not
// see its partials within ~200 us gives up, ctr[1] stays short, and the tail computes z
// itself -- no spin can hang, whatever the residency.
struct CoarseAsideArgs {
  int n_sub, ng, nc;
  int giveup;  // test hook: act as if the partials never arrived
  const double2* Cinv;
  const int* corner_slots;  // [nc][4]
  double2* zpart;           // [nc][ng]
  unsigned int* ctr;        // [1] coarse CTAs done (reset by the tail)
  unsigned long long* tstamp;  // FETIGPU_TAIL_TIMES: slots 10..14 of the step (coarse CTA 0)
  const int* it_ptr;
};
constexpr int kAsideCpgMax = 32;  // corners per coarse group (4 poll threads each: one CTA)
template <int SYM_BATCH, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, (WARPS == 8 ? 4 : 8)) k_sym_gemv_aside(SymGemvArgs a, CoarseAsideArgs ca) {
  static_assert(WARPS * 32 >= 4 * kAsideCpgMax, "one poll thread per (corner, partial)");
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((int)blockIdx.x < ca.n_sub) {
    const int NT = a.NT, noff = NT * (NT - 1) / 2;
    if (warp < noff) {
      const double2* O = a.pack + (size_t)blockIdx.x * sym_tile_entries(NT) + NT * 17 * 32 + (size_t)warp * 1024;
#pragma unroll
      for (int u = 0; u < FETIGPU_GEMV_PF_ROWS_ASIDE; ++u) prefetch_l1(O + u * 32 + lane);
    }
    // solve-constant coupling entries of this warp's corner (NB <= 128: four rows per lane)
    double2 cp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = lane + 32 * q;
      cp[q] = (warp < a.NC && k < a.NB) ? a.cpl_b[((size_t)blockIdx.x * a.NB + k) * a.NC + warp] : cz();
    }
    const SymPre pre = sym_pre_load<1>(a, blockIdx.x);
    pdl_wait();
    if (a.cont_ptr != nullptr && *a.cont_ptr == 0) return;
    sym_gemv_run<1, SYM_BATCH, WARPS, true>(a, &pre, cp);
    return;
  }
  // ---- coarse CTA: quarter `qd` of the columns of group `gq` ----
  __shared__ double2 gs[kAsideCpgMax];
  const int x = blockIdx.x - ca.n_sub, gq = x >> 2, qd = x & 3, nc = ca.nc;
  const int cpg = (nc + ca.ng - 1) / ca.ng;
  const int c0 = gq * cpg, ncs = max(0, min(cpg, nc - c0));  // the group's corners [c0, c0 + ncs)
  // thread t < 4 ncs polls partial t & 3 of corner c0 + t / 4; its slot is solve-constant
  const int my_slot = (int)threadIdx.x < 4 * ncs ? ca.corner_slots[(size_t)c0 * 4 + threadIdx.x] : -1;
  // columns of this CTA: [j_lo, j_hi), thread t takes j_lo + t + 128 m
  const int jq = (nc + 3) / 4, j_lo = qd * jq, j_hi = min(nc, j_lo + jq);
  const bool stamp = ca.tstamp != nullptr && x == 0 && threadIdx.x == 0;
  unsigned long long ts0 = 0;
  if (stamp) ts0 = gtimer();
  pdl_wait();
  if (a.cont_ptr != nullptr && *a.cont_ptr == 0) return;
  unsigned long long* ts = stamp ? ca.tstamp + (size_t)(*ca.it_ptr) * 16 : nullptr;
  if (stamp) {
    ts[10] = ts0;
    ts[11] = gtimer();
  }
  bool ok = ca.giveup == 0;
  {
    double2 p = cz();
    if (my_slot >= 0 && ok) {
      const unsigned long long t0 = gtimer();
      for (;;) {
        asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(p.x), "=d"(p.y) : "l"(a.gcp + my_slot) : "memory");
        if (__double_as_longlong(p.x) != -1LL && __double_as_longlong(p.y) != -1LL) break;
        if (gtimer() - t0 > 200000ULL) {
          ok = false;
          break;
        }
      }
    }
    // g_c = ((0 - p0) - p1) - p2 - p3 on the corner's first lane
    const double2 p1 = shfl2(p, (lane & ~3) + 1), p2 = shfl2(p, (lane & ~3) + 2), p3 = shfl2(p, (lane & ~3) + 3);
    if ((threadIdx.x & 3) == 0 && (int)threadIdx.x < 4 * ncs)
      gs[threadIdx.x >> 2] = csub(csub(csub(csub(cz(), p), p1), p2), p3);
  }
  if (!__syncthreads_and(ok ? 1 : 0)) return;
  if (stamp) ts[12] = ts[13] = gtimer();
  // zpart[j][gq] = sum_i g_i C^-1[c0 + i][j] for this CTA's columns, rows in ascending order,
  // RB rows (RB x 2 loads per thread) in flight
  constexpr int TPB = WARPS * 32, RB = 4;
  for (int j0 = j_lo; j0 < j_hi; j0 += 2 * TPB) {
    const int ja = min(j0 + (int)threadIdx.x, nc - 1), jb = min(j0 + (int)threadIdx.x + TPB, nc - 1);
    double2 acc_a = cz(), acc_b = cz();
    for (int i0 = 0; i0 < ncs; i0 += RB) {
      double2 va[RB], vb[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const double2* cr = ca.Cinv + (size_t)(c0 + min(i0 + u, ncs - 1)) * nc;
        va[u] = __ldg(cr + ja);
        vb[u] = __ldg(cr + jb);
      }
#pragma unroll
      for (int u = 0; u < RB; ++u)
        if (i0 + u < ncs) {
          const double2 g = gs[i0 + u];
          acc_a = cfma(va[u], g, acc_a);
          acc_b = cfma(vb[u], g, acc_b);
        }
    }
    if (j0 + (int)threadIdx.x < j_hi) __stcg(ca.zpart + (size_t)(j0 + threadIdx.x) * ca.ng + gq, acc_a);
    if (j0 + (int)threadIdx.x + TPB < j_hi) __stcg(ca.zpart + (size_t)(j0 + threadIdx.x + TPB) * ca.ng + gq, acc_b);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ca.ctr + 1) : "memory");
  }
  if (stamp) ts[14] = gtimer();
}

// Grid barrier on a monotonically increasing 64-bit arrival counter: barrier k of the
// kernel's lifetime completes when the counter reaches (k+1) G.  Arrival is one acq_rel
// atomic (release: the block's writes, ordered by the preceding bar.sync; acquire: for the
// last arriver); the others poll with acquire loads.  No reset step, no generation word.
__device__ __forceinline__ void grid_sync_plain(unsigned int* bar) {
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(bar);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ticket;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(ticket) : "l"(ctr) : "memory");
    const unsigned long long target = (ticket / gridDim.x + 1) * gridDim.x;
    if (ticket + 1 != target) {
      const long long t0 = clock64();
      unsigned long long v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (clock64() - t0 > 4000000000LL) __trap();  // ~2 s: never hang the device
      } while (v < target);
    }
  }
  __syncthreads();
}

// every block: out[i] = sum_b part[i][b] for i < nout, fixed order (identical in all blocks)
template <int THREADS>
__device__ __forceinline__ void block_reduce_parts(const double2* __restrict__ part, int G, int nout,
                                                   double2* out_sh) {
  constexpr int SEGS = 16, PER = THREADS / SEGS;
  const int seg = threadIdx.x % SEGS;
  for (int i0 = 0; i0 < nout; i0 += PER) {
    const int i = i0 + threadIdx.x / SEGS;
    double2 t = cz();
    if (i < nout) {
      const double2* pp = part + (size_t)i * G;
      constexpr int QB = 10;  // G <= 160 (one block per SM): all of a thread's loads in one batch
      if (G <= SEGS * QB) {
        double2 v[QB];
#pragma unroll
        for (int q = 0; q < QB; ++q) v[q] = (seg + SEGS * q < G) ? __ldcg(pp + seg + SEGS * q) : cz();
#pragma unroll
        for (int q = 0; q < QB; ++q) t = cadd(t, v[q]);
      } else {
#pragma unroll 8
        for (int bb = seg; bb < G; bb += SEGS) t = cadd(t, __ldcg(pp + bb));
      }
    }
#pragma unroll
    for (int m = SEGS / 2; m > 0; m >>= 1) t = cadd(t, shfl_xor2(t, m));
    if (seg == 0 && i < nout) out_sh[i] = t;
  }
  __syncthreads();
}

// Fused tail, one multiplier row per thread, THREADS rows per block, one block per SM.
// dynamic smem: w_sh / g_sh [wg = max(THREADS, nc)] | h1[kTailHcs] | h2[kTailHcs] | Givens
// staging[640] | z_sh[nc] (ASIDE).  The dot vectors h1 / h2 (nv + 1 entries) live in shared
// memory while they fit kTailHcs entries and in a per-block global scratch beyond (long
// cycles): the tail's footprint does not grow with max_iter (it used to: the fused tail was
// then unavailable for small and for very large max_iter).
template <int THREADS, int NCM, int MINB, bool ASIDE>
__global__ void __launch_bounds__(THREADS, MINB) k_arnoldi_tail(ArnoldiTailArgs a) {
  constexpr int WARPS = THREADS / 32, LPR = THREADS / 32;
  extern __shared__ double2 tail_sh[];
  double2* w_sh = tail_sh;
  double2* hs1s = w_sh + a.wg;
  double2* hs2s = hs1s + kTailHcs;
  double2* stage = hs2s + kTailHcs;
  double2* z_sh = stage + 640;  // [nc], aside path only (host sizes the dynamic smem)
  __shared__ double2 cred[WARPS];
  __shared__ double inv_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rows_pb (<= THREADS) rows per block so that the grid can fill every SM
  const int row0 = blockIdx.x * a.rows_pb, r = row0 + threadIdx.x;
  const bool act = (int)threadIdx.x < a.rows_pb && r < a.n;
  const int row_end = min(a.n, row0 + a.rows_pb);  // exclusive
  pdl_trigger();
  // ---- before pdl_wait: solve-constant data only (PDL contract, common.cuh) ----
  // dual-tail index/coupling operands of this thread's multiplier row
  int slots[2] = {0, 0};
  double2 cpv[2][NCM];
  int cgv[2][NCM];
  if (act) {
    slots[0] = a.lam_lo[r];
    slots[1] = a.lam_hi[r];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int s = slots[q] / a.NB;
#pragma unroll
      for (int c = 0; c < NCM; ++c) {
        cgv[q][c] = c < a.NC ? a.cglob[(size_t)s * a.NC + c] : -1;
        cpv[q][c] = c < a.NC ? a.cpl_b[(size_t)slots[q] * a.NC + c] : cz();
      }
    }
  }
  // ASIDE (the coarse solve ran beside the dual GEMV, k_sym_gemv_aside): 4 threads per corner
  // of the block's list sum its aside_nx partials; the coarse phase below is only the path
  // taken when that launch gave up.  Otherwise: warm L1 with the coarse phase's constant
  // operands -- the corner-slot lists of this thread's first two coarse rows in registers
  // (the rest, for large coarse spaces, warmed into L1) and this block's first round of
  // C^-1 rows.
  static_assert(!ASIDE || kTailCorners * 4 == THREADS, "one pass over the block's corner list");
  constexpr int PB = 10;  // partials per thread in one batch (aside_nx <= 40 groups)
  int csl[2][4];
  int bc = -1;
  if constexpr (!ASIDE) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = threadIdx.x + h * THREADS;
#pragma unroll
      for (int q = 0; q < 4; ++q) csl[h][q] = k < a.nc ? a.corner_slots[k * 4 + q] : -1;
    }
    for (int k = threadIdx.x + 2 * THREADS; k < a.nc; k += THREADS) prefetch_l1(a.corner_slots + k * 4);
    const int row = blockIdx.x * (WARPS / 2) + (warp >> 1);
    if (row < a.nc) {
      const double2* cr = a.Cinv + (size_t)row * a.nc;
      for (int k0 = (warp & 1) * 32 + lane; k0 < a.nc; k0 += 64) prefetch_l1(cr + k0);
    }
  } else {
    bc = a.blk_corners[(size_t)blockIdx.x * kTailCorners + threadIdx.x / 4];
  }
  pdl_wait();
  // requested together (one latency): the cycle state, the coarse CTAs' done count (ASIDE) or
  // the dual GEMV's coarse partials, and the dual-tail operands that do not depend on z
  unsigned int aside_done = 0;
  double2 gv[2][4];
  if constexpr (ASIDE) {
    aside_done = __ldcg(a.aside_ctr + 1);
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < 4; ++q) gv[h][q] = csl[h][q] >= 0 ? a.gcp[csl[h][q]] : cz();
  }
  double2 u[2] = {cz(), cz()};
  if (act) {
    u[0] = a.u1b[slots[0]];
    u[1] = a.u1b[slots[1]];
  }
  if (a.st->cont == 0) {  // unrolled WHILE body: the cycle already stopped (or never started:
    // zero rhs) -- make sure the WHILE node exits
    if (a.ga.in_graph && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.ga.handle, 0u);
    return;
  }
  if (a.pf_bytes != 0u) {
    const int per = (a.pf_count + (int)gridDim.x - 1) / (int)gridDim.x;
    const int sidx = blockIdx.x * per + threadIdx.x;
    if ((int)threadIdx.x < per && sidx < a.pf_count) prefetch_l2_bulk(a.pf_base + (size_t)sidx * a.pf_stride, a.pf_bytes);
  }
  // z already there?  (the same answer in every block: the count was final when the dual
  // GEMV's launch ended and is reset only after this kernel's last barrier)
  const bool aside = ASIDE && aside_done == 4u * a.aside_nx;
  const int nv = a.st->j + 1, nout = nv + 1, G = gridDim.x;
  const int it = a.st->iterations;
  double2* hs1 = nout <= a.hcs ? hs1s : a.hbuf + (size_t)blockIdx.x * 2 * a.hcap;
  double2* hs2 = nout <= a.hcs ? hs2s : hs1 + a.hcap;
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 0] = gtimer();
  // Givens operands known now (block 0): loaded during the coarse phase, off the critical path
  __shared__ GivensPre gpre;
  if (!a.split_givens && blockIdx.x == 0 && warp == 0)
    givens_prefetch(a.ga, &gpre, reinterpret_cast<double*>(stage), stage + 128);
  span_mark(a.span, &it, 2, 0);
  if constexpr (ASIDE) {
    if (aside) {
      // z at the block's corners = sum of the coarse groups' partials, fixed order: each of the
      // corner's 4 threads sums partials sub, sub + 4, ..., then a xor tree over the 4 lanes
      // (loading the partials before the count is known costs registers across the prologue:
      // measured slower)
      const int sub = threadIdx.x & 3;
      double2 zp[PB];
#pragma unroll
      for (int q = 0; q < PB; ++q)
        zp[q] = (bc >= 0 && sub + 4 * q < (int)a.aside_nx) ? __ldcg(a.zpart + (size_t)bc * a.aside_nx + sub + 4 * q) : cz();
      double2 t = cz();
#pragma unroll
      for (int q = 0; q < PB; ++q) t = cadd(t, zp[q]);
      t = cadd(t, shfl_xor2(t, 2));
      t = cadd(t, shfl_xor2(t, 1));
      if ((threadIdx.x & 3) == 0 && bc >= 0) z_sh[bc] = t;
      __syncthreads();
    }
  }
  // ---- phase 0: z = C^-1 g.  g staged in smem (reusing the w buffer); each warp takes one
  // coarse row at a time with all of its lane's loads in one batch (clamped addresses) ----
  if (!aside) {
    double2* g_sh = w_sh;  // (wg >= nc entries)
    // coarse rhs g = -sum_s gcp over the (up to 4) subdomains of each corner, assembled
    // redundantly by every block (same order as k_coarse_rhs)
    if constexpr (!ASIDE) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = threadIdx.x + h * THREADS;
        double2 acc = cz();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (csl[h][q] >= 0) acc = csub(acc, gv[h][q]);
        if (k < a.nc) g_sh[k] = acc;
      }
    }
    for (int k = threadIdx.x + (ASIDE ? 0 : 2 * THREADS); k < a.nc; k += THREADS) {
      double2 acc = cz();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int slot = a.corner_slots[k * 4 + q];
        if (slot >= 0) acc = csub(acc, a.gcp[slot]);
      }
      g_sh[k] = acc;
    }
    __syncthreads();
    // two warps per coarse row (column halves interleaved by 32), 16 loads per lane in flight
    constexpr int CB = 16;
    const int half = warp & 1;
    for (int base = blockIdx.x * (WARPS / 2); base < a.nc; base += G * (WARPS / 2)) {
      const int row = base + (warp >> 1);
      double2 acc = cz();
      if (row < a.nc) {
        const double2* cr = a.Cinv + (size_t)row * a.nc;
        for (int k0 = half * 32 + lane; k0 < a.nc; k0 += 64 * CB) {
          double2 v[CB];
#pragma unroll
          for (int q = 0; q < CB; ++q) v[q] = __ldg(cr + min(k0 + 64 * q, a.nc - 1));
#pragma unroll
          for (int q = 0; q < CB; ++q)
            if (k0 + 64 * q < a.nc) acc = cfma(v[q], g_sh[k0 + 64 * q], acc);
        }
      }
      acc = warp_sum2(acc);
      if (lane == 0) cred[warp] = acc;
      __syncthreads();
      if ((int)threadIdx.x < WARPS / 2 && base + (int)threadIdx.x < a.nc)
        a.z[base + threadIdx.x] = cadd(cred[2 * threadIdx.x], cred[2 * threadIdx.x + 1]);
      __syncthreads();
    }
  }
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 1] = gtimer();
  if (!aside) grid_sync_plain(a.bar);
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 2] = gtimer();
  // block partials of conj(V_i) w (i < nv) and |w|^2 (i = nv), one warp per vector
  // pass-1 and pass-2 partials live in separate halves of `part`: every block reduces the
  // pass-1 partials after barrier B while faster blocks already write pass-2 partials
  auto dots = [&](double2 w, double2* part) {
    w_sh[threadIdx.x] = w;
    __syncthreads();
    for (int i = warp; i < nout; i += WARPS) {
      double2 acc = cz();
      if (i < nv) {
        const double2* v = a.V + (size_t)i * a.ldv + row0;
        double2 x[LPR];
#pragma unroll
        for (int q = 0; q < LPR; ++q) x[q] = v[min(lane + 32 * q, row_end - 1 - row0)];
#pragma unroll
        for (int q = 0; q < LPR; ++q) acc = cfma_conj(x[q], w_sh[lane + 32 * q], acc);
      } else {
#pragma unroll
        for (int q = 0; q < LPR; ++q) acc.x += cabs2(w_sh[lane + 32 * q]);
      }
      acc = warp_sum2(acc);
      if (lane == 0) part[(size_t)i * G + blockIdx.x] = acc;
    }
  };
  double2* part2 = a.part + (size_t)a.hcap * G;
  auto sub_vh = [&](double2 w, const double2* h) {  // w - sum_i h_i V_i[r], h in smem
    if (!act) return w;
    double2 acc = cz();
    int i = 0;
    for (; i + 8 <= nv; i += 8) {
      double2 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = a.V[(size_t)(i + q) * a.ldv + r];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = cfma(h[i + q], v[q], acc);
    }
    for (; i < nv; ++i) acc = cfma(h[i], a.V[(size_t)i * a.ldv + r], acc);
    return csub(w, acc);
  };
  // ---- phase 1: w = F z (dual tail), h1 = V^H w, |w|^2 ----
  double2 w = cz();
  if (act) {
    double2 ud[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      double2 cz_ = cz();
#pragma unroll
      for (int c = 0; c < NCM; ++c)
        if (cgv[q][c] >= 0) cz_ = cfma(cpv[q][c], (ASIDE && aside) ? z_sh[cgv[q][c]] : __ldcg(a.z + cgv[q][c]), cz_);
      ud[q] = csub(u[q], cz_);
    }
    const double2 d = csub(ud[0], ud[1]);
    w = make_double2(-d.x, -d.y);
  }
  dots(w, a.part);
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 3] = gtimer();
  grid_sync_plain(a.bar);
  block_reduce_parts<THREADS>(a.part, G, nout, hs1);
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 4] = gtimer();
  // ---- phase 2: w -= V h1, h2 = V^H w, |w|^2 ----
  w = sub_vh(w, hs1);
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 5] = gtimer();
  __syncthreads();  // w_sh reuse
  dots(w, part2);
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 6] = gtimer();
  grid_sync_plain(a.bar);
  block_reduce_parts<THREADS>(part2, G, nout, hs2);
  if (warp == 0) {
    bool finite;
    const double hn = warp_hnext<true>(hs1, hs2, nv - 1, finite);
    if (lane == 0) inv_sh = 1.0 / hn;
  }
  __syncthreads();
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 7] = gtimer();
  // ---- phase 3: V_{j+1} = (w - V h2) / h_{j+1,j} (written even if the cycle stops: unused) ----
  if (nv < a.vcap) {
    w = sub_vh(w, hs2);
    if (act) a.V[(size_t)nv * a.ldv + r] = cscale(w, inv_sh);
  }
  if (a.tstamp && blockIdx.x == 0 && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 8] = gtimer();
  // block 0: Givens, stopping tests, WHILE-node condition; h1/h2 published for the host side
  if (blockIdx.x == 0) {
    if (ASIDE && threadIdx.x == 0) a.aside_ctr[1] = 0u;  // (every block read it before the barriers above)
    for (int i = threadIdx.x; i < nout; i += THREADS) {
      a.h1[i] = hs1[i];
      a.h2[i] = hs2[i];
    }
    if (a.split_givens) {
      if (threadIdx.x == 0) a.st->jcol = nv;  // the next step's basis column (k_givens runs aside)
    } else if (warp == 0) {
      givens_warp<true>(a.ga, reinterpret_cast<double*>(stage), stage + 128, stage + 384, hs1, hs2, &gpre);
    }
    if (a.tstamp && threadIdx.x == 0) a.tstamp[(size_t)it * 16 + 9] = gtimer();
  }
  // coarse partials back to the all-ones sentinel for the next step's k_sym_gemv_aside
  if constexpr (ASIDE) {
    const double ones = __longlong_as_double(-1LL);
    for (int i = blockIdx.x * THREADS + threadIdx.x; i < a.n_gcp; i += G * THREADS)
      __stcg(const_cast<double2*>(a.gcp) + i, make_double2(ones, ones));
  }
  if (a.span != nullptr) {
    __syncthreads();
    span_mark(a.span, &it, 2, 1);
  }
}

// Multi-row form of the fused tail for interfaces with more multiplier rows than one row per
// thread of a co-resident grid (n > SMs x THREADS; BASELINE config 3: 250k rows): every thread
// carries up to RPT rows (row0 + threadIdx.x + q THREADS), the coarse solve z = C^-1 g has
// already been computed by the coarse kernels of the step (large coarse spaces use the packed
// symmetric inverse), and the launch is CGS2 pass 1 (+ dual-tail gather), pass 2 and the
// normalisation with two grid barriers.  dynamic smem: w_sh[THREADS RPT] | h1[kTailHcs] |
// h2[kTailHcs] | Givens staging[640].  Same reduction order as k_arnoldi_tail (block partials
// in block order), same Givens / split-Givens protocol.
template <int THREADS, int RPT>
__global__ void __launch_bounds__(THREADS, 1) k_arnoldi_tail_mr(ArnoldiTailArgs a) {
  constexpr int WARPS = THREADS / 32, ROWS = THREADS * RPT, DB = 16;
  extern __shared__ double2 tail_sh[];
  double2* w_sh = tail_sh;
  double2* hs1s = w_sh + ROWS;
  double2* hs2s = hs1s + kTailHcs;
  double2* stage = hs2s + kTailHcs;
  __shared__ double inv_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * a.rows_pb;
  const int row_end = min(a.n, row0 + a.rows_pb);  // exclusive
  const int nrows = max(row_end - row0, 0);
  pdl_trigger();
  pdl_wait();
  if (a.st->cont == 0) {
    if (a.ga.in_graph && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.ga.handle, 0u);
    return;
  }
  const int nv = a.st->j + 1, nout = nv + 1, G = gridDim.x;
  const int it = a.st->iterations;
  double2* hs1 = nout <= a.hcs ? hs1s : a.hbuf + (size_t)blockIdx.x * 2 * a.hcap;
  double2* hs2 = nout <= a.hcs ? hs2s : hs1 + a.hcap;
  span_mark(a.span, &it, 2, 0);
  auto dots = [&](const double2* w, double2* part) {
#pragma unroll
    for (int q = 0; q < RPT; ++q) w_sh[threadIdx.x + q * THREADS] = w[q];  // (zero beyond the block's rows)
    __syncthreads();
    for (int i = warp; i < nout; i += WARPS) {
      double2 acc = cz();
      if (i < nv) {
        const double2* v = a.V + (size_t)i * a.ldv + row0;
        for (int k0 = lane; k0 < nrows; k0 += 32 * DB) {
          double2 x[DB];
#pragma unroll
          for (int u = 0; u < DB; ++u) x[u] = v[min(k0 + 32 * u, nrows - 1)];
#pragma unroll
          for (int u = 0; u < DB; ++u)
            if (k0 + 32 * u < nrows) acc = cfma_conj(x[u], w_sh[k0 + 32 * u], acc);
        }
      } else {
        for (int k0 = lane; k0 < nrows; k0 += 32) acc.x += cabs2(w_sh[k0]);
      }
      acc = warp_sum2(acc);
      if (lane == 0) part[(size_t)i * G + blockIdx.x] = acc;
    }
  };
  auto sub_vh = [&](double2 w, int r, const double2* h) {  // w - sum_i h_i V_i[r]
    double2 acc = cz();
    int i = 0;
    for (; i + 8 <= nv; i += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a.V[(size_t)(i + u) * a.ldv + r];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = cfma(h[i + u], v[u], acc);
    }
    for (; i < nv; ++i) acc = cfma(h[i], a.V[(size_t)i * a.ldv + r], acc);
    return csub(w, acc);
  };
  // ---- phase 1: w = F z (dual tail), h1 = V^H w, |w|^2 ----
  double2 w[RPT];
  bool act[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int lr = threadIdx.x + q * THREADS;
    act[q] = lr < nrows;
    // augmented dual problem: w = P F z was gathered and projected per edge (k_gather_project_edges)
    w[q] = !act[q] ? cz() : a.w_in != nullptr ? a.w_in[row0 + lr] : dual_tail_row(a, row0 + lr, true);
  }
  dots(w, a.part);
  grid_sync_plain(a.bar);
  block_reduce_parts<THREADS>(a.part, G, nout, hs1);
  // ---- phase 2: w -= V h1, h2 = V^H w, |w|^2 ----
#pragma unroll
  for (int q = 0; q < RPT; ++q)
    if (act[q]) w[q] = sub_vh(w[q], row0 + threadIdx.x + q * THREADS, hs1);
  __syncthreads();  // w_sh reuse
  double2* part2 = a.part + (size_t)a.hcap * G;
  dots(w, part2);
  grid_sync_plain(a.bar);
  block_reduce_parts<THREADS>(part2, G, nout, hs2);
  if (warp == 0) {
    bool finite;
    const double hn = warp_hnext<true>(hs1, hs2, nv - 1, finite);
    if (lane == 0) inv_sh = 1.0 / hn;
  }
  __syncthreads();
  // ---- phase 3: V_{j+1} = (w - V h2) / h_{j+1,j} ----
  if (nv < a.vcap) {
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (act[q]) {
        const int r = row0 + threadIdx.x + q * THREADS;
        a.V[(size_t)nv * a.ldv + r] = cscale(sub_vh(w[q], r, hs2), inv_sh);
      }
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < nout; i += THREADS) {
      a.h1[i] = hs1[i];
      a.h2[i] = hs2[i];
    }
    if (a.split_givens) {
      if (threadIdx.x == 0) a.st->jcol = nv;
    } else if (warp == 0) {
      givens_warp<true>(a.ga, reinterpret_cast<double*>(stage), stage + 128, stage + 384, hs1, hs2);
    }
  }
  if (a.span != nullptr) {
    __syncthreads();
    span_mark(a.span, &it, 2, 1);
  }
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
// y = a - b and, in the same pass, the block partials (sum |y|^2, max |y|) of k_norm_max_part
// (same grid-stride order: the sums are bit-identical to k_sub followed by k_norm_max_part)
__global__ void k_sub_norm_part(int n, const double2* __restrict__ a, const double2* __restrict__ b,
                                double2* __restrict__ y, double2* __restrict__ part) {
  __shared__ double ssum[32], smax[32];
  double s = 0.0, m = 0.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const double2 v = csub(a[k], b[k]);
    y[k] = v;
    const double a2 = cabs2(v);
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
  // each lane sums its partials b = lane, lane + 32, ... in that order; the loads of 8
  // consecutive ones are issued together (same sum as the one-at-a-time loop)
  double s = 0.0, m = 0.0;
  for (int b0 = threadIdx.x; b0 < nblk; b0 += 32 * 8) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b0 + 32 * u < nblk ? part[b0 + 32 * u] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b0 + 32 * u < nblk) s += v[u].x, m = fmax(m, v[u].y);
  }
  s = warp_sum(s);
  m = warp_max(m);
  if (threadIdx.x == 0) *out = make_double2(s, m);
}

// the same over many partials (the stencil residual's one-per-row-segment blocks): 1024
// threads, each summing partials t, t + 1024, ... in order, then a fixed-order block reduce
// out = (sum part.x, max part.y) over nblk partials; out_q (optional) likewise over the next nblk
__global__ void __launch_bounds__(1024) k_norm_max_final_big(int nblk, const double2* __restrict__ part,
                                                             double2* __restrict__ out, double2* __restrict__ out_q = nullptr) {
  __shared__ double ws[32], wm[32];
  if (out_q != nullptr && blockIdx.x == 1) {
    part += nblk;
    out = out_q;
  }
  double s = 0.0, m = 0.0;
  for (int b0 = threadIdx.x; b0 < nblk; b0 += 1024 * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = b0 + 1024 * u < nblk ? part[b0 + 1024 * u] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b0 + 1024 * u < nblk) s += v[u].x, m = fmax(m, v[u].y);
  }
  s = warp_sum(s);
  m = warp_max(m);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) ws[warp] = s, wm[warp] = m;
  __syncthreads();
  if (warp == 0) {
    s = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0.0;
    m = lane < (int)(blockDim.x >> 5) ? wm[lane] : 0.0;
    s = warp_sum(s);
    m = warp_max(m);
    if (lane == 0) *out = make_double2(s, m);
  }
}
// max over block partials of k_imag_max_part -> out->y (out->x = 0)
__global__ void k_max_final(int nblk, const double* __restrict__ part, double2* __restrict__ out) {
  double m = 0.0;
  for (int b0 = threadIdx.x; b0 < nblk; b0 += 32 * 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b0 + 32 * u < nblk ? part[b0 + 32 * u] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) m = fmax(m, v[u]);
  }
  m = warp_max(m);
  if (threadIdx.x == 0) *out = make_double2(0.0, m);
}

// ---- real vector helpers of the full-space method (3n-vectors) --------------------------
__global__ void k_rdot_part(long long n, const double* __restrict__ x, const double* __restrict__ y,
                            double* __restrict__ part) {
  __shared__ double sm[32];
  double s = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    s = fma(x[k], y[k], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm[w];
    part[blockIdx.x] = t;
  }
}
__global__ void k_rdot_final(int nb, const double* __restrict__ part, double* __restrict__ out) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) s += part[b];
  s = warp_sum(s);
  if (threadIdx.x == 0) *out = s;
}
// y = a x + b y
__global__ void k_axpby(long long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = b == 0.0 ? a * x[k] : fma(a, x[k], b * y[k]);
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
__global__ void k_apply_global(MeshLayout M, ElemKM KM, int n, const int* __restrict__ free_dofs, const int* __restrict__ free_map,
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
          const double kv = KM.k[ra * ed + dpn * b + cb], mv = KM.m[ra * ed + dpn * b + cb];
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

// Structured fast path of k_apply_global (scalar physics, every boundary node constrained):
// the free dofs are the (nx-1) x (ny-1) interior nodes in lexicographic order, so the
// assembled Q1 operator kc K + mc M is one 9-point stencil (coef[dy+1][dx+1], built on the
// host from the element matrices).  No constrained-value term (xc == nullptr only).
struct Stencil9 {
  double2 c[9];
};
// rows [j0, j0 + gridDim.y) of y = stencil x for a REAL x, written as complex (the Schur rhs
// K ybar, control.cpp:15, row block by row block as ybar arrives from the host)
__global__ void k_apply_stencil9_rc(int fx, int fy, int j0, Stencil9 S, const double* __restrict__ x,
                                    double2* __restrict__ y) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x, J = j0 + blockIdx.y;
  if (I >= fx) return;
  double2 acc = cz();
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    const int jj = J + dy;
    if (jj < 0 || jj >= fy) continue;
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      const int ii = I + dx;
      if (ii < 0 || ii >= fx) continue;
      acc = cfma(S.c[(dy + 1) * 3 + dx + 1], as_c<double>(x[(size_t)jj * fx + ii]), acc);
    }
  }
  y[(size_t)J * fx + I] = acc;
}
template <typename T>
__global__ void k_apply_stencil9(int fx, int fy, Stencil9 S, const T* __restrict__ x, T* __restrict__ y) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y;
  if (I >= fx) return;
  double2 acc = cz();
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    const int jj = J + dy;
    if (jj < 0 || jj >= fy) continue;
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      const int ii = I + dx;
      if (ii < 0 || ii >= fx) continue;
      acc = cfma(S.c[(dy + 1) * 3 + dx + 1], as_c<T>(x[(size_t)jj * fx + ii]), acc);
    }
  }
  store_c<T>(y + (size_t)J * fx + I, acc);
}

// Statistics without materialising the vectors: block partials (|v|^2, max|v|) of the
// interface jump v_r = u_lo - u_hi (feti.cpp:708-709) and of the primal residual
// v = (kc K + mc V) x - rhs on the structured stencil (feti.cpp:711-713).
__device__ __forceinline__ void block_sum_max(double s, double m, double2* part) {
  __shared__ double ss[32], sm_[32];
  s = warp_sum(s);
  m = warp_max(m);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) ss[warp] = s, sm_[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tm = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ts += ss[w], tm = fmax(tm, sm_[w]);
    part[blockIdx.x] = make_double2(ts, tm);
  }
}
__global__ void k_jump_norm_part(int nl, const int* __restrict__ lo, const int* __restrict__ hi,
                                 const double2* __restrict__ u1b, double2* __restrict__ part) {
  double s = 0.0, m = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double a2 = cabs2(csub(u1b[lo[r]], u1b[hi[r]]));
    s += a2;
    m = fmax(m, sqrt(a2));
  }
  block_sum_max(s, m, part);
}
// as block_sum_max, plus a second sum q -> part_q[blockIdx.x] = (q, 0)
__device__ __forceinline__ void block_sum_max_q(double s, double m, double q, double2* part, double2* part_q) {
  __shared__ double ss[32], sm_[32], sq[32];
  s = warp_sum(s);
  m = warp_max(m);
  q = warp_sum(q);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) ss[warp] = s, sm_[warp] = m, sq[warp] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tm = 0.0, tq = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ts += ss[w], tm = fmax(tm, sm_[w]), tq += sq[w];
    part[blockIdx.x] = make_double2(ts, tm);
    part_q[blockIdx.x] = make_double2(tq, 0.0);
  }
}
// primal residual |A x - rhs|^2 / max (feti.cpp:711-713) by the 9-point stencil, per block; the
// same pass sums |rhs|^2 (the residual's scale) into part[nblk + blk]
__global__ void k_stencil_residual_part(int fx, int fy, Stencil9 S, const double2* __restrict__ x,
                                        const double2* __restrict__ rhs, double2* __restrict__ part) {
  double s = 0.0, m = 0.0, q = 0.0;
  // one row per blockIdx.y, one column per thread: every load of the launch in flight at once
  const int J = blockIdx.y, I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I < fx) {
    const size_t f = (size_t)J * fx + I;
    double2 acc = cz();
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int jj = J + dy;
      if (jj < 0 || jj >= fy) continue;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int ii = I + dx;
        if (ii < 0 || ii >= fx) continue;
        acc = cfma(S.c[(dy + 1) * 3 + dx + 1], x[(size_t)jj * fx + ii], acc);
      }
    }
    const double2 b = rhs[f];
    const double a2 = cabs2(csub(acc, b));
    s += a2;
    m = fmax(m, sqrt(a2));
    q += cabs2(b);
  }
  const size_t nblk = (size_t)gridDim.x * gridDim.y;
  block_sum_max_q(s, m, q, part + (size_t)blockIdx.y * gridDim.x, part + nblk + (size_t)blockIdx.y * gridDim.x);
}

// Kronecker mass solve V^-1 = (M_y ⊗ M_x ⊗ I_dpn)^-1: batches of identical SPD tridiagonal
// systems (constant off-diagonal 'off', pre-factored Thomas coefficients cp, dinv).
// Each line is split into 32 segments; the Thomas recurrences
//   forward  d'_i = d_i dinv_i - off dinv_i d'_{i-1},   backward x_i = d'_i - cp_i x_{i+1}
// are affine maps, composed per segment, scanned across segments and re-applied, so the
// sequential depth is ~4 len/32 instead of 2 len.  Same arithmetic as Thomas up to the
// order of the affine compositions (|off dinv| < 1/3: forward stable).
// Element i of line t sits at v[(t / G) * S1 + (t % G) * S2 + i * es].
// SEG_FAST: block = (32 segments, LPB lines) — for lines contiguous in memory;
// otherwise block = (LPB lines, 32 segments) so a warp reads 32 adjacent lines (coalesced).
template <int LPB, bool SEG_FAST>
__global__ void __launch_bounds__(32 * LPB)
    k_tridiag_lines(double* __restrict__ v, int nlines, int len, int G, long long S1, long long S2, long long es,
                    const double* __restrict__ cp, const double* __restrict__ dinv, double off) {
  // segments of up to MAXL entries live in registers: one batch of independent loads, the
  // four recurrences on registers, one batch of stores (the in-place global version waits
  // on a load behind every store: 58 us -> see DESIGN §4)
  constexpr int MAXL = 32;
  __shared__ double sa[LPB][33], sb[LPB][33], sx[LPB][33];
  const int seg = SEG_FAST ? threadIdx.x : threadIdx.y, ly = SEG_FAST ? threadIdx.y : threadIdx.x;
  const int line = blockIdx.x * LPB + ly;
  const bool act = line < nlines;
  double* p = v + (act ? (long long)(line / G) * S1 + (long long)(line % G) * S2 : 0);
  const int L = (len + 31) / 32;
  const int i0 = min(len, seg * L), i1 = min(len, i0 + L), cnt = i1 - i0;
  const bool reg = L <= MAXL;
  double r[MAXL];
  if (reg) {
#pragma unroll
    for (int k = 0; k < MAXL; ++k) r[k] = (act && k < cnt) ? p[(long long)(i0 + k) * es] : 0.0;
  }
  // forward: compose x -> A + B x over the segment
  double a = 0.0, b = 1.0;
  if (act) {
    if (reg) {
#pragma unroll
      for (int k = 0; k < MAXL; ++k)
        if (k < cnt) {
          const double di = dinv[i0 + k];
          a = fma(-off * di, a, r[k] * di);
          b *= -off * di;
        }
    } else {
      for (int i = i0; i < i1; ++i) {
        const double di = dinv[i];
        a = fma(-off * di, a, p[(long long)i * es] * di);
        b *= -off * di;
      }
    }
  }
  sa[ly][seg] = a;
  sb[ly][seg] = b;
  __syncthreads();
  if (seg == 0) {
    double x = 0.0;
    for (int q = 0; q < 32; ++q) {
      sx[ly][q] = x;
      x = fma(sb[ly][q], x, sa[ly][q]);
    }
  }
  __syncthreads();
  double x = sx[ly][seg];
  if (act) {
    if (reg) {
#pragma unroll
      for (int k = 0; k < MAXL; ++k)
        if (k < cnt) {
          x = (r[k] - off * x) * dinv[i0 + k];
          r[k] = x;
        }
    } else {
      for (int i = i0; i < i1; ++i) {
        x = (p[(long long)i * es] - off * x) * dinv[i];
        p[(long long)i * es] = x;
      }
    }
  }
  // backward: x_i = d'_i - cp_i x_{i+1}
  a = 0.0;
  b = 1.0;
  if (act) {
    if (reg) {
#pragma unroll
      for (int k = MAXL - 1; k >= 0; --k)
        if (k < cnt) {
          a = fma(-cp[i0 + k], a, r[k]);
          b *= -cp[i0 + k];
        }
    } else {
      for (int i = i1 - 1; i >= i0; --i) {
        a = fma(-cp[i], a, p[(long long)i * es]);
        b *= -cp[i];
      }
    }
  }
  __syncthreads();
  sa[ly][seg] = a;
  sb[ly][seg] = b;
  __syncthreads();
  if (seg == 0) {
    double xx = 0.0;
    for (int q = 31; q >= 0; --q) {
      sx[ly][q] = xx;
      xx = fma(sb[ly][q], xx, sa[ly][q]);
    }
  }
  __syncthreads();
  x = sx[ly][seg];
  if (act) {
    if (reg) {
#pragma unroll
      for (int k = MAXL - 1; k >= 0; --k)
        if (k < cnt) {
          x = r[k] - cp[i0 + k] * x;
          r[k] = x;
        }
#pragma unroll
      for (int k = 0; k < MAXL; ++k)
        if (k < cnt) p[(long long)(i0 + k) * es] = r[k];
    } else {
      for (int i = i1 - 1; i >= i0; --i) {
        x = p[(long long)i * es] - cp[i] * x;
        p[(long long)i * es] = x;
      }
    }
  }
}
// Contiguous lines (x direction, one dof per node): the block's LPB lines (one contiguous
// range of LPB * len doubles) are staged through shared memory with coalesced loads and
// stores; segment k of a line is read from a padded layout (one pad per 32 entries: lanes
// reading entry k of their segments hit 32 different banks), then the same register
// recurrences as k_tridiag_lines.  len <= 32 * 32.
template <int LPB>
__global__ void __launch_bounds__(32 * LPB)
    k_tridiag_rows(double* __restrict__ v, int nlines, int len, const double* __restrict__ cp,
                   const double* __restrict__ dinv, double off) {
  constexpr int MAXL = 32;
  extern __shared__ double tr_sh[];
  __shared__ double sa[LPB][33], sb[LPB][33], sx[LPB][33];
  const int seg = threadIdx.x, ly = threadIdx.y;
  const int line0 = blockIdx.x * LPB, nb = min(LPB, nlines - line0);
  const int stride = len + len / 32 + 1;  // padded line length in shared memory
  double* base = v + (long long)line0 * len;
  const int tid = threadIdx.y * 32 + threadIdx.x, tot = nb * len;
  constexpr int NT = 32 * LPB, UB = 16;  // 16 loads in flight per thread
  for (int e0 = tid; e0 < tot; e0 += UB * NT) {
    double t[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) t[u] = e0 + u * NT < tot ? base[e0 + u * NT] : 0.0;
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int e = e0 + u * NT;
      if (e < tot) {
        const int l = e / len, i = e - l * len;
        tr_sh[l * stride + i + i / 32] = t[u];
      }
    }
  }
  // the line-independent Thomas coefficients, same padded layout (conflict-free per lane)
  double* sdinv = tr_sh + LPB * stride;
  double* scp = sdinv + stride;
  for (int i = tid; i < len; i += NT) {
    sdinv[i + i / 32] = dinv[i];
    scp[i + i / 32] = cp[i];
  }
  __syncthreads();
  const bool act = ly < nb;
  const int L = (len + 31) / 32;
  const int i0 = min(len, seg * L), i1 = min(len, i0 + L), cnt = i1 - i0;
  double* sl = tr_sh + ly * stride;
  double r[MAXL];
#pragma unroll
  for (int k = 0; k < MAXL; ++k) r[k] = (act && k < cnt) ? sl[i0 + k + (i0 + k) / 32] : 0.0;
  double a = 0.0, b = 1.0;
#pragma unroll
  for (int k = 0; k < MAXL; ++k)
    if (k < cnt) {
      const double di = sdinv[i0 + k + (i0 + k) / 32];
      a = fma(-off * di, a, r[k] * di);
      b *= -off * di;
    }
  sa[ly][seg] = a;
  sb[ly][seg] = b;
  __syncthreads();
  if (seg == 0) {
    double x = 0.0;
    for (int q = 0; q < 32; ++q) {
      sx[ly][q] = x;
      x = fma(sb[ly][q], x, sa[ly][q]);
    }
  }
  __syncthreads();
  double x = sx[ly][seg];
#pragma unroll
  for (int k = 0; k < MAXL; ++k)
    if (k < cnt) {
      x = (r[k] - off * x) * sdinv[i0 + k + (i0 + k) / 32];
      r[k] = x;
    }
  a = 0.0;
  b = 1.0;
#pragma unroll
  for (int k = MAXL - 1; k >= 0; --k)
    if (k < cnt) {
      a = fma(-scp[i0 + k + (i0 + k) / 32], a, r[k]);
      b *= -scp[i0 + k + (i0 + k) / 32];
    }
  __syncthreads();
  sa[ly][seg] = a;
  sb[ly][seg] = b;
  __syncthreads();
  if (seg == 0) {
    double xx = 0.0;
    for (int q = 31; q >= 0; --q) {
      sx[ly][q] = xx;
      xx = fma(sb[ly][q], xx, sa[ly][q]);
    }
  }
  __syncthreads();
  x = sx[ly][seg];
#pragma unroll
  for (int k = MAXL - 1; k >= 0; --k)
    if (k < cnt) {
      x = r[k] - scp[i0 + k + (i0 + k) / 32] * x;
      r[k] = x;
    }
#pragma unroll
  for (int k = 0; k < MAXL; ++k)
    if (act && k < cnt) sl[i0 + k + (i0 + k) / 32] = r[k];
  __syncthreads();
  for (int e = threadIdx.y * 32 + threadIdx.x; e < nb * len; e += 32 * LPB) {
    const int l = e / len, i = e - l * len;
    base[e] = tr_sh[l * stride + i + i / 32];
  }
}
// ------------------------------------------------------------------ separable interior solve
// Heat on the structured mesh: every subdomain interior is the same mx x my grid and
//   A_ii = K1x (x) M1y + M1x (x) K1y + mc M1x (x) M1y        (Q1 on squares, exact)
// with K1 = tridiag(-1, 2, -1)/h, M1 = h tridiag(1, 4, 1)/6 on mx (my) interior nodes.  Both
// are diagonalised by the orthonormal, symmetric DST-I matrix S (S S = I), so
//   A_ii^-1 X = Sy ((Sy X Sx) ./ D) Sx,   D[j][i] = nu_y,j ka_x,i + ka_y,j nu_x,i + mc nu_y,j nu_x,i
// (fast diagonalisation: an exact direct solve).  One CTA per subdomain; the four real
// 32 x 32 x 32 products per plane run on the FP64 tensor cores (mma.sync m8n8k4): each
// warp owns one 8-row block and two 8-column blocks of both the real and the imaginary
// plane, so the division by D happens on the accumulator fragments.
__device__ __forceinline__ void fdm_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
constexpr int FDM_LD = 36;  // padded row of a 32 x 32 plane in shared memory
#ifndef FETIGPU_FDM_MINB
#define FETIGPU_FDM_MINB 3  // (80 registers: 3 CTAs per SM; measured 32.6 -> 29.6 us)
#endif
__global__ void __launch_bounds__(256, FETIGPU_FDM_MINB) k_fdm_solve(double2* __restrict__ X, size_t ldx, int mx, int my,
                                                   const double* __restrict__ Sx, const double* __restrict__ Sy,
                                                   const double2* __restrict__ invD,
                                                   const double2* __restrict__ Xin = nullptr) {
  __shared__ double pre[32 * FDM_LD], pim[32 * FDM_LD], qre[32 * FDM_LD], qim[32 * FDM_LD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double2* x = X + (size_t)blockIdx.x * ldx;
  const double2* xin = Xin != nullptr ? Xin + (size_t)blockIdx.x * ldx : x;  // out of place when given
  const int n = mx * my;
  pdl_trigger();
  pdl_wait();
  {  // all four loads of a thread in flight together
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u, j = e >> 5, i = e & 31;
      v[u] = (j < my && i < mx) ? xin[j * mx + i] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u, j = e >> 5, i = e & 31;
      pre[j * FDM_LD + i] = v[u].x;
      pim[j * FDM_LD + i] = v[u].y;
    }
  }
  __syncthreads();
  const int rb = (warp & 3) * 8, cb = (warp >> 2) * 16;  // rows rb..rb+7, columns cb..cb+15
  double cr[2][2], ci[2][2];
  // left product: C = Sy P (A = Sy, B = P)
  auto left = [&](const double* Pr, const double* Pi) {
#pragma unroll
    for (int q = 0; q < 2; ++q) cr[q][0] = cr[q][1] = ci[q][0] = ci[q][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      const double a = __ldg(Sy + (rb + g) * 32 + k0 + t);  // (8 KB, L1-resident)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        fdm_dmma(cr[q][0], cr[q][1], a, Pr[(k0 + t) * FDM_LD + cb + 8 * q + g]);
        fdm_dmma(ci[q][0], ci[q][1], a, Pi[(k0 + t) * FDM_LD + cb + 8 * q + g]);
      }
    }
  };
  // right product: C = P Sx (A = P, B = Sx)
  auto right = [&](const double* Pr, const double* Pi) {
#pragma unroll
    for (int q = 0; q < 2; ++q) cr[q][0] = cr[q][1] = ci[q][0] = ci[q][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      const double ar = Pr[(rb + g) * FDM_LD + k0 + t], ai = Pi[(rb + g) * FDM_LD + k0 + t];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double b = __ldg(Sx + (k0 + t) * 32 + cb + 8 * q + g);
        fdm_dmma(cr[q][0], cr[q][1], ar, b);
        fdm_dmma(ci[q][0], ci[q][1], ai, b);
      }
    }
  };
  auto store = [&](double* Qr, double* Qi) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        Qr[(rb + g) * FDM_LD + cb + 8 * q + 2 * t + e] = cr[q][e];
        Qi[(rb + g) * FDM_LD + cb + 8 * q + 2 * t + e] = ci[q][e];
      }
  };
  left(pre, pim);
  store(qre, qim);
  __syncthreads();
  right(qre, qim);
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int e = 0; e < 2; ++e) {  // divide by D (zero in the padding)
      const double2 d = invD[(rb + g) * 32 + cb + 8 * q + 2 * t + e];
      const double a = cr[q][e], b = ci[q][e];
      cr[q][e] = a * d.x - b * d.y;
      ci[q][e] = a * d.y + b * d.x;
    }
  store(pre, pim);
  __syncthreads();
  left(pre, pim);
  store(qre, qim);
  __syncthreads();
  right(qre, qim);
  store(pre, pim);
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += 256) {
    const int j = e / mx, i = e - j * mx;
    x[e] = make_double2(pre[j * FDM_LD + i], pim[j * FDM_LD + i]);
  }
}

// y = ybar - v ; u = lam / phi ; lam = Re t ; leak partial
__global__ void k_realify(int n, const double2* __restrict__ t, double* __restrict__ lam) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) lam[k] = t[k].x;
}
// lambda = Re t and u = lambda / phi (control.cpp:325) in one pass
__global__ void k_realify_u(int n, const double2* __restrict__ t, double inv_phi, double* __restrict__ lam,
                            double* __restrict__ u) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double l = t[k].x;
  lam[k] = l;
  u[k] = l * inv_phi;
}
__global__ void k_recover_y(int n, const double* __restrict__ ybar, const double* __restrict__ vk,
                            double* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[k] = ybar[k] - vk[k];
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
// lambda = Re t, u = lambda / phi (control.cpp:318-325) and, in the same pass, the block maxima
// of |Im t| (imag_leak) and |Re t| (|lambda|_inf of the leak warning): part[blk] = (max|Im|, max|Re|)
__global__ void __launch_bounds__(256) k_realify_stats(int n, const double2* __restrict__ t, double inv_phi,
                                                       double* __restrict__ lam, double* __restrict__ u,
                                                       double2* __restrict__ part) {
  __shared__ double2 sm[8];
  double mi = 0.0, mr = 0.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const double2 v = t[k];
    lam[k] = v.x;
    u[k] = v.x * inv_phi;
    mi = fmax(mi, fabs(v.y));
    mr = fmax(mr, fabs(v.x));
  }
  mi = warp_max(mi);
  mr = warp_max(mr);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = make_double2(mi, mr);
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 m = sm[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = make_double2(fmax(m.x, sm[w].x), fmax(m.y, sm[w].y));
    part[blockIdx.x] = m;
  }
}
// out[0] = (0, max_b part[b].x), out[1] = (0, max_b part[b].y); one warp
__global__ void __launch_bounds__(32) k_max2_final(int nblk, const double2* __restrict__ part, double2* __restrict__ out) {
  double a = 0.0, b = 0.0;
  for (int k = threadIdx.x; k < nblk; k += 32) {
    const double2 v = part[k];
    a = fmax(a, v.x);
    b = fmax(b, v.y);
  }
  a = warp_max(a);
  b = warp_max(b);
  if (threadIdx.x == 0) {
    out[0] = make_double2(0.0, a);
    out[1] = make_double2(0.0, b);
  }
}
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
