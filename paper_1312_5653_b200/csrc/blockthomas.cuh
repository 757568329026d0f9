// blockthomas.cuh — block-tridiagonal ("block Thomas") interior solve x = A_ii^-1 b, the
// per-solve replacement of the banded substitution (K5) when the band half-width W <= 32.
//
// A band matrix with W <= 32 is block tridiagonal in 32 x 32 blocks:
//   A = tridiag(B_k, A_kk, B_{k+1}^T),  B_k = A[block k, block k-1] (upper triangular part of
//   the band).  Block LDL^T:  D_0 = A_00,  D_k = A_kk - B_k D_{k-1}^-1 B_k^T, and
//   forward   z_k = b_k - B_k w_{k-1},   w_k = D_k^-1 z_k
//   backward  x_{m-1} = w_{m-1},          x_k = w_k - D_k^-1 B_{k+1}^T x_{k+1}.
// The pivot blocks D_k (complex symmetric with a positive definite Hermitian part, since
// Re A = K_ii is SPD: Schur complements keep it) are inverted explicitly at setup and kept in
// the packed symmetric 32 x 32 "diagonal tile" format of the Dirichlet GEMV (17 x 32 entries);
// B_k keeps only its structural nonzeros (<= BT_E per row, ELL, both orientations).
//
// Why: the banded substitution is a 2 n_i-step serial chain per subdomain (one pivot per
// step) and runs at the chain's latency, not at HBM speed.  Here the chain has 2 n_i / 32
// block steps, each a 32-wide symmetric GEMV done by one warp, so the solve becomes
// bandwidth-bound; the bytes streamed are 2 x (Dinv + B) ~= 0.66 MB per 961-row interior
// versus 2 x 0.51 MB of band factor.
//
// Record per block k (double2 units), streamed by 1-D TMA bulk copies into a smem ring:
//   [Bf_idx 8 | Bf_val 128 | Dinv 544 | Bb_val 128 | Bb_idx 8]   (Bf: gather rows of block k
//   from block k-1; Bb: gather rows of block k from block k+1, i.e. B_{k+1}^T).
// The forward sweep copies the first BT_HALF entries, the backward sweep the last BT_HALF.
#pragma once

#include "common.cuh"

namespace fetigpu {

constexpr int BT_Q = 32, BT_E = 4;
constexpr int BT_OFF_BF_IDX = 0, BT_OFF_BF_VAL = 8, BT_OFF_D = 136, BT_OFF_BB_VAL = 680, BT_OFF_BB_IDX = 808;
constexpr int BT_REC = 816, BT_HALF = 680;

// ---------------------------------------------------------------------------------------
// Setup: one CTA per subdomain, the block recursion in shared memory.  colband holds the
// lower band of A_ii (colband[j][d] = A(j + d, j), d <= W) BEFORE the band factorization.
// status[s] = 0 ok, 1 + k singular / non-finite pivot block k, -1 a B row with > BT_E nonzeros.
__global__ void __launch_bounds__(256) k_bt_factor(const double2* __restrict__ colband, size_t band_stride, int W,
                                                   int NI, int nb, double2* __restrict__ recs,
                                                   int* __restrict__ status) {
  extern __shared__ double2 bt_sh[];
  double2 (*D)[33] = reinterpret_cast<double2 (*)[33]>(bt_sh);
  double2 (*P)[33] = reinterpret_cast<double2 (*)[33]>(bt_sh + 32 * 33);
  double2 (*B)[33] = reinterpret_cast<double2 (*)[33]>(bt_sh + 2 * 32 * 33);
  double2 (*T)[33] = reinterpret_cast<double2 (*)[33]>(bt_sh + 3 * 32 * 33);
  double2* colp = bt_sh + 4 * 32 * 33;  // [32]
  double2* rowp = colp + 32;            // [32]
  __shared__ int bad;
  const int s = blockIdx.x, tid = threadIdx.x;
  const double2* A = colband + (size_t)s * band_stride;
  const int LD = W + 1;
  double2* R = recs + (size_t)s * nb * BT_REC;
  if (tid == 0) bad = 0;
  for (int k = 0; k < nb; ++k) {
    double2* rec = R + (size_t)k * BT_REC;
    // A_kk and B_k from the band
    for (int idx = tid; idx < 1024; idx += blockDim.x) {
      const int r = idx >> 5, c = idx & 31;
      const int gr = k * BT_Q + r, gc = k * BT_Q + c;
      double2 v;
      if (gr >= NI || gc >= NI) {
        v = make_double2(r == c ? 1.0 : 0.0, 0.0);
      } else {
        const int lo = max(gr, gc), hi = min(gr, gc), d = lo - hi;
        v = d <= W ? A[(size_t)hi * LD + d] : cz();
      }
      D[r][c] = v;
      double2 b = cz();
      if (k > 0) {
        const int gb = (k - 1) * BT_Q + c, d = gr - gb;
        if (gr < NI && gb < NI && d <= W) b = A[(size_t)gb * LD + d];
      }
      B[r][c] = b;
    }
    __syncthreads();
    // ELL of B_k (rows of block k <- block k-1) and of B_k^T (rows of block k-1 <- block k)
    if (tid < 32) {
      const int r = tid;
      int e = 0;
      unsigned char* bidx = reinterpret_cast<unsigned char*>(rec + BT_OFF_BF_IDX);
      for (int c = 0; c < 32; ++c) {
        const double2 v = B[r][c];
        if (v.x != 0.0 || v.y != 0.0) {
          if (e < BT_E) {
            rec[BT_OFF_BF_VAL + e * 32 + r] = v;
            bidx[e * 32 + r] = (unsigned char)c;
          }
          ++e;
        }
      }
      if (e > BT_E) bad = -1;
      for (; e < BT_E; ++e) {
        rec[BT_OFF_BF_VAL + e * 32 + r] = cz();
        bidx[e * 32 + r] = (unsigned char)r;
      }
    } else if (tid < 64 && k > 0) {
      const int c = tid - 32;
      double2* prev = R + (size_t)(k - 1) * BT_REC;
      unsigned char* bidx = reinterpret_cast<unsigned char*>(prev + BT_OFF_BB_IDX);
      int e = 0;
      for (int r = 0; r < 32; ++r) {
        const double2 v = B[r][c];
        if (v.x != 0.0 || v.y != 0.0) {
          if (e < BT_E) {
            prev[BT_OFF_BB_VAL + e * 32 + c] = v;
            bidx[e * 32 + c] = (unsigned char)r;
          }
          ++e;
        }
      }
      if (e > BT_E) bad = -1;
      for (; e < BT_E; ++e) {
        prev[BT_OFF_BB_VAL + e * 32 + c] = cz();
        bidx[e * 32 + c] = (unsigned char)c;
      }
    }
    if (k > 0) {  // D -= B P B^T  (T = P B^T first)
      for (int idx = tid; idx < 1024; idx += blockDim.x) {
        const int i = idx >> 5, r = idx & 31;
        double2 acc = cz();
#pragma unroll 8
        for (int c = 0; c < 32; ++c) acc = cfma(P[i][c], B[r][c], acc);
        T[i][r] = acc;
      }
      __syncthreads();
      for (int idx = tid; idx < 1024; idx += blockDim.x) {
        const int r = idx >> 5, j = idx & 31;
        double2 acc = D[r][j];
#pragma unroll 8
        for (int i = 0; i < 32; ++i) acc = cfms(B[r][i], T[i][j], acc);
        D[r][j] = acc;
      }
    }
    __syncthreads();
    // in-place Gauss-Jordan inverse of D (no pivoting: Hermitian part positive definite)
    for (int p = 0; p < 32; ++p) {
      const double2 dp = D[p][p];
      const double2 piv = crecip(dp);
      if (tid == 0) {
        const double a2 = cabs2(dp);
        if (!(a2 > 0.0) || !isfinite(a2)) bad = bad ? bad : 1 + k;
      }
      if (tid < 32) colp[tid] = D[tid][p];
      else if (tid < 64) rowp[tid - 32] = (tid - 32 == p) ? piv : cmul(D[p][tid - 32], piv);
      __syncthreads();
      for (int idx = tid; idx < 1024; idx += blockDim.x) {
        const int i = idx >> 5, j = idx & 31;
        if (i == p) {
          D[i][j] = rowp[j];
        } else if (j == p) {
          const double2 f = colp[i];
          D[i][j] = make_double2(-(f.x * piv.x - f.y * piv.y), -(f.x * piv.y + f.y * piv.x));
        } else {
          D[i][j] = cfms(colp[i], rowp[j], D[i][j]);
        }
      }
      __syncthreads();
    }
    // packed symmetric Dinv (entry (l, l + c) at c * 32 + l, c = 0..16), and P = Dinv
    for (int idx = tid; idx < 17 * 32; idx += blockDim.x) {
      const int c = idx >> 5, l = idx & 31;
      rec[BT_OFF_D + idx] = D[l][(l + c) & 31];
    }
    for (int idx = tid; idx < 1024; idx += blockDim.x) P[idx >> 5][idx & 31] = D[idx >> 5][idx & 31];
    if (k == nb - 1 && tid < 32) {  // no block below the last one
      unsigned char* bidx = reinterpret_cast<unsigned char*>(rec + BT_OFF_BB_IDX);
      for (int e = 0; e < BT_E; ++e) {
        rec[BT_OFF_BB_VAL + e * 32 + tid] = cz();
        bidx[e * 32 + tid] = (unsigned char)tid;
      }
    }
    __syncthreads();
  }
  if (tid == 0) status[s] = bad;
}

constexpr size_t bt_factor_smem() { return sizeof(double2) * (4 * 32 * 33 + 64); }

// y = D z for one packed symmetric 32 x 32 block D (diagonal-tile format), one warp
__device__ __forceinline__ double2 bt_symv(const double2* __restrict__ Dp, double2 z, double2* zsh, int lane) {
  zsh[lane] = z;
  __syncwarp();
  double2 yr = cmul(Dp[lane], z), yc = cz();
#pragma unroll
  for (int c = 1; c < 16; ++c) {
    const double2 m = Dp[c * 32 + lane];
    yr = cfma(m, zsh[(lane + c) & 31], yr);
    yc = shfl2(yc, (lane + 1) & 31);  // carry column (l + c + 1) into lane l
    yc = cfma(m, z, yc);
  }
  yr = cfma(Dp[16 * 32 + lane], zsh[(lane + 16) & 31], yr);
  yc = shfl2(yc, (lane + 17) & 31);  // lane l <- column l
  __syncwarp();
  return cadd(yr, yc);
}

// ---------------------------------------------------------------------------------------
// Per-solve: one warp per subdomain, in place on X (one right-hand side per subdomain).
// Block records stream through a STAGES-deep smem ring of 1-D TMA bulk copies.
template <int STAGES>
__global__ void __launch_bounds__(32) k_bt_solve(const double2* __restrict__ recs, int nb, int NI,
                                                 double2* __restrict__ X, size_t x_stride) {
  extern __shared__ __align__(128) unsigned char bt_raw[];
  double2* stage = reinterpret_cast<double2*>(bt_raw);
  double2* zsh = stage + (size_t)STAGES * BT_HALF;
  uint64_t* full = reinterpret_cast<uint64_t*>(zsh + 32);
  const int s = blockIdx.x, lane = threadIdx.x;
  const double2* R = recs + (size_t)s * nb * BT_REC;
  double2* x = X + (size_t)s * x_stride;
  const int total = 2 * nb - 1;
  constexpr uint32_t BYTES = BT_HALF * sizeof(double2);
  // q < nb: forward block q (record head); q >= nb: backward block 2 nb - 2 - q (record tail)
  auto src = [&](int q) -> const double2* {
    return q < nb ? R + (size_t)q * BT_REC : R + (size_t)(2 * nb - 2 - q) * BT_REC + BT_OFF_D;
  };
  if (lane == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0) {
    for (int q = 0; q < STAGES && q < total; ++q) {
      mbar_arrive_expect_tx(&full[q], BYTES);
      tma_load_1d(stage + (size_t)q * BT_HALF, src(q), BYTES, &full[q]);
    }
  }
  auto refill = [&](int q, int st) {
    __syncwarp();
    if (lane == 0 && q + STAGES < total) {
      mbar_arrive_expect_tx(&full[st], BYTES);
      tma_load_1d(stage + (size_t)st * BT_HALF, src(q + STAGES), BYTES, &full[st]);
    }
  };
  // ---- forward: z_k = b_k - B_k w_{k-1}, w_k = D_k^-1 z_k (w stored in place) ----
  double2 wprev = cz();
  double2 bcur = lane < NI ? x[lane] : cz();
  for (int k = 0; k < nb; ++k) {
    const int st = k % STAGES;
    const int rn = (k + 1) * BT_Q + lane;
    const double2 bnext = (k + 1 < nb && rn < NI) ? x[rn] : cz();
    mbar_wait(&full[st], (uint32_t)(k / STAGES) & 1u);
    const double2* rec = stage + (size_t)st * BT_HALF;
    const unsigned char* bidx = reinterpret_cast<const unsigned char*>(rec + BT_OFF_BF_IDX);
    double2 z = bcur;
#pragma unroll
    for (int e = 0; e < BT_E; ++e) z = cfms(rec[BT_OFF_BF_VAL + e * 32 + lane], shfl2(wprev, bidx[e * 32 + lane]), z);
    const double2 w = bt_symv(rec + BT_OFF_D, z, zsh, lane);
    if (k * BT_Q + lane < NI) x[k * BT_Q + lane] = w;
    wprev = w;
    bcur = bnext;
    refill(k, st);
  }
  // ---- backward: x_k = w_k - D_k^-1 (B_{k+1}^T x_{k+1}) ----
  double2 xnext = wprev;
  for (int k = nb - 2; k >= 0; --k) {
    const int q = 2 * nb - 2 - k, st = q % STAGES;
    const int r = k * BT_Q + lane;
    const double2 wk = r < NI ? x[r] : cz();
    mbar_wait(&full[st], (uint32_t)(q / STAGES) & 1u);
    const double2* rec = stage + (size_t)st * BT_HALF;  // [Dinv | Bb_val | Bb_idx]
    const unsigned char* bidx = reinterpret_cast<const unsigned char*>(rec + (BT_OFF_BB_IDX - BT_OFF_D));
    double2 t = cz();
#pragma unroll
    for (int e = 0; e < BT_E; ++e)
      t = cfma(rec[(BT_OFF_BB_VAL - BT_OFF_D) + e * 32 + lane], shfl2(xnext, bidx[e * 32 + lane]), t);
    const double2 y = bt_symv(rec, t, zsh, lane);
    const double2 xk = csub(wk, y);
    if (r < NI) x[r] = xk;
    xnext = xk;
    refill(q, st);
  }
}

template <int STAGES>
constexpr size_t bt_solve_smem() {
  return sizeof(double2) * ((size_t)STAGES * BT_HALF + 32) + sizeof(uint64_t) * STAGES;
}

}  // namespace fetigpu
