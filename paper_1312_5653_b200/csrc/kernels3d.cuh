// kernels3d.cuh — sm_100a kernels of the 3D FETI-DP(H) path (fetigpu3d.cu).
//
// Per-subdomain operators (natural local order, SURVEY.md §8a a4 restated for hexahedra):
//   A_ii  block-banded in 32x32 blocks: block (K, K-d), d = 0..P, at bb[s][K][d]; after the
//         block LDL^T (k3_bb_factor) bb[s][K][0] = D_K^-1 and bb[s][K][d] = L_{K,K-d}
//   A_bi / A_ib  ELL rows;  A_ic, A_bc, A_cc dense (<= 24 corner dofs per subdomain)
//   S_bb = A_bb - A_bi A_ii^-1 A_ib and S_bb^-1, dense at setup (chunks of subdomains),
//         then packed symmetric in 32x32 tiles for the per-iteration GEMVs
// Every 32x32 tile is stored "diagonal-major": entry (r, c) at ((c - r) & 31) * 32 + r, so a
// warp's load of one 512 B row of storage gives lane l the element (l, l + cc): the row
// product sum_c T[l][c] x[c] and the transposed product (rotating shuffle carry) are both
// coalesced.  Diagonal tiles of the symmetric packs keep only cc = 0..16 (17 x 32).
#pragma once

#include "common.cuh"

namespace fetigpu {
namespace k3 {

__device__ __forceinline__ int tpos(int r, int c) { return (((c - r) & 31) << 5) | r; }
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------------------
// Assembly (K1): one thread per (subdomain, local mesh dof) row; the row owner adds every
// element contribution of its row into the block it belongs to (deterministic, no atomics).
struct Asm3 {
  int S, nld, ex, ey, ez, dpn, ed;
  int NI, NB, NC, P, EBI, EIB;
  const int* ldof;        // [S][nld]
  const double2* ae;      // [ed][ed] element matrix K_e + c M_e
  double2* bb;            // [S][NI/32][P+1][1024]
  int* bi_idx;            // [S][NB][EBI]
  double2* bi_val;
  int* ib_idx;            // [S][NI][EIB]
  double2* ib_val;
  double2* aic;           // [S][NI][NC]
  double2* abc;           // [S][NB][NC]
  double2* acc;           // [S][NC][NC]
  // mode 1: only A_bb of subdomains [s0, s0 + cnt) into dense [s - s0][NBP][NBP]
  int mode, s0, cnt, NBP;
  double2* dense;
};

__device__ __forceinline__ void ell_add(int* idx, double2* val, int width, int key, double2 v) {
  for (int e = 0; e < width; ++e) {
    const int k = idx[e];
    if (k == key) {
      val[e] = cadd(val[e], v);
      return;
    }
    if (k < 0) {
      idx[e] = key;
      val[e] = v;
      return;
    }
  }
}

__global__ void k3_assemble(Asm3 a) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nsub = a.mode == 0 ? a.S : a.cnt;
  if (gid >= (long long)nsub * a.nld) return;
  const int s = (a.mode == 0 ? 0 : a.s0) + (int)(gid / a.nld);
  const int l = (int)(gid % a.nld);
  const int* ld = a.ldof + (size_t)s * a.nld;
  const int code = ld[l], cat = code >> 24, row = code & 0xFFFFFF;
  if (cat == 0) return;
  if (a.mode == 1 && cat != 3) return;
  const int dpn = a.dpn, lx = a.ex + 1, ly = a.ey + 1;
  const int c = l % dpn, node = l / dpn;
  const int li = node % lx, lj = (node / lx) % ly, lk = node / (lx * ly);
  const int hx[8] = {0, 1, 1, 0, 0, 1, 1, 0}, hy[8] = {0, 0, 1, 1, 0, 0, 1, 1};
  for (int ek = max(lk - 1, 0); ek <= min(lk, a.ez - 1); ++ek)
    for (int ej = max(lj - 1, 0); ej <= min(lj, a.ey - 1); ++ej)
      for (int ei = max(li - 1, 0); ei <= min(li, a.ex - 1); ++ei) {
        const int dx = li - ei, dy = lj - ej, dz = lk - ek;
        const int an = dz * 4 + (dy == 0 ? dx : 3 - dx);  // local node of this dof in the element
        for (int b = 0; b < 8; ++b) {
          const int nb = ((ek + (b >> 2)) * ly + (ej + hy[b])) * lx + (ei + hx[b]);
          for (int c2 = 0; c2 < dpn; ++c2) {
            const int code2 = ld[nb * dpn + c2], cat2 = code2 >> 24, col = code2 & 0xFFFFFF;
            if (cat2 == 0) continue;
            const double2 v = a.ae[(an * dpn + c) * a.ed + b * dpn + c2];
            if (a.mode == 1) {
              if (cat2 == 3) {
                double2* d = a.dense + ((size_t)(s - a.s0) * a.NBP + row) * a.NBP + col;
                *d = cadd(*d, v);
              }
              continue;
            }
            if (cat == 1) {  // corner row
              if (cat2 == 1) {
                double2* d = a.acc + ((size_t)s * a.NC + row) * a.NC + col;
                *d = cadd(*d, v);
              }
            } else if (cat == 2) {  // interior row
              if (cat2 == 2) {
                const int K = row >> 5, d = K - (col >> 5);
                if (d >= 0 && d <= a.P) {
                  double2* t = a.bb + (((size_t)s * (a.NI >> 5) + K) * (a.P + 1) + d) * 1024 + tpos(row & 31, col & 31);
                  *t = cadd(*t, v);
                }
              } else if (cat2 == 3) {
                const size_t r0 = ((size_t)s * a.NI + row) * a.EIB;
                ell_add(a.ib_idx + r0, a.ib_val + r0, a.EIB, col, v);
              } else {
                double2* d = a.aic + ((size_t)s * a.NI + row) * a.NC + col;
                *d = cadd(*d, v);
              }
            } else {  // interface row
              if (cat2 == 2) {
                const size_t r0 = ((size_t)s * a.NB + row) * a.EBI;
                ell_add(a.bi_idx + r0, a.bi_val + r0, a.EBI, col, v);
              } else if (cat2 == 1) {
                double2* d = a.abc + ((size_t)s * a.NB + row) * a.NC + col;
                *d = cadd(*d, v);
              }
            }
          }
        }
      }
}

// identity on the padded interior rows (n_i <= i < NI) so every block row is regular
__global__ void k3_pad_identity(int S, int NI, int P, const int* __restrict__ n_i, double2* bb) {
  const int s = blockIdx.x;
  for (int i = n_i[s] + threadIdx.x; i < NI; i += blockDim.x)
    bb[(((size_t)s * (NI >> 5) + (i >> 5)) * (P + 1)) * 1024 + tpos(i & 31, i & 31)] = make_double2(1.0, 0.0);
}

// ---------------------------------------------------------------------------------------
// 32x32 complex block helpers for 256-thread CTAs.  Shared tiles are row-major [32][33].
typedef double2 Tile[32][33];

__device__ __forceinline__ void tile_load(Tile& t, const double2* __restrict__ g) {  // g in tpos layout
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    const int cc = e >> 5, r = e & 31;
    t[r][(r + cc) & 31] = g[e];
  }
}
__device__ __forceinline__ void tile_store(double2* __restrict__ g, const Tile& t) {
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    const int cc = e >> 5, r = e & 31;
    g[e] = t[r][(r + cc) & 31];
  }
}
// dense row-major block (leading dimension ld) <-> shared tile
__device__ __forceinline__ void tile_load_rm(Tile& t, const double2* __restrict__ g, size_t ld) {
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) t[e >> 5][e & 31] = g[(size_t)(e >> 5) * ld + (e & 31)];
}
__device__ __forceinline__ void tile_store_rm(double2* __restrict__ g, size_t ld, const Tile& t) {
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) g[(size_t)(e >> 5) * ld + (e & 31)] = t[e >> 5][e & 31];
}
// acc[q] (rows r, cols c0..c0+3 of the owning thread) of A B (TB = false) or A B^T (TB = true)
template <bool TB>
__device__ __forceinline__ void tile_mma(const Tile& A, const Tile& B, double2 acc[4]) {
  const int r = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    const double2 a = A[r][k];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = cfma(a, TB ? B[c0 + q][k] : B[k][c0 + q], acc[q]);
  }
}
// in-place inverse of a shared 32x32 tile by Gauss-Jordan without pivoting (complex
// symmetric with positive definite real part: every leading pivot is nonzero); returns the
// smallest |pivot| relative to the largest in *pivrat (thread 0)
__device__ void tile_invert(Tile& t, double* pivrat) {
  __shared__ double2 prow[32], pcol[32];
  __shared__ double pmin, pmax;
  if (threadIdx.x == 0) pmin = 1e300, pmax = 0.0;
  __syncthreads();
  for (int p = 0; p < 32; ++p) {
    const double2 piv = t[p][p];
    const double2 pinv = crecip(piv);
    if (threadIdx.x < 32) {
      const int c = threadIdx.x;
      prow[c] = c == p ? pinv : cmul(t[p][c], pinv);
      pcol[c] = c == p ? cz() : t[c][p];
    }
    if (threadIdx.x == 0) {
      const double a = sqrt(cabs2(piv));
      pmin = fmin(pmin, a);
      pmax = fmax(pmax, a);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int r = e >> 5, c = e & 31;
      if (r == p) {
        t[r][c] = prow[c];
      } else {
        const double2 base = c == p ? cz() : t[r][c];
        t[r][c] = cfms(pcol[r], prow[c], base);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *pivrat = pmax > 0.0 ? pmin / pmax : 0.0;
}

// ---------------------------------------------------------------------------------------
// K2: block LDL^T of A_ii (right-looking, one CTA of 256 threads per subdomain).  For each
// block column K: D_K^-1 (in-tile Gauss-Jordan), L_IK = Abar_IK D_K^-1, trailing update
// A_IJ -= Abar_IK L_JK^T (K < J <= I <= K+P), then L replaces Abar.  Scratch: [S][P][1024].
__global__ void __launch_bounds__(256) k3_bb_factor(int NBK, int P, double2* __restrict__ bb,
                                                    double2* __restrict__ scratch, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char k3f_raw[];
  Tile& A = *reinterpret_cast<Tile*>(k3f_raw);
  Tile& B = *reinterpret_cast<Tile*>(k3f_raw + sizeof(Tile));
  const int s = blockIdx.x;
  double2* band = bb + (size_t)s * NBK * (P + 1) * 1024;
  double2* Lc = scratch + (size_t)s * P * 1024;
  __shared__ double rat;
  double worst = 1.0;
  for (int K = 0; K < NBK; ++K) {
    double2* blkKK = band + ((size_t)K * (P + 1)) * 1024;
    tile_load(A, blkKK);
    __syncthreads();
    tile_invert(A, &rat);
    __syncthreads();
    worst = fmin(worst, rat);
    tile_store(blkKK, A);  // D_K^-1
    const int nd = min(P, NBK - 1 - K);
    // L_dI = Abar_dI D^-1
    for (int dI = 1; dI <= nd; ++dI) {
      __syncthreads();
      tile_load(B, band + ((size_t)(K + dI) * (P + 1) + dI) * 1024);
      __syncthreads();
      double2 acc[4] = {cz(), cz(), cz(), cz()};
      tile_mma<false>(B, A, acc);
      const int r = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) Lc[(size_t)(dI - 1) * 1024 + tpos(r, c0 + q)] = acc[q];
    }
    __syncthreads();
    // trailing update: block (K+dI, K+dJ) -= Abar_dI L_dJ^T
    for (int dI = 1; dI <= nd; ++dI) {
      __syncthreads();
      tile_load(A, band + ((size_t)(K + dI) * (P + 1) + dI) * 1024);  // Abar (still unscaled)
      for (int dJ = 1; dJ <= dI; ++dJ) {
        __syncthreads();
        tile_load(B, Lc + (size_t)(dJ - 1) * 1024);
        __syncthreads();
        double2 acc[4] = {cz(), cz(), cz(), cz()};
        tile_mma<true>(A, B, acc);
        double2* tgt = band + ((size_t)(K + dI) * (P + 1) + (dI - dJ)) * 1024;
        const int r = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = tpos(r, c0 + q);
          tgt[p] = csub(tgt[p], acc[q]);
        }
      }
    }
    __syncthreads();
    for (int dI = 1; dI <= nd; ++dI)
      for (int e = threadIdx.x; e < 1024; e += blockDim.x)
        band[((size_t)(K + dI) * (P + 1) + dI) * 1024 + e] = Lc[(size_t)(dI - 1) * 1024 + e];
    __syncthreads();
  }
  if (threadIdx.x == 0) status[s] = (worst > 1e-14) ? 0 : 1;
}

// The same block LDL^T with every block column K spread over the whole grid (4 launches per
// K, all subdomains at once): pivot inverse (CTA per subdomain), L blocks (CTA per (d, s)),
// trailing update (CTA per (dI, dJ, s)), write-back of L.  Used when the subdomains are
// too few to fill the GPU one CTA each (config 5: 64 subdomains, P = 26).
__global__ void __launch_bounds__(256) k3_bbf_pivot(int NBK, int P, int K, double2* __restrict__ bb,
                                                    int* __restrict__ status) {
  __shared__ Tile A;
  __shared__ double rat;
  const int s = blockIdx.x;
  double2* blk = bb + (((size_t)s * NBK + K) * (P + 1)) * 1024;
  tile_load(A, blk);
  __syncthreads();
  tile_invert(A, &rat);
  __syncthreads();
  tile_store(blk, A);
  if (threadIdx.x == 0 && !(rat > 1e-14)) status[s] = 1;
}
__global__ void __launch_bounds__(256) k3_bbf_lcol(int NBK, int P, int K, const double2* __restrict__ bb,
                                                   double2* __restrict__ scratch) {
  __shared__ Tile A, D;
  const int dI = blockIdx.x + 1, s = blockIdx.y;
  const double2* band = bb + (size_t)s * NBK * (P + 1) * 1024;
  tile_load(D, band + ((size_t)K * (P + 1)) * 1024);
  tile_load(A, band + ((size_t)(K + dI) * (P + 1) + dI) * 1024);
  __syncthreads();
  double2 acc[4] = {cz(), cz(), cz(), cz()};
  tile_mma<false>(A, D, acc);
  const int r = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
  double2* L = scratch + ((size_t)s * P + (dI - 1)) * 1024;
#pragma unroll
  for (int q = 0; q < 4; ++q) L[tpos(r, c0 + q)] = acc[q];
}
__global__ void __launch_bounds__(256) k3_bbf_update(int NBK, int P, int K, double2* __restrict__ bb,
                                                     const double2* __restrict__ scratch) {
  __shared__ Tile A, B;
  // pair index -> (dI, dJ), 1 <= dJ <= dI
  const int t = blockIdx.x, s = blockIdx.y;
  int dI = (int)((sqrt(8.0 * t + 1.0) - 1.0) / 2.0) + 1;
  while (dI * (dI - 1) / 2 > t) --dI;
  while ((dI + 1) * dI / 2 <= t) ++dI;
  const int dJ = t - dI * (dI - 1) / 2 + 1;
  double2* band = bb + (size_t)s * NBK * (P + 1) * 1024;
  tile_load(A, band + ((size_t)(K + dI) * (P + 1) + dI) * 1024);
  tile_load(B, scratch + ((size_t)s * P + (dJ - 1)) * 1024);
  __syncthreads();
  double2 acc[4] = {cz(), cz(), cz(), cz()};
  tile_mma<true>(A, B, acc);
  double2* tgt = band + ((size_t)(K + dI) * (P + 1) + (dI - dJ)) * 1024;
  const int r = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int p = tpos(r, c0 + q);
    tgt[p] = csub(tgt[p], acc[q]);
  }
}
__global__ void k3_bbf_store(int NBK, int P, int K, double2* __restrict__ bb, const double2* __restrict__ scratch) {
  const int dI = blockIdx.x + 1, s = blockIdx.y;
  double2* dst = bb + (((size_t)s * NBK + K + dI) * (P + 1) + dI) * 1024;
  const double2* src = scratch + ((size_t)s * P + (dI - 1)) * 1024;
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) dst[e] = src[e];
}


// Interior block-band substitution (K5 eliminate, 4 per Schur solve): a producer warp streams
// every 16 KB block of the substitution, in consumption order, through a STAGES-deep shared-memory ring (1-D bulk
// copies, full/empty mbarrier pairs), so the block loads run ahead of the recurrence and the
// bytes in flight no longer depend on the consumers' progress.  Item order: forward
// K = 0..: the blocks (K, K-d), d = 1..min(P,K), then D_K^-1; backward K = NBK-1..0: the
// blocks (K+d, K), d = 1..min(P, NBK-1-K).  Item j always goes to consumer warp j % W
// (W divides STAGES), so every ring slot is waited on by one warp in phase order (a warp
// never waits on round r+1 of a slot before round r completed — the parity would alias).
// Each warp keeps a partial of the step; the warp that owns D_K^-1 closes the step.
template <int STAGES, int W>
__global__ void __launch_bounds__((W + 1) * 32, 1) k3_bb_solve_tma(int NBK, int P, const double2* __restrict__ bb,
                                                                   int NI, double2* __restrict__ X) {
  static_assert(STAGES % W == 0, "slot -> warp must be fixed");
  extern __shared__ __align__(128) unsigned char k3t_raw[];
  double2* ring = reinterpret_cast<double2*>(k3t_raw);                                    // [STAGES][1024]
  double2 (*yr)[32] = reinterpret_cast<double2 (*)[32]>(ring + (size_t)STAGES * 1024);     // [33][32]
  double2 (*part)[32] = yr + 33;                                                          // [W][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(part + W);
  uint64_t* empty = full + STAGES;
  const int s = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* band = bb + (size_t)s * NBK * (P + 1) * 1024;
  double2* x = X + (size_t)s * NI;
  if (threadIdx.x == 0) {
    for (int q = 0; q < STAGES; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  constexpr uint32_t BYTES = 1024 * sizeof(double2);
  if (warp == W) {  // ---- producer ----
    if (lane == 0) {
      long long i = 0;
      auto issue = [&](const double2* src) {
        const int st = (int)(i % STAGES);
        const uint32_t round = (uint32_t)(i / STAGES);
        if (round > 0) mbar_wait(&empty[st], (round - 1) & 1u);
        mbar_arrive_expect_tx(&full[st], BYTES);
        tma_load_1d(ring + (size_t)st * 1024, src, BYTES, &full[st]);
        ++i;
      };
      for (int K = 0; K < NBK; ++K) {
        for (int d = 1; d <= P && K - d >= 0; ++d) issue(band + ((size_t)K * (P + 1) + d) * 1024);
        issue(band + ((size_t)K * (P + 1)) * 1024);
      }
      for (int K = NBK - 1; K >= 0; --K)
        for (int d = 1; d <= P && K + d < NBK; ++d) issue(band + ((size_t)(K + d) * (P + 1) + d) * 1024);
    }
    return;
  }
  // ---- consumers ----
  auto consume = [&](long long item) -> const double2* {
    mbar_wait(&full[item % STAGES], (uint32_t)(item / STAGES) & 1u);
    return ring + (size_t)(item % STAGES) * 1024;
  };
  auto release = [&](long long item) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[item % STAGES]);
  };
  // first item of this warp at or after `base`
  auto first_mine = [&](long long base) { return base + (((long long)warp - base % W) % W + W) % W; };
  long long base = 0;
  for (int K = 0; K < NBK; ++K) {
    const int nd = min(P, K);
    double2 acc = cz();
    for (long long it = first_mine(base); it < base + nd; it += W) {
      const int d = (int)(it - base) + 1;
      const double2* T = consume(it);
      const double2* y = yr[(K - d) % 33];
#pragma unroll 8
      for (int cc = 0; cc < 32; ++cc) acc = cfma(T[cc * 32 + lane], y[(lane + cc) & 31], acc);
      release(it);
    }
    part[warp][lane] = acc;
    named_bar_sync(1, W * 32);
    const long long itd = base + nd;  // D_K^-1: its warp closes the step
    if (warp == (int)(itd % W)) {
      double2 v = x[(size_t)K * 32 + lane];
      for (int w = 0; w < W; ++w) v = csub(v, part[w][lane]);
      yr[K % 33][lane] = v;
      __syncwarp();
      const double2* D = consume(itd);
      double2 z = cz();
#pragma unroll 8
      for (int cc = 0; cc < 32; ++cc) z = cfma(D[cc * 32 + lane], yr[K % 33][(lane + cc) & 31], z);
      release(itd);
      x[(size_t)K * 32 + lane] = z;
    }
    named_bar_sync(1, W * 32);
    base += nd + 1;
  }
  for (int K = NBK - 1; K >= 0; --K) {
    const int nd = min(P, NBK - 1 - K);
    double2 acc = cz();
    for (long long it = first_mine(base); it < base + nd; it += W) {
      const int d = (int)(it - base) + 1;
      const double2* T = consume(it);
      const double2 xr = yr[(K + d) % 33][lane];
      double2 yc = cz();
#pragma unroll 8
      for (int cc = 0; cc < 32; ++cc) {
        yc = cfma(T[cc * 32 + lane], xr, yc);
        yc = shfl2(yc, (lane + 1) & 31);
      }
      acc = cadd(acc, yc);
      release(it);
    }
    part[warp][lane] = acc;
    named_bar_sync(1, W * 32);
    if (warp == 0) {
      double2 v = x[(size_t)K * 32 + lane];
      for (int w = 0; w < W; ++w) v = csub(v, part[w][lane]);
      yr[K % 33][lane] = v;
      x[(size_t)K * 32 + lane] = v;
    }
    named_bar_sync(1, W * 32);
    base += nd;
  }
}
template <int STAGES, int W>
constexpr size_t bb_solve_tma_smem() {
  return sizeof(double2) * ((size_t)STAGES * 1024 + 33 * 32 + W * 32) + sizeof(uint64_t) * 2 * STAGES;
}

// Setup multi-RHS substitution, register-blocked (K3): a CTA solves 64 right-hand sides
// (RHS tiles 2t, 2t+1 of [sub][tile][NI][32]) of one subdomain.  Every block product is a
// 32 x 64 x 32 complex GEMM on shared-memory tiles, 256 threads each owning 2 rows x 4
// columns.  Forward values y_K stay in Y until the backward sweep, which forms
// z_K = D_K^-1 y_K and x_K = z_K - sum_d L_{K+d,K}^T x_{K+d} block row by block row.
__device__ __forceinline__ void msv_stage(double2 (*Ls)[33], double2 (*Ys)[65], const double2* __restrict__ T,
                                          const double2* __restrict__ y0, const double2* __restrict__ y1, int two) {
  for (int e = threadIdx.x; e < 1024; e += 256) {
    const int cc = e >> 5, r = e & 31;
    Ls[r][(r + cc) & 31] = T[e];
  }
  for (int e = threadIdx.x; e < 32 * 64; e += 256) {
    const int r = e >> 6, c = e & 63;
    Ys[r][c] = c < 32 ? y0[(size_t)r * 32 + c] : (two ? y1[(size_t)r * 32 + c - 32] : cz());
  }
}
template <bool TRANS>
__device__ __forceinline__ void msv_mma(const double2 (*Ls)[33], const double2 (*Ys)[65], double2 acc[2][4],
                                        bool sub) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    double2 a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = TRANS ? Ls[k][ty * 2 + i] : Ls[ty * 2 + i][k];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Ys[k][tx + 16 * j];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = sub ? cfms(a[i], b[j], acc[i][j]) : cfma(a[i], b[j], acc[i][j]);
  }
}
__global__ void __launch_bounds__(256) k3_bb_msolve2(int NBK, int P, const double2* __restrict__ bb, int NI,
                                                     int ntile, int tile0, int ntiles, int s0,
                                                     double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 k3v_sm[];
  double2 (*Ls)[33] = reinterpret_cast<double2 (*)[33]>(k3v_sm);
  double2 (*Ys)[65] = reinterpret_cast<double2 (*)[65]>(k3v_sm + 32 * 33);
  const int t2 = blockIdx.x, sc = blockIdx.y, s = s0 + sc;
  const int ta = tile0 + 2 * t2, two = (2 * t2 + 1 < ntiles) ? 1 : 0;
  const double2* band = bb + (size_t)s * NBK * (P + 1) * 1024;
  double2* ya = Y + ((size_t)sc * ntile + ta) * NI * 32;
  double2* yb = two ? ya + (size_t)NI * 32 : ya;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  auto load_acc = [&](int K, double2 acc[2][4]) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = K * 32 + ty * 2 + i, c = tx + 16 * j;
        acc[i][j] = c < 32 ? ya[(size_t)r * 32 + c] : (two ? yb[(size_t)r * 32 + c - 32] : cz());
      }
  };
  auto store_acc = [&](int K, double2 acc[2][4]) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = K * 32 + ty * 2 + i, c = tx + 16 * j;
        if (c < 32) ya[(size_t)r * 32 + c] = acc[i][j];
        else if (two) yb[(size_t)r * 32 + c - 32] = acc[i][j];
      }
  };
  // forward: y_K = b_K - sum_d L_{K,K-d} y_{K-d}
  for (int K = 0; K < NBK; ++K) {
    double2 acc[2][4];
    load_acc(K, acc);
    for (int d = 1; d <= P && K - d >= 0; ++d) {
      __syncthreads();
      msv_stage(Ls, Ys, band + ((size_t)K * (P + 1) + d) * 1024, ya + (size_t)(K - d) * 1024,
                yb + (size_t)(K - d) * 1024, two);
      __syncthreads();
      msv_mma<false>(Ls, Ys, acc, true);
    }
    __syncthreads();
    store_acc(K, acc);
  }
  __syncthreads();
  // backward: x_K = D_K^-1 y_K - sum_d L_{K+d,K}^T x_{K+d}
  for (int K = NBK - 1; K >= 0; --K) {
    double2 acc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = cz();
    __syncthreads();
    msv_stage(Ls, Ys, band + ((size_t)K * (P + 1)) * 1024, ya + (size_t)K * 1024, yb + (size_t)K * 1024, two);
    __syncthreads();
    msv_mma<false>(Ls, Ys, acc, false);
    for (int d = 1; d <= P && K + d < NBK; ++d) {
      __syncthreads();
      msv_stage(Ls, Ys, band + ((size_t)(K + d) * (P + 1) + d) * 1024, ya + (size_t)(K + d) * 1024,
                yb + (size_t)(K + d) * 1024, two);
      __syncthreads();
      msv_mma<true>(Ls, Ys, acc, true);
    }
    __syncthreads();
    store_acc(K, acc);
  }
}

// RHS tiles of the setup solves: tile T < NTB holds columns 32T.. of A_ib (column k = the
// interior entries of interface dof k), tile NTB holds A_ic.
__global__ void k3_build_rhs(int cnt, int s0, int NI, int NB, int NC, int EBI, int ntile, int NTB,
                             const int* __restrict__ bi_idx, const double2* __restrict__ bi_val,
                             const double2* __restrict__ aic, double2* __restrict__ Y) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)NTB * 32 + 32;  // columns per subdomain
  if (gid >= (long long)cnt * per) return;
  const int sc = (int)(gid / per), col = (int)(gid % per), s = s0 + sc;
  const int tile = col >> 5, c = col & 31;
  double2* y = Y + ((size_t)sc * ntile + tile) * NI * 32 + c;
  if (tile < NTB) {
    const int k = col;
    if (k >= NB) return;
    for (int e = 0; e < EBI; ++e) {
      const int i = bi_idx[((size_t)s * NB + k) * EBI + e];
      if (i >= 0) y[(size_t)i * 32] = bi_val[((size_t)s * NB + k) * EBI + e];  // A_ib(i,k) = A_bi(k,i)
    }
  } else if (c < NC) {
    for (int i = 0; i < NI; ++i) y[(size_t)i * 32] = aic[((size_t)s * NI + i) * NC + c];
  }
}

// S_bb = A_bb - A_bi X in the dense chunk buffer (A_bb assembled there by k3_assemble mode 1);
// padding: identity rows/columns beyond n_b
__global__ void k3_schur_build(int cnt, int s0, int NI, int NB, int NBP, int EBI, int ntile,
                               const int* __restrict__ n_b, const int* __restrict__ bi_idx,
                               const double2* __restrict__ bi_val, const double2* __restrict__ X,
                               double2* __restrict__ dense) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)cnt * NBP * NBP) return;
  const int sc = (int)(gid / ((long long)NBP * NBP));
  const int r = (int)((gid / NBP) % NBP), c = (int)(gid % NBP), s = s0 + sc;
  const int nb = n_b[s];
  double2* d = dense + gid;
  if (r >= nb || c >= nb) {
    *d = (r == c) ? make_double2(1.0, 0.0) : cz();
    return;
  }
  double2 v = *d;
  const double2* x = X + ((size_t)sc * ntile + (c >> 5)) * NI * 32 + (c & 31);
  for (int e = 0; e < EBI; ++e) {
    const int i = bi_idx[((size_t)s * NB + r) * EBI + e];
    if (i >= 0) v = cfms(bi_val[((size_t)s * NB + r) * EBI + e], x[(size_t)i * 32], v);
  }
  *d = v;
}

// ---------------------------------------------------------------------------------------
// Blocked Gauss-Jordan inverse of the dense S_bb chunk (no pivoting, see tile_invert),
// NT x NT blocks of 32.  Step K: (1) P = A_KK^-1; (2) row panel A_KJ <- P A_KJ and saved
// column panel C_I = A_IK; (3) A_IJ -= C_I A_KJ, A_IK = -C_I P.
__global__ void __launch_bounds__(256) k3_gj_pivot(int NBP, int K, double2* __restrict__ dense,
                                                   double2* __restrict__ pbuf, double* __restrict__ prat) {
  __shared__ Tile A;
  __shared__ double rat;
  const int sc = blockIdx.x;
  double2* M = dense + (size_t)sc * NBP * NBP;
  tile_load_rm(A, M + (size_t)(K * 32) * NBP + K * 32, NBP);
  __syncthreads();
  tile_invert(A, &rat);
  __syncthreads();
  tile_store_rm(pbuf + (size_t)sc * 1024, 32, A);
  if (threadIdx.x == 0) prat[sc] = fmin(prat[sc], rat);
}
__global__ void __launch_bounds__(256) k3_gj_panel(int NBP, int NT, int K, double2* __restrict__ dense,
                                                   const double2* __restrict__ pbuf, double2* __restrict__ cbuf) {
  __shared__ Tile A, B;
  const int J = blockIdx.x, sc = blockIdx.y;
  double2* M = dense + (size_t)sc * NBP * NBP;
  // save the old column block (J, K)
  for (int e = threadIdx.x; e < 1024; e += blockDim.x)
    cbuf[((size_t)sc * NT + J) * 1024 + e] = M[(size_t)(J * 32 + (e >> 5)) * NBP + K * 32 + (e & 31)];
  if (J == K) return;
  tile_load_rm(A, pbuf + (size_t)sc * 1024, 32);
  tile_load_rm(B, M + (size_t)(K * 32) * NBP + J * 32, NBP);
  __syncthreads();
  double2 acc[4] = {cz(), cz(), cz(), cz()};
  tile_mma<false>(A, B, acc);
  const int r = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
#pragma unroll
  for (int q = 0; q < 4; ++q) M[(size_t)(K * 32 + r) * NBP + J * 32 + c0 + q] = acc[q];
}

// Trailing update of step K as a register-blocked rank-32 GEMM on 64x64 tiles of C (the
// dense chunk; NBP % 64 == 0): C[r][c] -= Cpanel[r][:] R[:][c] with R = the new row panel
// (A_KJ) for columns outside block K and R = P for the columns of block K (which become
// -Cpanel P, the new column panel).  Rows of block K (the row panel) are left alone.
// 256 threads = 16 x 16, each owning a 4 x 4 patch (16 complex accumulators); per k step a
// thread reads 4 + 4 operands from shared memory for 16 complex FMAs.
__global__ void __launch_bounds__(256) k3_gj_update64(int NBP, int NT, int K, double2* __restrict__ dense,
                                                      const double2* __restrict__ pbuf,
                                                      const double2* __restrict__ cbuf) {
  extern __shared__ __align__(16) double2 k3g_sm[];
  double2 (*As)[33] = reinterpret_cast<double2 (*)[33]>(k3g_sm);             // [64][33]  rows x k
  double2 (*Bs)[65] = reinterpret_cast<double2 (*)[65]>(k3g_sm + 64 * 33);   // [32][65]  k x cols
  const int J0 = blockIdx.x * 64, I0 = blockIdx.y * 64, sc = blockIdx.z;
  const int kr = K * 32;
  if (I0 == kr && I0 + 64 <= kr + 32) return;  // (never: tiles are 64 wide)
  double2* M = dense + (size_t)sc * NBP * NBP;
  const double2* P = pbuf + (size_t)sc * 1024;
  // A: old column panel of rows I0..I0+63 (cbuf holds block rows of 32)
  for (int e = threadIdx.x; e < 64 * 32; e += 256) {
    const int r = e >> 5, k = e & 31, I = (I0 + r) >> 5;
    As[r][k] = cbuf[((size_t)sc * NT + I) * 1024 + ((I0 + r) & 31) * 32 + k];
  }
  for (int e = threadIdx.x; e < 32 * 64; e += 256) {
    const int k = e >> 6, c = e & 63, gc = J0 + c;
    Bs[k][c] = (gc >= kr && gc < kr + 32) ? P[k * 32 + (gc - kr)] : M[(size_t)(kr + k) * NBP + gc];
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = cz();
#pragma unroll 2
  for (int k = 0; k < 32; ++k) {
    double2 a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = As[ty * 4 + i][k];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx + 16 * j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = cfma(a[i], b[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = I0 + ty * 4 + i;
    if (gr >= kr && gr < kr + 32) continue;  // row panel: already final
    double2* row = M + (size_t)gr * NBP;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = J0 + tx + 16 * j;
      if (gc >= kr && gc < kr + 32) row[gc] = make_double2(-acc[i][j].x, -acc[i][j].y);
      else row[gc] = csub(row[gc], acc[i][j]);
    }
  }
}
// the pivot block of step K becomes P (after the update kernel has read the row panel)
__global__ void k3_gj_setpivot(int NBP, int K, double2* __restrict__ dense, const double2* __restrict__ pbuf) {
  const int sc = blockIdx.x;
  double2* M = dense + (size_t)sc * NBP * NBP;
  for (int e = threadIdx.x; e < 1024; e += blockDim.x)
    M[(size_t)(K * 32 + (e >> 5)) * NBP + K * 32 + (e & 31)] = pbuf[(size_t)sc * 1024 + e];
}

// ---------------------------------------------------------------------------------------
// Packed symmetric storage of a dense chunk (subdomain s = s0 + sc, NT_s tiles):
// row I = [off-diagonal tiles J < I (1024 each) | diagonal tile (17 x 32)]
__device__ __forceinline__ long long sym_row_off(int I) { return 1024LL * I * (I - 1) / 2 + 544LL * I; }
__device__ __forceinline__ long long sym_size(int NT) { return sym_row_off(NT); }

__global__ void k3_pack_sym(int cnt, int s0, int NBP, const int* __restrict__ nt, const long long* __restrict__ off,
                            const double2* __restrict__ dense, double2* __restrict__ pack) {
  const int sc = blockIdx.y, s = s0 + sc;
  const long long sz = sym_size(nt[s]);
  const double2* M = dense + (size_t)sc * NBP * NBP;
  double2* out = pack + off[s];
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < sz; e += (long long)gridDim.x * blockDim.x) {
    // row I: largest I with sym_row_off(I) <= e
    int I = (int)sqrt((double)e / 512.0);
    while (I > 0 && sym_row_off(I) > e) --I;
    while (sym_row_off(I + 1) <= e) ++I;
    const long long w = e - sym_row_off(I);
    int r, c;
    if (w < 1024LL * I) {
      const int J = (int)(w >> 10), q = (int)(w & 1023);
      r = 32 * I + (q & 31);
      c = 32 * J + (((q >> 5) + (q & 31)) & 31);
    } else {
      const int q = (int)(w - 1024LL * I);
      r = 32 * I + (q & 31);
      c = 32 * I + (((q >> 5) + (q & 31)) & 31);
    }
    out[e] = M[(size_t)r * NBP + c];
  }
}

// ---------------------------------------------------------------------------------------
// Per-iteration packed symmetric GEMV y = S x (K5/K6), one CTA (4 warps) per tile row
// (s, I): y_I (rows) is complete in the CTA; the transposed contributions of the
// off-diagonal tiles go to colpart[s][t = I(I-1)/2 + J] and k3_sym_reduce adds them.
struct SymArgs {
  const int4* work;          // (s, I, J0, J1) per CTA: tiles J0 <= J < J1 of row I (J1 = I + 1: + diagonal)
  const int* rslot;          // row-partial slot of each work item
  const int* nt;             // tiles per subdomain
  const long long* off;      // packed offset per subdomain
  const long long* coff;     // column-partial offset per subdomain (units of 32 entries)
  const double2* pack;
  const double2* xin;        // [S][NB]
  int NB;
  double2* rowpart;          // [items][32]
  double2* colpart;          // [sum_s NT_s (NT_s - 1) / 2][32]
};
template <int BATCH>
__global__ void __launch_bounds__(128) k3_sym_rows(SymArgs a) {
  extern __shared__ double2 k3s_x[];  // x_J0 .. x_{J1-1}, then x_I
  __shared__ double2 red[4][32];
  const int4 wk = a.work[blockIdx.x];
  const int s = wk.x, I = wk.y, J0 = wk.z, J1 = wk.w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* x = a.xin + (size_t)s * a.NB;
  const int nx = 32 * (J1 - J0);
  for (int k = threadIdx.x; k < nx + 32; k += blockDim.x) {
    const int g = k < nx ? 32 * J0 + k : 32 * I + (k - nx);
    k3s_x[k] = g < a.NB ? x[g] : cz();
  }
  __syncthreads();
  const double2* row = a.pack + a.off[s] + sym_row_off(I);
  double2* cp = a.colpart + (a.coff[s] + (long long)I * (I - 1) / 2) * 32;
  const double2 xi = k3s_x[nx + lane];
  double2 yr = cz();
  const int Jend = min(J1, I);
  for (int J = J0 + warp; J < Jend; J += 4) {
    const double2* T = row + (size_t)J * 1024;
    double2 yc = cz();
#pragma unroll
    for (int cb = 0; cb < 32; cb += BATCH) {
      double2 m[BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) m[u] = __ldcs(T + (cb + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        yr = cfma(m[u], k3s_x[32 * (J - J0) + ((lane + cb + u) & 31)], yr);
        yc = cfma(m[u], xi, yc);
        yc = shfl2(yc, (lane + 1) & 31);
      }
    }
    cp[(size_t)J * 32 + lane] = yc;
  }
  if (J1 == I + 1 && warp == (I & 3)) {  // diagonal tile: cc = 0 diagonal, 1..15 both halves, 16 both (l, l+16)
    const double2* D = row + (size_t)I * 1024;
    double2 yc = cz();
#pragma unroll
    for (int cb = 0; cb < 16; cb += BATCH) {
      double2 m[BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) m[u] = __ldcs(D + (cb + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int c = cb + u;
        if (c == 0) {
          yr = cfma(m[u], xi, yr);
        } else {
          yr = cfma(m[u], k3s_x[nx + ((lane + c) & 31)], yr);
          yc = shfl2(yc, (lane + 1) & 31);
          yc = cfma(m[u], xi, yc);
        }
      }
    }
    const double2 m16 = __ldcs(D + 16 * 32 + lane);
    yr = cfma(m16, k3s_x[nx + ((lane + 16) & 31)], yr);
    yc = shfl2(yc, (lane + 17) & 31);
    yr = cadd(yr, yc);
  }
  red[warp][lane] = yr;
  __syncthreads();
  if (warp == 0) {
    const double2 v = cadd(cadd(red[0][lane], red[1][lane]), cadd(red[2][lane], red[3][lane]));
    a.rowpart[(size_t)a.rslot[blockIdx.x] * 32 + lane] = v;
  }
}
// y[s][32J + l] = sum of the row partials of tile row J + sum_{I > J} colpart[s][I(I-1)/2 + J][l]
// (one warp per tile row (s, J); rows: first row-partial slot and count per tile row)
__global__ void k3_sym_reduce(int nwork, const int2* __restrict__ work, const int2* __restrict__ rows,
                              const int* __restrict__ nt, const long long* __restrict__ coff, int NB,
                              const double2* __restrict__ rowpart, const double2* __restrict__ colpart,
                              double2* __restrict__ y) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= nwork) return;
  const int2 wk = work[w];
  const int s = wk.x, J = wk.y, k = 32 * J + lane;
  if (k >= NB) return;
  const int2 rr = rows[w];
  double2 v = rowpart[(size_t)rr.x * 32 + lane];
  for (int q = 1; q < rr.y; ++q) v = cadd(v, rowpart[(size_t)(rr.x + q) * 32 + lane]);
  const double2* cp = colpart + coff[s] * 32;
  for (int I = J + 1; I < nt[s]; ++I) v = cadd(v, cp[((size_t)I * (I - 1) / 2 + J) * 32 + lane]);
  y[(size_t)s * NB + k] = v;
}

// ---------------------------------------------------------------------------------------
// Jump operators (K5/K6): B^T gathers onto interface slots and B gathers onto multipliers.
// mode 0: xin = alpha sum_e sign_e w_row lam[row]   (Dirichlet: alpha = 1, weights W)
// mode 1: xin = -sum_e sign_e lam[row]               (dual operator input t_b = -B^T lam)
// mode 2: xin = fb - sum_e sign_e lam[row]           (t_b = f_b - B^T lam, final eliminate)
__global__ void k3_gather_in(int S, int NB, int MR, int mode, const int* __restrict__ n_b,
                             const int* __restrict__ brow, const double* __restrict__ bsgn,
                             const double* __restrict__ lam_w, const double2* __restrict__ lam,
                             const double2* __restrict__ fb, double2* __restrict__ xin) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)S * NB) return;
  const int s = (int)(gid / NB), k = (int)(gid % NB);
  double2 v = mode == 2 ? fb[gid] : cz();
  if (k < n_b[s]) {
    for (int e = 0; e < MR; ++e) {
      const int r = brow[gid * MR + e];
      if (r < 0) break;
      const double sg = bsgn[gid * MR + e];
      if (mode == 0) v = cadd(v, cscale(lam[r], sg * lam_w[r]));
      else v = csub(v, cscale(lam[r], sg));
    }
  }
  xin[gid] = v;
}
// Dirichlet output: out[row] = w_row (wb[lo] - wb[hi])
__global__ void k3_lam_pre(int nl, const int* __restrict__ lo, const int* __restrict__ hi,
                           const double* __restrict__ lam_w, const double2* __restrict__ wb, double2* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nl) return;
  const int a = lo[r], b = hi[r];  // -1: owner on another rank (sharded: partial sum)
  out[r] = cscale(csub(a >= 0 ? wb[a] : cz(), b >= 0 ? wb[b] : cz()), lam_w[r]);
}
// jump of u_b = u1_b - cpl_b z: out[row] = sign (u_b[lo] - u_b[hi])  (sign -1: F lam)
__global__ void k3_lam_jump(int nl, int NB, int NC, double sign, const int* __restrict__ lo, const int* __restrict__ hi,
                            const double2* __restrict__ u1, const double2* __restrict__ cpl_b,
                            const int* __restrict__ cglob, const double2* __restrict__ z, double2* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nl) return;
  double2 u[2];
  const int sl[2] = {lo[r], hi[r]};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int slot = sl[q], s = slot / NB;
    if (slot < 0) {  // owner on another rank (sharded: partial sum)
      u[q] = cz();
      continue;
    }
    double2 v = u1[slot];
    if (z != nullptr)
      for (int c = 0; c < NC; ++c) {
        const int g = cglob[(size_t)s * NC + c];
        if (g >= 0) v = cfms(cpl_b[(size_t)slot * NC + c], z[g], v);
      }
    u[q] = v;
  }
  out[r] = cscale(csub(u[0], u[1]), sign);
}
// u_b = u1_b - cpl_b z (in place)
__global__ void k3_ub_correct(int S, int NB, int NC, const int* __restrict__ cglob, const double2* __restrict__ z,
                              const double2* __restrict__ cpl_b, double2* __restrict__ u) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)S * NB) return;
  const int s = (int)(gid / NB);
  double2 v = u[gid];
  for (int c = 0; c < NC; ++c) {
    const int g = cglob[(size_t)s * NC + c];
    if (g >= 0) v = cfms(cpl_b[gid * NC + c], z[g], v);
  }
  u[gid] = v;
}

// ---------------------------------------------------------------------------------------
// Coarse problem (K4).  gcp[s][c] = cpl_b^T xin (+ cpl_i^T fi): one CTA per subdomain,
// one warp per local corner dof; g = fc - sum_slots gcp; z = C^-1 g (dense, row per warp).
// gcp partials: CTA (s, g) covers the slice g of the row-major [k][c] entries of cpl_b (and
// of cpl_i); thread t reads entries t, t + 256, .. of its slice (coalesced) with c fixed
// (256 % NC == 0 is not required: threads t >= per idle); per-c partials in fixed order.
// Output part[s][g][c]; k3_coarse_rhs sums the G slices of a slot in order.
__global__ void __launch_bounds__(256) k3_gcp(int NB, int NC, int NI, int G, const double2* __restrict__ cpl_b,
                                              const double2* __restrict__ xin, const double2* __restrict__ cpl_i,
                                              const double2* __restrict__ fi, double2* __restrict__ part) {
  __shared__ double2 red[256];
  const int s = blockIdx.x, g = blockIdx.y, t = threadIdx.x;
  const int per = 256 / NC * NC;
  double2 acc = cz();
  if (t < per) {
    const long long nb = (long long)NB * NC, ni = cpl_i != nullptr ? (long long)NI * NC : 0;
    const long long tot = nb + ni, len = (tot + G - 1) / G;
    const long long e0 = g * len, e1 = min(tot, e0 + len);
    // align the slice start to a multiple of NC so that thread t keeps c = t % NC
    long long e = e0 - e0 % NC + t;
    if (e < e0) e += per;
    const double2* cb = cpl_b + (size_t)s * NB * NC;
    const double2* x = xin + (size_t)s * NB;
    const double2* ci = cpl_i != nullptr ? cpl_i + (size_t)s * NI * NC : nullptr;
    const double2* f = fi != nullptr ? fi + (size_t)s * NI : nullptr;
    for (; e < e1; e += per) {
      if (e < nb) acc = cfma(cb[e], x[e / NC], acc);
      else acc = cfma(ci[e - nb], f[(e - nb) / NC], acc);
    }
  }
  red[t] = acc;
  __syncthreads();
  if (t < NC) {
    double2 v = cz();
    for (int q = t; q < per; q += NC) v = cadd(v, red[q]);
    part[((size_t)s * G + g) * NC + t] = v;
  }
}
// g = fc - sum_slots gcp, gcp of slot (s, k) = sum of its G partials part[s][g][k]
__global__ void k3_coarse_rhs(int nc, int NC, int G, const int* __restrict__ slots, const double2* __restrict__ part,
                              const double2* __restrict__ fc, double2* __restrict__ g) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double2 acc = fc ? fc[c] : cz();
  for (int q = 0; q < 8; ++q) {
    const int sl = slots[c * 8 + q];
    if (sl < 0) continue;
    const int s = sl / NC, k = sl % NC;
    double2 v = cz();
    for (int gg = 0; gg < G; ++gg) v = cadd(v, part[((size_t)s * G + gg) * NC + k]);
    acc = csub(acc, v);
  }
  g[c] = acc;
}
__global__ void k3_dense_gemv(int n, const double2* __restrict__ A, const double2* __restrict__ x,
                              double2* __restrict__ y) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= n) return;
  double2 acc = cz();
  for (int c = lane; c < n; c += 32) acc = cfma(A[(size_t)r * n + c], x[c], acc);
  acc = warp_sum2(acc);
  if (lane == 0) y[r] = acc;
}

// coupling pieces at setup (chunk): R = A_bc - A_bi Yc (Yc = tile NTB of X)
__global__ void k3_cpl_rhs(int cnt, int s0, int NI, int NB, int NC, int EBI, int ntile, int NTB,
                           const int* __restrict__ bi_idx, const double2* __restrict__ bi_val,
                           const double2* __restrict__ abc, const double2* __restrict__ X, double2* __restrict__ R) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)cnt * NB * NC) return;
  const int sc = (int)(gid / ((long long)NB * NC)), k = (int)((gid / NC) % NB), c = (int)(gid % NC), s = s0 + sc;
  double2 v = abc[((size_t)s * NB + k) * NC + c];
  const double2* yc = X + ((size_t)sc * ntile + NTB) * NI * 32 + c;
  for (int e = 0; e < EBI; ++e) {
    const int i = bi_idx[((size_t)s * NB + k) * EBI + e];
    if (i >= 0) v = cfms(bi_val[((size_t)s * NB + k) * EBI + e], yc[(size_t)i * 32], v);
  }
  R[gid] = v;
}
// cpl_b[s][k][:] = Sinv[k][:] R  (one warp per (sc, k); NC <= 32 accumulators in lanes' loop)
__global__ void k3_cpl_b(int cnt, int s0, int NB, int NBP, int NC, const int* __restrict__ n_b,
                         const double2* __restrict__ sinv, const double2* __restrict__ R, double2* __restrict__ cpl_b) {
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= (long long)cnt * NB) return;
  const int sc = (int)(w / NB), k = (int)(w % NB), s = s0 + sc;
  const int nb = n_b[s];
  double2* out = cpl_b + ((size_t)s * NB + k) * NC;
  if (k >= nb) {
    if (lane < NC) out[lane] = cz();
    return;
  }
  const double2* row = sinv + ((size_t)sc * NBP + k) * NBP;
  const double2* Rs = R + (size_t)sc * NB * NC;
  for (int c = 0; c < NC; ++c) {
    double2 acc = cz();
    for (int k2 = lane; k2 < nb; k2 += 32) acc = cfma(row[k2], Rs[(size_t)k2 * NC + c], acc);
    acc = warp_sum2(acc);
    if (lane == 0) out[c] = acc;
  }
}
// second coupling rhs A_ic - A_ib cpl_b into tile NTB of X
__global__ void k3_cpl_i_rhs(int cnt, int s0, int NI, int NB, int NC, int EIB, int ntile, int NTB,
                             const int* __restrict__ ib_idx, const double2* __restrict__ ib_val,
                             const double2* __restrict__ aic, const double2* __restrict__ cpl_b, double2* __restrict__ X) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)cnt * NI * 32) return;
  const int sc = (int)(gid / ((long long)NI * 32)), i = (int)((gid / 32) % NI), c = (int)(gid % 32), s = s0 + sc;
  double2 v = cz();
  if (c < NC) {
    v = aic[((size_t)s * NI + i) * NC + c];
    for (int e = 0; e < EIB; ++e) {
      const int k = ib_idx[((size_t)s * NI + i) * EIB + e];
      if (k >= 0) v = cfms(ib_val[((size_t)s * NI + i) * EIB + e], cpl_b[((size_t)s * NB + k) * NC + c], v);
    }
  }
  X[(((size_t)sc * ntile + NTB) * NI + i) * 32 + c] = v;
}
// cpl_i = tile NTB; contrib = A_cc - A_ic^T cpl_i - A_bc^T cpl_b (transpose, feti.cpp:433)
__global__ void k3_coarse_contrib(int cnt, int s0, int NI, int NB, int NC, int ntile, int NTB,
                                  const double2* __restrict__ X, const double2* __restrict__ aic,
                                  const double2* __restrict__ abc, const double2* __restrict__ acc,
                                  const double2* __restrict__ cpl_b, double2* __restrict__ cpl_i,
                                  double2* __restrict__ contrib) {
  const int sc = blockIdx.x, s = s0 + sc;
  const double2* Xc = X + ((size_t)sc * ntile + NTB) * NI * 32;
  for (long long e = threadIdx.x; e < (long long)NI * NC; e += blockDim.x) {
    const int i = (int)(e / NC), c = (int)(e % NC);
    cpl_i[((size_t)s * NI + i) * NC + c] = Xc[(size_t)i * 32 + c];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int p = warp; p < NC * NC; p += nw) {
    const int c1 = p / NC, c2 = p % NC;
    double2 v = cz();
    for (int i = lane; i < NI; i += 32)
      v = cfma(aic[((size_t)s * NI + i) * NC + c1], Xc[(size_t)i * 32 + c2], v);
    for (int k = lane; k < NB; k += 32)
      v = cfma(abc[((size_t)s * NB + k) * NC + c1], cpl_b[((size_t)s * NB + k) * NC + c2], v);
    v = warp_sum2(v);
    if (lane == 0) contrib[((size_t)s * NC + c1) * NC + c2] = csub(acc[((size_t)s * NC + c1) * NC + c2], v);
  }
}
// dense coarse matrix sum_s (A_cc - contrib) over the corner slots (feti.cpp:440-454)
__global__ void k3_coarse_assemble(int nc, int NC, const int* __restrict__ slots, const double2* __restrict__ contrib,
                                   double2* __restrict__ C) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)nc * nc) return;
  const int a = (int)(gid / nc), b = (int)(gid % nc);
  double2 v = cz();
  for (int qa = 0; qa < 8; ++qa) {
    const int sa = slots[a * 8 + qa];
    if (sa < 0) continue;
    for (int qb = 0; qb < 8; ++qb) {
      const int sb = slots[b * 8 + qb];
      if (sb < 0 || sb / NC != sa / NC) continue;
      const int s = sa / NC;
      v = cadd(v, contrib[((size_t)s * NC + sa % NC) * NC + sb % NC]);
    }
  }
  C[gid] = v;
}
// Gauss-Jordan with partial pivoting on the equilibrated coarse matrix (PartialPivLU's
// pivots; the 1e-13 singularity check of feti.cpp:469-474 is applied on the host)
__global__ void k3_cgj_pivot(int n, int k, double2* __restrict__ A, int* __restrict__ piv, double* __restrict__ pabs,
                             double2* __restrict__ col) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = -1.0;
  int arg = k;
  for (int r = k + threadIdx.x; r < n; r += blockDim.x) {
    const double v = cabs2(A[(size_t)r * n + k]);
    if (v > best) best = v, arg = r;
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = arg;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v = bv[threadIdx.x + o];
      const int j = bi[threadIdx.x + o];
      if (v > bv[threadIdx.x] || (v == bv[threadIdx.x] && j < bi[threadIdx.x])) bv[threadIdx.x] = v, bi[threadIdx.x] = j;
    }
    __syncthreads();
  }
  const int p = bi[0];
  if (p != k)
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      const double2 t = A[(size_t)k * n + c];
      A[(size_t)k * n + c] = A[(size_t)p * n + c];
      A[(size_t)p * n + c] = t;
    }
  __syncthreads();
  const double2 pv = A[(size_t)k * n + k];
  if (threadIdx.x == 0) {
    piv[k] = p;
    pabs[k] = sqrt(cabs2(pv));
  }
  const double2 inv = crecip(pv);
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) A[(size_t)k * n + c] = c == k ? inv : cmul(A[(size_t)k * n + c], inv);
  for (int r = threadIdx.x; r < n; r += blockDim.x) col[r] = r == k ? cz() : A[(size_t)r * n + k];
}
__global__ void k3_cgj_update(int n, int k, double2* __restrict__ A, const double2* __restrict__ col) {
  const int r = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (r == k || c >= n) return;
  const double2 f = col[r];
  const double2 pk = A[(size_t)k * n + c];
  A[(size_t)r * n + c] = c == k ? make_double2(-(f.x * pk.x - f.y * pk.y), -(f.x * pk.y + f.y * pk.x))
                                : cfms(f, pk, A[(size_t)r * n + c]);
}
// undo the row exchanges of Gauss-Jordan: columns swapped in reverse order
__global__ void k3_cgj_unpermute(int n, double2* __restrict__ A, const int* __restrict__ piv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int k = n - 1; k >= 0; --k) {
    const int p = piv[k];
    if (p != k) {
      const double2 t = A[(size_t)r * n + k];
      A[(size_t)r * n + k] = A[(size_t)r * n + p];
      A[(size_t)r * n + p] = t;
    }
  }
}
__global__ void k3_scale_sym(int n, double2* __restrict__ A, const double* __restrict__ sc) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)n * n) return;
  A[gid] = cscale(A[gid], sc[gid / n] * sc[gid % n]);
}
__global__ void k3_diag_scale(int n, const double2* __restrict__ A, double* __restrict__ sc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = sqrt(cabs2(A[(size_t)i * n + i]));
  sc[i] = d > 0.0 ? 1.0 / sqrt(d) : 1.0;
}

// ---------------------------------------------------------------------------------------
// Eliminate pieces (feti.cpp:493-556)
// split_rhs: f_i = rhs[idof], f_b = w rhs[bdof], f_c = rhs[corner dof]
__global__ void k3_split(int S, int NI, int NB, const int* __restrict__ idof, const int* __restrict__ bdof,
                         const double* __restrict__ bw, const double2* __restrict__ rhs, double2* __restrict__ fi,
                         double2* __restrict__ fb) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long ni = (long long)S * NI;
  if (gid < ni) {
    const int f = idof[gid];
    fi[gid] = f >= 0 ? rhs[f] : cz();
  } else if (gid < ni + (long long)S * NB) {
    const long long k = gid - ni;
    const int f = bdof[k];
    fb[k] = f >= 0 ? cscale(rhs[f], bw[k]) : cz();
  }
}
__global__ void k3_gather_corner(int nc, const int* __restrict__ cdof, const double2* __restrict__ rhs,
                                 double2* __restrict__ fc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc) fc[c] = rhs[cdof[c]];
}
// tb' = tb - A_bi yi
__global__ void k3_tb_minus(int S, int NB, int NI, int EBI, const int* __restrict__ bi_idx,
                            const double2* __restrict__ bi_val, const double2* __restrict__ yi,
                            const double2* __restrict__ tb, double2* __restrict__ out) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)S * NB) return;
  const int s = (int)(gid / NB);
  double2 v = tb[gid];
  for (int e = 0; e < EBI; ++e) {
    const int i = bi_idx[gid * EBI + e];
    if (i >= 0) v = cfms(bi_val[gid * EBI + e], yi[(size_t)s * NI + i], v);
  }
  out[gid] = v;
}
// r_i = f_i - A_ib u_b - A_ic z
__global__ void k3_ri_rhs(int S, int NI, int NB, int NC, int EIB, const int* __restrict__ ib_idx,
                          const double2* __restrict__ ib_val, const double2* __restrict__ aic,
                          const int* __restrict__ cglob, const double2* __restrict__ z, const double2* __restrict__ ub,
                          const double2* __restrict__ fi, double2* __restrict__ ri) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)S * NI) return;
  const int s = (int)(gid / NI);
  double2 v = fi[gid];
  for (int e = 0; e < EIB; ++e) {
    const int k = ib_idx[gid * EIB + e];
    if (k >= 0) v = cfms(ib_val[gid * EIB + e], ub[(size_t)s * NB + k], v);
  }
  for (int c = 0; c < NC; ++c) {
    const int g = cglob[(size_t)s * NC + c];
    if (g >= 0) v = cfms(aic[gid * NC + c], z[g], v);
  }
  ri[gid] = v;
}
// primal assembly x[f] (feti.cpp:700-708): interior u_i, weighted interface slots, corner z
__global__ void k3_assemble_x(int n, const int* __restrict__ kind, const int* __restrict__ ref,
                              const double* __restrict__ xw, const double2* __restrict__ ui,
                              const double2* __restrict__ ub, const double2* __restrict__ z, double2* __restrict__ x) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const int k = kind[f];
  const int* r = ref + (size_t)f * 4;
  double2 v = cz();
  if (k < 0) {  // sharded: owned by other ranks
  } else if (k == 0) {
    v = ui[r[0]];
  } else if (k == 2) {
    v = z[r[0]];
  } else {
    for (int q = 0; q < 4 && r[q] >= 0; ++q) v = cadd(v, cscale(ub[r[q]], xw[f]));
  }
  x[f] = v;
}

// ---------------------------------------------------------------------------------------
// Global operators on the structured mesh (K8): y = (kc K + mc M) x (+ Kc xc), one thread
// per free dof gathering its <= 8 elements (element-by-element, exact like the CSR apply).
struct Glob3 {
  int nx, ny, nz, dpn, ed, n;
  const int* free_dofs;
  const int* free_map;
  const int* cons_map;
  const double* ke;
  const double* me;
};
template <typename T>
__device__ __forceinline__ double2 to_c(T v);
template <>
__device__ __forceinline__ double2 to_c<double>(double v) { return make_double2(v, 0.0); }
template <>
__device__ __forceinline__ double2 to_c<double2>(double2 v) { return v; }
template <typename T>
__device__ __forceinline__ void from_c(T* p, double2 v);
template <>
__device__ __forceinline__ void from_c<double>(double* p, double2 v) { *p = v.x; }
template <>
__device__ __forceinline__ void from_c<double2>(double2* p, double2 v) { *p = v; }

template <typename T>
__global__ void k3_apply_global(Glob3 g, const T* __restrict__ x, const double* __restrict__ xc, double2 kc,
                                double2 mc, T* __restrict__ y) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= g.n) return;
  const int md = g.free_dofs[f], dpn = g.dpn, c = md % dpn, node = md / dpn;
  const int nnx = g.nx + 1, nny = g.ny + 1;
  const int i = node % nnx, j = (node / nnx) % nny, k = node / (nnx * nny);
  const int hx[8] = {0, 1, 1, 0, 0, 1, 1, 0}, hy[8] = {0, 0, 1, 1, 0, 0, 1, 1};
  double2 acc = cz();
  for (int ek = max(k - 1, 0); ek <= min(k, g.nz - 1); ++ek)
    for (int ej = max(j - 1, 0); ej <= min(j, g.ny - 1); ++ej)
      for (int ei = max(i - 1, 0); ei <= min(i, g.nx - 1); ++ei) {
        const int dx = i - ei, dy = j - ej, dz = k - ek;
        const int an = dz * 4 + (dy == 0 ? dx : 3 - dx);
        for (int b = 0; b < 8; ++b) {
          const int nb = ((ek + (b >> 2)) * nny + (ej + hy[b])) * nnx + (ei + hx[b]);
          for (int c2 = 0; c2 < dpn; ++c2) {
            const int md2 = nb * dpn + c2, q = (an * dpn + c) * g.ed + b * dpn + c2;
            const double2 coef = cadd(cscale(kc, g.ke[q]), cscale(mc, g.me[q]));
            const int f2 = g.free_map[md2];
            if (f2 >= 0) acc = cfma(coef, to_c<T>(x[f2]), acc);
            else if (xc != nullptr) acc = cfma(make_double2(g.ke[q], 0.0), make_double2(xc[g.cons_map[md2]], 0.0), acc);
          }
        }
      }
  from_c<T>(y + f, acc);
}

// y = S x with a constant 27-point stencil on the Lx x Ly x Lz grid of interior nodes
// (free dofs in lexicographic order, zero outside): heat with whole-boundary Dirichlet.
// The stencil entries are the element sums of the element matrix at an interior node, so
// this equals the element-by-element apply up to the order of the additions.
struct Stencil27 {
  double2 c[27];
};
template <typename T>
__global__ void k3_apply_stencil27(int Lx, int Ly, int Lz, Stencil27 S, const T* __restrict__ x, T* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= Lx) return;
  double2 acc = cz();
#pragma unroll
  for (int dz = -1; dz <= 1; ++dz) {
    const int kk = k + dz;
    if (kk < 0 || kk >= Lz) continue;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int jj = j + dy;
      if (jj < 0 || jj >= Ly) continue;
      const T* row = x + ((size_t)kk * Ly + jj) * Lx;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int ii = i + dx;
        if (ii < 0 || ii >= Lx) continue;
        acc = cfma(S.c[((dz + 1) * 3 + (dy + 1)) * 3 + dx + 1], to_c<T>(row[ii]), acc);
      }
    }
  }
  from_c<T>(y + ((size_t)k * Ly + j) * Lx + i, acc);
}

// V^-1 v in place for V = M_z (x) M_y (x) M_x (x) I_dpn: Thomas along lines, one thread per
// line; line l starts at (l / G) * S1 + (l % G) * S2, element stride es
__global__ void k3_tridiag(double* __restrict__ v, int nlines, int len, int G, long long S1, long long S2,
                           long long es, const double* __restrict__ cp, const double* __restrict__ dinv, double off) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlines) return;
  double* p = v + (long long)(l / G) * S1 + (long long)(l % G) * S2;
  double x = 0.0;
  for (int i = 0; i < len; ++i) {
    x = (p[(long long)i * es] - off * x) * dinv[i];
    p[(long long)i * es] = x;
  }
  for (int i = len - 2; i >= 0; --i) {
    x = p[(long long)i * es] - cp[i] * x;
    p[(long long)i * es] = x;
  }
}

// ---------------------------------------------------------------------------------------
// Krylov vector kernels (K7)
// part[b][j] = sum_{rows of block b} conj(V_j) w  (j < nv), plus |w|^2 in slot nv.
// The block's rows of w are staged in shared memory once; warp q then takes the vectors
// j = q, q + 8, ... (coalesced loads of V_j), so all dots of the block run concurrently.
// rows_pb <= 2048 (32 KB of staging).
__global__ void __launch_bounds__(256) k3_mdot_part(int n, int nv, const double2* __restrict__ V, size_t ldv,
                                                    const double2* __restrict__ w, double2* __restrict__ part, int rows_pb) {
  __shared__ double2 ws[2048];
  const int r0 = blockIdx.x * rows_pb, cnt = min(n, r0 + rows_pb) - r0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) ws[q] = w[r0 + q];
  __syncthreads();
  for (int j = warp; j <= nv; j += 8) {
    double2 acc = cz();
    if (j < nv) {
      const double2* v = V + (size_t)j * ldv + r0;
#pragma unroll 4
      for (int q = lane; q < cnt; q += 32) acc = cfma_conj(v[q], ws[q], acc);
    } else {
      for (int q = lane; q < cnt; q += 32) acc.x += cabs2(ws[q]);
    }
    acc = warp_sum2(acc);
    if (lane == 0) part[(size_t)blockIdx.x * (nv + 1) + j] = acc;
  }
}
// one warp per dot: lanes stride over the block partials, fixed-order butterfly
__global__ void k3_mdot_final(int nblk, int nv, const double2* __restrict__ part, double2* __restrict__ out) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j > nv) return;
  double2 t = cz();
  for (int b0 = lane; b0 < nblk; b0 += 32 * 8) {  // 8 loads in flight, same summation order
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b0 + 32 * u < nblk ? part[(size_t)(b0 + 32 * u) * (nv + 1) + j] : cz();
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b0 + 32 * u < nblk) t = cadd(t, v[u]);
  }
  t = warp_sum2(t);
  if (lane == 0) out[j] = t;
}
// w -= sum_j V_j h_j
__global__ void k3_mupdate(int n, int nv, const double2* __restrict__ V, size_t ldv, const double2* __restrict__ h,
                           double2* __restrict__ w) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double2 v = w[r];
#pragma unroll 8
  for (int j = 0; j < nv; ++j) v = cfms(V[(size_t)j * ldv + r], h[j], v);
  w[r] = v;
}
// y += sum_j V_j c_j
__global__ void k3_mcombine(int n, int nv, const double2* __restrict__ V, size_t ldv, const double2* __restrict__ c,
                            double2* __restrict__ y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double2 v = y[r];
  for (int j = 0; j < nv; ++j) v = cfma(V[(size_t)j * ldv + r], c[j], v);
  y[r] = v;
}
__global__ void k3_scale_to(int n, double2 a, const double2* __restrict__ x, double2* __restrict__ y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = cmul(a, x[r]);
}
// y = a x + b y
__global__ void k3_axpby(int n, double2 a, const double2* __restrict__ x, double2 b, double2* __restrict__ y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = cadd(cmul(a, x[r]), cmul(b, y[r]));
}
// (|x|^2 sum, max |x|) partials and final
__global__ void k3_norm_part(int n, const double2* __restrict__ x, double2* __restrict__ part) {
  __shared__ double ss[8], sm[8];
  double s = 0.0, m = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const double a = cabs2(x[r]);
    s += a;
    m = fmax(m, a);
  }
  s = warp_sum(s);
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) ss[threadIdx.x >> 5] = s, sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) a += ss[q], b = fmax(b, sm[q]);
    part[blockIdx.x] = make_double2(a, b);
  }
}
__global__ void k3_norm_final(int nblk, const double2* __restrict__ part, double2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  double a = 0.0, b = 0.0;
  for (int q0 = lane; q0 < nblk; q0 += 32 * 8) {  // 8 loads in flight, same summation order
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = q0 + 32 * u < nblk ? part[q0 + 32 * u] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (q0 + 32 * u < nblk) a += v[u].x, b = fmax(b, v[u].y);
  }
  a = warp_sum(a);
  b = warp_max(b);
  if (lane == 0) *out = make_double2(a, sqrt(b));
}
__global__ void k3_real_to_complex(int n, const double* __restrict__ x, double2* __restrict__ y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = make_double2(x[r], 0.0);
}
__global__ void k3_conj(int n, const double2* x, double2* y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = cconj(x[r]);
}
__global__ void k3_sub(int n, const double2* a, const double2* b, double2* y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = csub(a[r], b[r]);
}
// lambda = Re t, leak partial = max |Im t| (as |.|^2 in the max slot)
__global__ void k3_realify(int n, const double2* __restrict__ t, double* __restrict__ lam) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) lam[r] = t[r].x;
}
__global__ void k3_imag(int n, const double2* __restrict__ t, double2* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) out[r] = make_double2(0.0, t[r].y);
}
// y = ybar - w, u = lam / phi
__global__ void k3_recover(int n, const double* __restrict__ ybar, const double* __restrict__ w,
                           const double* __restrict__ lam, double phi, double* __restrict__ y, double* __restrict__ u) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  y[r] = ybar[r] - w[r];
  u[r] = lam[r] / phi;
}

// ------------------------------------------------------------------ separable interior solve
// Heat on the structured mesh (configs 4 and the 3D heat tests): every subdomain interior is
// the same mx x my x mz grid (x fastest) and A_ii = sum over axes of K1 (x) M1 (x) M1 + mc
// M1 (x) M1 (x) M1 (heat_hex builds exactly these tensor products).  With the orthonormal,
// symmetric DST-I matrices S of each axis: A_ii^-1 X = T (T X ./ D) with T = Sz (x) Sy (x) Sx
// applied axis by axis (fast diagonalisation, exact).  One CTA per subdomain; the grid
// lives in shared memory (two ping-pong copies), one thread per output entry and axis pass.
__global__ void __launch_bounds__(256) k3_fdm_solve(double2* __restrict__ X, size_t ldx, int mx, int my, int mz,
                                                    const double* __restrict__ Sx, const double* __restrict__ Sy,
                                                    const double* __restrict__ Sz, const double2* __restrict__ invD) {
  extern __shared__ double2 f3_sh[];
  const int n = mx * my * mz;
  double2* A = f3_sh;
  double2* B = f3_sh + n;
  double* sx = reinterpret_cast<double*>(B + n);  // [32][32] each
  double* sy = sx + 1024;
  double* sz = sy + 1024;
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    sx[e] = Sx[e];
    sy[e] = Sy[e];
    sz[e] = Sz[e];
  }
  double2* x = X + (size_t)blockIdx.x * ldx;
  for (int e = threadIdx.x; e < n; e += blockDim.x) A[e] = x[e];
  __syncthreads();
  const int pxy = mx * my;
  // One thread per line of the axis: the line's <= 32 entries are loaded into registers once
  // and all outputs of the line formed from them (S entries are warp-uniform broadcasts):
  // out[c] = sum_q S[c][q] in[q] along the line.  FP64 FMA on registers instead of one
  // shared-memory load per multiply-add.
  auto pass = [&](const double2* in, double2* out, int len, int lines, int stride, const double* Sa,
                  const double2* dv) {
    for (int l = threadIdx.x; l < lines; l += blockDim.x) {
      int base;
      if (stride == 1) base = l * mx;                                   // x lines: (k, j)
      else if (stride == mx) base = (l / mx) * pxy + (l % mx);          // y lines: (k, i)
      else base = l;                                                    // z lines: (j, i)
      double vr[32], vi[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const double2 v = q < len ? in[base + q * stride] : make_double2(0.0, 0.0);
        vr[q] = v.x;
        vi[q] = v.y;
      }
      for (int c = 0; c < len; ++c) {
        double ar = 0.0, ai = 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const double sc = Sa[c * 32 + q];  // zero beyond len
          ar = fma(sc, vr[q], ar);
          ai = fma(sc, vi[q], ai);
        }
        const int e = base + c * stride;
        if (dv != nullptr) {
          const double2 d = dv[e];
          out[e] = make_double2(ar * d.x - ai * d.y, ar * d.y + ai * d.x);
        } else {
          out[e] = make_double2(ar, ai);
        }
      }
    }
  };
  auto pass_x = [&](const double2* in, double2* out) { pass(in, out, mx, my * mz, 1, sx, nullptr); };
  auto pass_y = [&](const double2* in, double2* out) { pass(in, out, my, mx * mz, mx, sy, nullptr); };
  auto pass_z = [&](const double2* in, double2* out, bool divide) {
    pass(in, out, mz, pxy, pxy, sz, divide ? invD : nullptr);
  };
  pass_x(A, B);
  __syncthreads();
  pass_y(B, A);
  __syncthreads();
  pass_z(A, B, true);
  __syncthreads();
  pass_x(B, A);
  __syncthreads();
  pass_y(A, B);
  __syncthreads();
  pass_z(B, A, false);
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x) x[e] = A[e];
}
inline size_t fdm3_smem(int n) { return 2 * (size_t)n * sizeof(double2) + 3 * 1024 * sizeof(double); }

}  // namespace k3
}  // namespace fetigpu
