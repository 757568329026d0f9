// band.cuh — batched banded complex-symmetric LDL^T (K2) and the banded
// forward/backward substitution (K5) with TMA-staged factor panels.
//
// Replaces the Eigen SparseLU factorization and solves of the reference
// (feti.cpp:350-359 factor; solves at feti.cpp:432, 521, 615).  A = K_ii + c M_ii is
// complex symmetric (A = A^T, not Hermitian) with an SPD real part, so LDL^T without
// pivoting exists and is stable; it agrees with the reference's pivoted LU to rounding.
//
// Storage, per matrix (n rows, half-bandwidth W, LD = W + 1 entries per row/column):
//   colband[j][0]   = 1/d_j                   colband[j][k] = L(j+k, j),  k = 1..W
//   rowband[j][0]   = 1                       rowband[j][k] = L(j, j-k),  k = 1..W
// Before factorization colband holds the lower band of A (colband[j][k] = A(j+k, j)).
// Both sweeps are "column oriented" (an axpy per step): the forward sweep streams
// colband in increasing j, the backward sweep streams rowband in decreasing j, each
// exactly once per solve — the algorithmic bytes of a solve are 2 * n * LD * 16 B.
#pragma once

#include "common.cuh"

namespace fetigpu {

// ---------------------------------------------------------------------------------------
// K2: one CTA per matrix.  Right-looking band LDL^T with the active (W+1)-column window
// held in a shared-memory ring of W+2 columns, so one __syncthreads per column.
template <int W>
__global__ void __launch_bounds__(256) k_band_ldlt(double2* __restrict__ colband, double2* __restrict__ rowband,
                                                   size_t sub_stride, int n, int* __restrict__ status) {
  constexpr int LD = W + 1, R = W + 2;
  extern __shared__ __align__(16) unsigned char ldlt_smem[];
  double2 (*ring)[LD] = reinterpret_cast<double2 (*)[LD]>(ldlt_smem);
  const int s = blockIdx.x, tid = threadIdx.x;
  double2* A = colband + (size_t)s * sub_stride;
  double2* Rb = rowband + (size_t)s * sub_stride;
  for (int idx = tid; idx < (W + 1) * LD; idx += blockDim.x) {
    const int c = idx / LD, k = idx % LD;
    ring[c][k] = c < n ? A[(size_t)c * LD + k] : cz();
  }
  __syncthreads();
  int first_bad = 0;
  for (int j = 0; j < n; ++j) {
    const int slot = j % R;
    {  // prefetch column j+W+1 into the slot column j-1 vacated
      const int nc = j + W + 1, ns = nc % R;
      if (tid < LD) ring[ns][tid] = nc < n ? A[(size_t)nc * LD + tid] : cz();
    }
    const double2 d = ring[slot][0];
    const double2 dinv = crecip(d);
    for (int idx = tid; idx < W * W; idx += blockDim.x) {
      const int k = idx / W + 1, m = idx % W + 1;
      if (m >= k && j + m < n) {
        const double2 lk = cmul(ring[slot][k], dinv);
        double2& t = ring[(j + k) % R][m - k];
        t = cfms(ring[slot][m], lk, t);
      }
    }
    if (tid <= W) {
      const double2 v = tid == 0 ? dinv : cmul(ring[slot][tid], dinv);
      A[(size_t)j * LD + tid] = v;
      if (tid == 0)
        Rb[(size_t)j * LD] = make_double2(1.0, 0.0);
      else if (j + tid < n)
        Rb[(size_t)(j + tid) * LD + tid] = v;
    }
    if (tid == 0 && first_bad == 0) {
      const double a2 = cabs2(d);
      if (!(a2 > 0.0) || !isfinite(a2)) first_bad = j + 1;
    }
    __syncthreads();
  }
  if (tid == 0) status[s] = first_bad;
}

// ---------------------------------------------------------------------------------------
// K5: banded substitution x = L^-T D^-1 L^-1 b, in place, for nrhs right-hand sides per
// matrix.  grid = (n_matrices, ceil(nrhs / WARPS)); warp w of a CTA owns one RHS; all
// warps of a CTA share the factor panels, which one elected thread streams into a
// STAGES-deep shared-memory ring with 1-D TMA bulk copies (cp.async.bulk + mbarrier).
//
// Per step j a warp keeps the window rows j..j+32*NS-1 in registers; lane 0 holds the
// pivot row, broadcasts v_j, and every lane applies one complex FMA per slot with the
// band column staged in shared memory ("warp per band column").
template <int W, int WARPS, int CH, int STAGES>
__global__ void __launch_bounds__(WARPS * 32)
    k_band_solve(const double2* __restrict__ colband, const double2* __restrict__ rowband, size_t band_stride,
                 int n, double2* __restrict__ X, size_t x_sub_stride, size_t x_rhs_stride, int nrhs) {
  constexpr int LD = W + 1;
  constexpr int NS = (W < 32) ? 1 : 2;  // lane slots; window = 32*NS rows
  constexpr int WIN = 32 * NS;
  static_assert(W <= WIN, "band wider than the register window");
  static_assert(CH <= 32, "one entering row per lane");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* stage = reinterpret_cast<double2*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)STAGES * CH * LD);
  uint64_t* empty = full + STAGES;
  double2* bbuf = reinterpret_cast<double2*>(empty + STAGES) + 0;  // [WARPS][CH] new-row values

  // grid (rhs groups, matrices): the CTAs of one matrix are adjacent in launch order, so
  // they run together and all but the first read the band from L2
  const int s = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rhs = blockIdx.x * WARPS + warp;
  const bool active = rhs < nrhs;
  double2* x = X + (size_t)s * x_sub_stride + (size_t)(active ? rhs : 0) * x_rhs_stride;
  double2* myb = bbuf + warp * CH;
  const int nch = (n + CH - 1) / CH;
  const int total = 2 * nch;

  auto chunk_src = [&](int q, uint32_t& bytes) -> const double2* {
    const bool fwd = q < nch;
    const int c = fwd ? q : (2 * nch - 1 - q);
    const int rows = min(CH, n - c * CH);
    bytes = (uint32_t)rows * LD * sizeof(double2);
    return (fwd ? colband : rowband) + (size_t)s * band_stride + (size_t)c * CH * LD;
  };

  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < STAGES && q < total; ++q) {
      uint32_t bytes;
      const double2* src = chunk_src(q, bytes);
      mbar_arrive_expect_tx(&full[q], bytes);
      tma_load_1d(stage + (size_t)q * CH * LD, src, bytes, &full[q]);
    }
  }

  // Shifting window: at step j, lane l of slot sl holds row j + l + 32 sl.  The pivot is
  // always lane 0 of slot 0, and lane l's coefficient is always col[l + 1 + 32 sl], so a
  // step is one broadcast + one shift (shuffles), one coalesced LDS and one complex FMA
  // per slot — no per-lane index arithmetic.
  double2 y[NS];
  // ---------------- forward sweep: L v = b, write D^-1 v --------------------------------
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    const int row = lane + 32 * sl;
    y[sl] = (active && row < n) ? x[row] : cz();
  }
  // b values of the rows entering the window during chunk c: rows c*CH + t + WIN
  double2 bnext = cz();
  {
    const int row = lane + WIN;
    if (active && lane < CH && row < n) bnext = x[row];
  }
  for (int q = 0; q < nch; ++q) {
    const int st = q % STAGES;
    const uint32_t ph = (uint32_t)(q / STAGES) & 1u;
    if (lane < CH) myb[lane] = bnext;
    __syncwarp();
    {  // prefetch the next chunk's entering rows
      const int row = (q + 1) * CH + lane + WIN;
      bnext = (active && lane < CH && row < n) ? x[row] : cz();
    }
    mbar_wait(&full[st], ph);
    const double2* panel = stage + (size_t)st * CH * LD;
    const int rows = min(CH, n - q * CH);
    if (active) {
#pragma unroll 4
      for (int t = 0; t < rows; ++t) {
        const double2* col = panel + t * LD;
        double2 cf[NS];
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          const int k = lane + 1 + 32 * sl;
          cf[sl] = k <= W ? col[k] : cz();
        }
        const double2 dinv = col[0];
        const double2 nb = myb[t];
        const double2 v = shfl2(y[0], 0);
        double2 sh[NS];
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          const double2 up = shfl2(y[sl], (lane + 1) & 31);  // row j+1+l+32sl
          const double2 nxt = (sl + 1 < NS) ? shfl2(y[sl + 1 < NS ? sl + 1 : sl], 0) : nb;
          sh[sl] = lane == 31 ? nxt : up;
        }
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) y[sl] = cfms(cf[sl], v, sh[sl]);
        if (lane == 0) x[q * CH + t] = cmul(v, dinv);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (threadIdx.x == 0 && q + STAGES < total) {
      mbar_wait(&empty[st], ph);
      uint32_t bytes;
      const double2* src = chunk_src(q + STAGES, bytes);
      mbar_arrive_expect_tx(&full[st], bytes);
      tma_load_1d(stage + (size_t)st * CH * LD, src, bytes, &full[st]);
    }
  }
  __syncwarp();
  // ---------------- backward sweep: L^T x = z ------------------------------------------
  // lane l of slot sl holds row j - l - 32 sl; coefficient rowband[j][l + 1 + 32 sl]
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    const int row = n - 1 - lane - 32 * sl;
    y[sl] = (active && row >= 0) ? x[row] : cz();
  }
  {
    const int c = nch - 1;
    const int row = c * CH + lane - WIN;
    bnext = (active && lane < CH && row >= 0) ? x[row] : cz();
  }
  for (int qq = 0; qq < nch; ++qq) {
    const int q = nch + qq;
    const int c = nch - 1 - qq;
    const int st = q % STAGES;
    const uint32_t ph = (uint32_t)(q / STAGES) & 1u;
    if (lane < CH) myb[lane] = bnext;
    __syncwarp();
    {
      const int row = (c - 1) * CH + lane - WIN;
      bnext = (active && lane < CH && c > 0 && row >= 0) ? x[row] : cz();
    }
    mbar_wait(&full[st], ph);
    const double2* panel = stage + (size_t)st * CH * LD;
    const int rows = min(CH, n - c * CH);
    if (active) {
#pragma unroll 4
      for (int t = rows - 1; t >= 0; --t) {
        const double2* rw = panel + t * LD;
        double2 cf[NS];
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          const int k = lane + 1 + 32 * sl;
          cf[sl] = k <= W ? rw[k] : cz();
        }
        const double2 nb = myb[t];
        const double2 v = shfl2(y[0], 0);
        double2 sh[NS];
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          const double2 up = shfl2(y[sl], (lane + 1) & 31);
          const double2 nxt = (sl + 1 < NS) ? shfl2(y[sl + 1 < NS ? sl + 1 : sl], 0) : nb;
          sh[sl] = lane == 31 ? nxt : up;
        }
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) y[sl] = cfms(cf[sl], v, sh[sl]);
        if (lane == 0) x[c * CH + t] = v;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (threadIdx.x == 0 && q + STAGES < total) {
      mbar_wait(&empty[st], ph);
      uint32_t bytes;
      const double2* src = chunk_src(q + STAGES, bytes);
      mbar_arrive_expect_tx(&full[st], bytes);
      tma_load_1d(stage + (size_t)st * CH * LD, src, bytes, &full[st]);
    }
  }
}

template <int W, int WARPS, int CH, int STAGES>
constexpr size_t band_solve_smem() {
  return (size_t)STAGES * CH * (W + 1) * sizeof(double2) + 2 * STAGES * sizeof(uint64_t) +
         (size_t)WARPS * CH * sizeof(double2);
}

}  // namespace fetigpu
