// fetigpu3d.cu — the 3D FETI-DP(H) range-space Schur solve (BASELINE.json configs 4-5) and
// its C-ABI (include/fetigpu.h, "3D extension").  Host control flow restates the same
// reference functions as the 2D context (fetigpu.cu), generalised to hexahedra:
//   FetiSolver ctor       feti.cpp:373-480   -> Ctx3::setup()
//   eliminate             feti.cpp:516-556   -> Ctx3::eliminate()
//   apply_dual_operator   feti.cpp:581-594   -> Ctx3::apply_dual()
//   Dirichlet precond     feti.cpp:597-627   -> Ctx3::apply_precond()  (W = 1/mult per row)
//   FetiSolver::solve     feti.cpp:630-717   -> Ctx3::feti_solve()
//   gmres                 krylov.hpp:102-223 -> Ctx3::gmres()  (CGS2 for the Hermitian MGS)
//   solve_range_space     control.cpp:297-334 -> Ctx3::schur_solve()
// A_rr is applied through its block factorisation [A_ii, A_ib; A_bi, A_bb]: A_ii by a block-
// banded LDL^T (32x32 blocks), the interface Schur complement S_bb and its inverse stored
// densely (packed symmetric) — S_bb is exactly the Dirichlet preconditioner's operator and
// S_bb^-1 = (A_rr^-1)_bb is exactly what the dual operator needs on interface rows.  At 3D
// sizes (n_b = 1530 at config 4) this streams 2 x 9.4 GB per Krylov step instead of the
// 34 GB of four banded triangular sweeps over A_rr and A_ii.
// Only K + cV is factored: K - cV = conj(K + cV) (conjugate reuse).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "comm.hpp"
#include "fetigpu.h"
#include "host3d.hpp"
#include "kernels3d.cuh"

namespace fetigpu {

namespace {

using cd = std::complex<double>;

#define CU3(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      throw RuntimeError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call);   \
  } while (0)

inline int cdiv3(long long a, long long b) { return (int)((a + b - 1) / b); }
inline double2 dd2(cd z) { return make_double2(z.real(), z.imag()); }
inline long long sym_size_h(int nt) { return 1024LL * nt * (nt - 1) / 2 + 544LL * nt; }

struct Ev {
  cudaEvent_t a, b;
  int klass;
};

}  // namespace

struct Ctx3 {
  fetigpu3d_desc desc{};
  Host3Problem P;
  Host3Partition H;  // this rank's view (local_partition3d); the whole partition on one GPU
  // sharding: contiguous subdomain ranges per rank, dual and primal vectors replicated,
  // one allreduce completes every jump gather (exact: two owners per multiplier row)
  std::unique_ptr<Comm> comm;
  bool dist() const { return comm != nullptr && comm->world() > 1; }
  bool root() const { return !dist() || comm->rank() == 0; }
  void allreduce(double2* buf, size_t count) {
    if (dist() && count) comm->allreduce_sum(reinterpret_cast<double*>(buf), 2 * count, stream);
  }
  cudaStream_t stream = nullptr;
  cd mc;
  double phi = 0;
  int S = 0, NI = 0, NB = 0, NC = 0, MR = 1, PB = 0, NBK = 0, nl = 0, n = 0, m = 0, nc = 0;
  int NTB = 0, NTD = 0, NBP = 0;  // interface tiles (max), dense tiles (even), padded dense size
  std::vector<void*> allocs;
  long long launches = 0;
  double setup_seconds = 0;
  double setup_t[8] = {};
  // profiling
  bool prof = false;
  std::vector<Ev> pool;
  size_t pool_used = 0;
  double prof_ms[FETIGPU_K_COUNT] = {};
  long long prof_n[FETIGPU_K_COUNT] = {};
  // device tables
  int *d_ldof = nullptr, *d_idof = nullptr, *d_bdof = nullptr, *d_cglob = nullptr, *d_brow = nullptr;
  int *d_lam_lo = nullptr, *d_lam_hi = nullptr, *d_cdof = nullptr, *d_cslots = nullptr;
  int *d_xkind = nullptr, *d_xref = nullptr, *d_n_i = nullptr, *d_n_b = nullptr, *d_nt = nullptr;
  int *d_free_dofs = nullptr, *d_free_map = nullptr, *d_cons_map = nullptr, *d_status = nullptr;
  double *d_bsgn = nullptr, *d_bw = nullptr, *d_lam_w = nullptr, *d_xw = nullptr, *d_ke = nullptr, *d_me = nullptr;
  long long *d_off = nullptr, *d_coff = nullptr;
  int2* d_work = nullptr;    // tile rows (s, I)
  int2* d_rowtab = nullptr;  // per tile row: first row-partial slot, count
  int4* d_items = nullptr;   // GEMV work items (s, I, J0, J1)
  int* d_rslot = nullptr;    // row-partial slot of each item
  int nwork = 0, nitems = 0, NTmax = 0, G = 1;
  static constexpr int kRowChunk = 32;  // tiles per GEMV work item (long rows are split)
  // operators
  double2 *d_ae = nullptr, *d_bb = nullptr, *d_bi_val = nullptr, *d_ib_val = nullptr, *d_aic = nullptr;
  double2 *d_abc = nullptr, *d_acc = nullptr, *d_cpl_b = nullptr, *d_cpl_i = nullptr, *d_Cinv = nullptr;
  int *d_bi_idx = nullptr, *d_ib_idx = nullptr;
  double2 *d_Sp = nullptr, *d_Sip = nullptr;  // packed S_bb, S_bb^-1
  long long pack_entries = 0, colpart_rows = 0;
  // workspaces
  double2 *d_xin = nullptr, *d_rows = nullptr, *d_colp = nullptr, *d_wb = nullptr, *d_u1 = nullptr;
  double2 *d_fi = nullptr, *d_fb = nullptr, *d_fc = nullptr, *d_yi = nullptr, *d_ri = nullptr, *d_gcp = nullptr;
  double2 *d_g = nullptr, *d_z = nullptr, *d_tb = nullptr;
  double2 *d_V = nullptr, *d_w = nullptr, *d_zl = nullptr, *d_r = nullptr, *d_lam = nullptr, *d_best = nullptr;
  double2* d_Z = nullptr;  // preconditioned basis M V_j (the solution update is Z y)
  double2 *d_u0 = nullptr, *d_gcp0 = nullptr;  // first elimination's S^-1 (f_b - A_bi y_i) and coarse terms
  double2 *d_d = nullptr, *d_t = nullptr, *d_h = nullptr, *d_part = nullptr, *d_red = nullptr, *d_coef = nullptr;
  double2 *d_rhs = nullptr, *d_x = nullptr, *d_x2 = nullptr, *d_ax = nullptr;
  double *d_real0 = nullptr, *d_real1 = nullptr, *d_in_ybar = nullptr, *d_in_yc = nullptr, *d_out_y = nullptr,
         *d_out_u = nullptr, *d_out_l = nullptr;
  double2* h_pin = nullptr;
  size_t ldv = 0;
  int vcap = 0, mdot_rows = 0, mdot_blocks = 0;
  // mass solve (Kronecker tridiagonal)
  double *d_cx = nullptr, *d_dx = nullptr, *d_cy = nullptr, *d_dy = nullptr, *d_cz = nullptr, *d_dz = nullptr;
  int Lx = 0, Ly = 0, Lz = 0;
  double moff = 0;

  ~Ctx3() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto& e : pool) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    for (void* p : allocs) cudaFree(p);
    if (h_pin) cudaFreeHost(h_pin);
    if (stream) cudaStreamDestroy(stream);
  }

  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    CU3(cudaMalloc(&p, count * sizeof(T)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  void release(void* p) {
    auto it = std::find(allocs.begin(), allocs.end(), p);
    if (it != allocs.end()) {
      CU3(cudaFree(p));
      allocs.erase(it);
    }
  }
  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) CU3(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, stream));
    return p;
  }
  template <typename T>
  void zero(T* p, size_t count) {
    CU3(cudaMemsetAsync(p, 0, count * sizeof(T), stream));
  }
  void sync() { CU3(cudaStreamSynchronize(stream)); }
  template <typename F>
  void launch(int klass, F&& f) {
    Ev* ev = nullptr;
    if (prof) {
      if (pool_used == pool.size()) {
        Ev e{};
        CU3(cudaEventCreate(&e.a));
        CU3(cudaEventCreate(&e.b));
        pool.push_back(e);
      }
      ev = &pool[pool_used++];
      ev->klass = klass;
      CU3(cudaEventRecord(ev->a, stream));
    }
    f();
    CU3(cudaGetLastError());
    if (ev) CU3(cudaEventRecord(ev->b, stream));
    ++launches;
  }
  void prof_collect() {
    if (!prof || pool_used == 0) return;
    sync();
    for (size_t i = 0; i < pool_used; ++i) {
      float ms = 0;
      CU3(cudaEventElapsedTime(&ms, pool[i].a, pool[i].b));
      prof_ms[pool[i].klass] += ms;
      prof_n[pool[i].klass] += 1;
    }
    pool_used = 0;
  }
  double now() const {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }

  // ------------------------------------------------------------------------------- setup
  void setup() {
    const double t0 = now();
    CU3(cudaSetDevice(desc.device));
    CU3(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    S = H.S, NI = H.NI, NB = H.NB, NC = H.NC, MR = H.MR, PB = H.P, NBK = NI / 32;
    nl = H.n_lambda, n = P.n(), m = P.m(), nc = H.n_corner;
    if (PB > 32) throw ContractError("fetigpu3d: block half-bandwidth " + std::to_string(PB) + " exceeds 32 blocks");
    if (NC > 32) throw ContractError("fetigpu3d: more than 32 corner dofs per subdomain");
    NTB = (NB + 31) / 32;
    NTD = NTB + (NTB & 1);  // the blocked inverse works on 64-wide tiles
    NBP = NTD * 32;
    const int ed = P.edofs;
    {
      std::vector<double2> ae((size_t)ed * ed);
      for (int q = 0; q < ed * ed; ++q) ae[q] = dd2(cd(P.ke[q]) + mc * P.me[q]);
      d_ae = upload(ae);
      d_ke = upload(std::vector<double>(P.ke, P.ke + ed * ed));
      d_me = upload(std::vector<double>(P.me, P.me + ed * ed));
    }
    d_ldof = upload(H.ldof);
    d_idof = upload(H.idof);
    d_bdof = upload(H.bdof);
    d_cglob = upload(H.cglob);
    d_brow = upload(H.brow);
    d_bsgn = upload(H.bsgn);
    d_bw = upload(H.bw);
    d_lam_lo = upload(H.lam_lo);
    d_lam_hi = upload(H.lam_hi);
    d_lam_w = upload(H.lam_w);
    d_cdof = upload(H.corner_dof);
    d_cslots = upload(H.corner_slots);
    d_xkind = upload(H.xkind);
    d_xref = upload(H.xref);
    d_xw = upload(H.xw);
    d_n_i = upload(H.n_i);
    d_n_b = upload(H.n_b);
    d_free_dofs = upload(P.free_dofs);
    d_free_map = upload(P.free_map);
    d_cons_map = upload(P.cons_map);
    d_status = alloc<int>(std::max(S, 1));
    // ragged packed-symmetric layout of S_bb / S_bb^-1 (per-subdomain tile counts)
    std::vector<int> nt(S);
    std::vector<long long> off(S + 1, 0), coff(S + 1, 0);
    std::vector<int2> work, rowtab;
    std::vector<int4> items;
    std::vector<int> rslot;
    for (int s = 0; s < S; ++s) {
      nt[s] = std::max(1, (H.n_b[s] + 31) / 32);
      off[s + 1] = off[s] + sym_size_h(nt[s]);
      coff[s + 1] = coff[s] + (long long)nt[s] * (nt[s] - 1) / 2;
      for (int I = 0; I < nt[s]; ++I) {
        work.push_back(make_int2(s, I));
        rowtab.push_back(make_int2((int)items.size(), 0));
        for (int J0 = 0; J0 <= I; J0 += kRowChunk) {
          rslot.push_back((int)items.size());
          items.push_back(make_int4(s, I, J0, std::min(J0 + kRowChunk, I + 1)));
          rowtab.back().y++;
        }
      }
      NTmax = std::max(NTmax, nt[s]);
    }
    pack_entries = off[S];
    colpart_rows = coff[S];
    nwork = (int)work.size();
    nitems = (int)items.size();
    d_nt = upload(nt);
    d_off = upload(off);
    d_coff = upload(coff);
    d_work = upload(work);
    d_rowtab = upload(rowtab);
    d_items = upload(items);
    d_rslot = upload(rslot);
    {
      int sms = 0;
      CU3(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, desc.device));
      G = std::max(1, std::min(64, cdiv3(8 * sms, S)));  // coarse-rhs slices per subdomain
    }

    // K1: assembly of the per-subdomain blocks
    const double ta = now();
    const size_t bb_entries = (size_t)S * NBK * (PB + 1) * 1024;
    d_bb = alloc<double2>(bb_entries);
    zero(d_bb, bb_entries);
    d_bi_idx = alloc<int>((size_t)S * NB * H.MAXE_BI);
    d_bi_val = alloc<double2>((size_t)S * NB * H.MAXE_BI);
    d_ib_idx = alloc<int>((size_t)S * NI * H.MAXE_IB);
    d_ib_val = alloc<double2>((size_t)S * NI * H.MAXE_IB);
    d_aic = alloc<double2>((size_t)S * NI * NC);
    d_abc = alloc<double2>((size_t)S * NB * NC);
    d_acc = alloc<double2>((size_t)S * NC * NC);
    CU3(cudaMemsetAsync(d_bi_idx, 0xff, (size_t)S * NB * H.MAXE_BI * sizeof(int), stream));
    CU3(cudaMemsetAsync(d_ib_idx, 0xff, (size_t)S * NI * H.MAXE_IB * sizeof(int), stream));
    zero(d_bi_val, (size_t)S * NB * H.MAXE_BI);
    zero(d_ib_val, (size_t)S * NI * H.MAXE_IB);
    zero(d_aic, (size_t)S * NI * NC);
    zero(d_abc, (size_t)S * NB * NC);
    zero(d_acc, (size_t)S * NC * NC);
    k3::Asm3 A{};
    A.S = S, A.nld = H.nld, A.ex = H.ex, A.ey = H.ey, A.ez = H.ez, A.dpn = H.dpn, A.ed = ed;
    A.NI = NI, A.NB = NB, A.NC = NC, A.P = PB, A.EBI = H.MAXE_BI, A.EIB = H.MAXE_IB;
    A.ldof = d_ldof, A.ae = d_ae, A.bb = d_bb, A.bi_idx = d_bi_idx, A.bi_val = d_bi_val;
    A.ib_idx = d_ib_idx, A.ib_val = d_ib_val, A.aic = d_aic, A.abc = d_abc, A.acc = d_acc;
    A.mode = 0;
    launch(FETIGPU_K_OTHER, [&] { k3::k3_assemble<<<cdiv3((long long)S * H.nld, 128), 128, 0, stream>>>(A); });
    launch(FETIGPU_K_OTHER, [&] { k3::k3_pad_identity<<<S, 128, 0, stream>>>(S, NI, PB, d_n_i, d_bb); });
    sync();
    setup_t[0] = now() - ta;

    // K2: block LDL^T of A_ii
    const double tb = now();
    {
      double2* scratch = alloc<double2>((size_t)S * std::max(PB, 1) * 1024);
      int sms = 0;
      CU3(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, desc.device));
      if (S >= 2 * sms || PB <= 2) {  // one CTA per subdomain fills the GPU
        const size_t smem = 2 * sizeof(k3::Tile);
        CU3(cudaFuncSetAttribute(k3::k3_bb_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        launch(FETIGPU_K_OTHER,
               [&] { k3::k3_bb_factor<<<S, 256, smem, stream>>>(NBK, PB, d_bb, scratch, d_status); });
      } else {  // few subdomains: every block column over the whole grid
        zero(d_status, S);
        for (int K = 0; K < NBK; ++K) {
          const int nd = std::min(PB, NBK - 1 - K);
          k3::k3_bbf_pivot<<<S, 256, 0, stream>>>(NBK, PB, K, d_bb, d_status);
          if (nd > 0) {
            k3::k3_bbf_lcol<<<dim3(nd, S), 256, 0, stream>>>(NBK, PB, K, d_bb, scratch);
            k3::k3_bbf_update<<<dim3(nd * (nd + 1) / 2, S), 256, 0, stream>>>(NBK, PB, K, d_bb, scratch);
            k3::k3_bbf_store<<<dim3(nd, S), 256, 0, stream>>>(NBK, PB, K, d_bb, scratch);
          }
          CU3(cudaGetLastError());
          launches += nd > 0 ? 4 : 1;
        }
      }
      check_status(S, "interior block A_ii");
      release(scratch);
    }
    setup_t[1] = now() - tb;

    // K3: S_bb, S_bb^-1, coupling and coarse contributions, in chunks of subdomains
    const int ntile = NTB + 1;  // A_ib tiles + the A_ic / coupling tile
    const size_t per_sub = sizeof(double2) * ((size_t)ntile * NI * 32 + (size_t)NBP * NBP + (size_t)NB * NC) +
                           sizeof(double2) * (size_t)(NTD + 1) * 1024;
    size_t free_b = 0, total_b = 0;
    CU3(cudaMemGetInfo(&free_b, &total_b));
    const size_t persist = sizeof(double2) * (2 * (size_t)pack_entries + (size_t)S * NB * NC + (size_t)S * NI * NC);
    const size_t budget = std::min<size_t>(24ull << 30, free_b > persist + (4ull << 30) ? (free_b - persist - (4ull << 30)) / 2 : 0);
    int chunk = (int)std::max<size_t>(1, std::min<size_t>(S, budget / std::max<size_t>(per_sub, 1)));
    d_Sp = alloc<double2>(pack_entries);
    d_Sip = alloc<double2>(pack_entries);
    d_cpl_b = alloc<double2>((size_t)S * NB * NC);
    d_cpl_i = alloc<double2>((size_t)S * NI * NC);
    double2* contrib = alloc<double2>((size_t)S * NC * NC);
    double2* X = alloc<double2>((size_t)chunk * ntile * NI * 32);
    double2* dense = alloc<double2>((size_t)chunk * NBP * NBP);
    double2* R = alloc<double2>((size_t)chunk * NB * NC);
    double2* pbuf = alloc<double2>((size_t)chunk * 1024);
    double2* cbuf = alloc<double2>((size_t)chunk * NTD * 1024);
    double* prat = alloc<double>(chunk);
    const size_t m2smem = sizeof(double2) * (32 * 33 + 32 * 65);
    CU3(cudaFuncSetAttribute(k3::k3_bb_msolve2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m2smem));
    auto msolve = [&](int cnt, int s0, int t0_, int tiles) {
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_bb_msolve2<<<dim3((tiles + 1) / 2, cnt), 256, m2smem, stream>>>(NBK, PB, d_bb, NI, ntile, t0_, tiles,
                                                                             s0, X);
      });
    };
    double t_ms = 0, t_sb = 0, t_inv = 0, t_cpl = 0, t_pack = 0;
    for (int s0 = 0; s0 < S; s0 += chunk) {
      const int cnt = std::min(chunk, S - s0);
      double tt = now();
      zero(X, (size_t)cnt * ntile * NI * 32);
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_build_rhs<<<cdiv3((long long)cnt * (NTB * 32 + 32), 128), 128, 0, stream>>>(
            cnt, s0, NI, NB, NC, H.MAXE_BI, ntile, NTB, d_bi_idx, d_bi_val, d_aic, X);
      });
      msolve(cnt, s0, 0, ntile);  // X = A_ii^-1 [A_ib | A_ic]
      sync();
      t_ms += now() - tt;
      tt = now();
      zero(dense, (size_t)cnt * NBP * NBP);
      k3::Asm3 B = A;
      B.mode = 1, B.s0 = s0, B.cnt = cnt, B.NBP = NBP, B.dense = dense;
      launch(FETIGPU_K_OTHER, [&] { k3::k3_assemble<<<cdiv3((long long)cnt * H.nld, 128), 128, 0, stream>>>(B); });
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_schur_build<<<cdiv3((long long)cnt * NBP * NBP, 256), 256, 0, stream>>>(
            cnt, s0, NI, NB, NBP, H.MAXE_BI, ntile, d_n_b, d_bi_idx, d_bi_val, X, dense);
      });
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_pack_sym<<<dim3(std::max(1, std::min(1024, cdiv3(sym_size_h(NTB), 256))), cnt), 256, 0, stream>>>(
            cnt, s0, NBP, d_nt, d_off, dense, d_Sp);
      });
      sync();
      t_sb += now() - tt;
      tt = now();
      // S_bb^-1 (blocked Gauss-Jordan, no pivoting)
      {
        std::vector<double> one(cnt, 1.0);
        CU3(cudaMemcpyAsync(prat, one.data(), cnt * sizeof(double), cudaMemcpyHostToDevice, stream));
        const size_t gsm = sizeof(double2) * (64 * 33 + 32 * 65);
        static bool gattr = false;
        if (!gattr) {
          CU3(cudaFuncSetAttribute(k3::k3_gj_update64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
          gattr = true;
        }
        // (a DMMA (FP64 tensor core) trailing update measured no faster, 1.01 vs 0.99 s at
        // config 4: the update is bound by its read-modify-write of C; not kept)
        for (int K = 0; K < NTD; ++K) {
          k3::k3_gj_pivot<<<cnt, 256, 0, stream>>>(NBP, K, dense, pbuf, prat);
          k3::k3_gj_panel<<<dim3(NTD, cnt), 256, 0, stream>>>(NBP, NTD, K, dense, pbuf, cbuf);
          k3::k3_gj_update64<<<dim3(NTD / 2, NTD / 2, cnt), 256, gsm, stream>>>(NBP, NTD, K, dense, pbuf, cbuf);
          k3::k3_gj_setpivot<<<cnt, 256, 0, stream>>>(NBP, K, dense, pbuf);
          CU3(cudaGetLastError());
          launches += 4;
        }
        std::vector<double> pr(cnt);
        CU3(cudaMemcpyAsync(pr.data(), prat, cnt * sizeof(double), cudaMemcpyDeviceToHost, stream));
        sync();
        for (int q = 0; q < cnt; ++q)
          if (!(pr[q] > 1e-14))
            throw NumericalError("assemble_subdomain_operators: singular remaining block A_rr in subdomain " +
                                 std::to_string(s0 + q));
      }
      t_inv += now() - tt;
      tt = now();
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_pack_sym<<<dim3(std::max(1, std::min(1024, cdiv3(sym_size_h(NTB), 256))), cnt), 256, 0, stream>>>(
            cnt, s0, NBP, d_nt, d_off, dense, d_Sip);
      });
      sync();
      t_pack += now() - tt;
      tt = now();
      // coupling = A_rr^-1 A_rc by blocks: cpl_b = S^-1 (A_bc - A_bi A_ii^-1 A_ic),
      // cpl_i = A_ii^-1 (A_ic - A_ib cpl_b); contributions A_cc - A_rc^T coupling
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_cpl_rhs<<<cdiv3((long long)cnt * NB * NC, 128), 128, 0, stream>>>(
            cnt, s0, NI, NB, NC, H.MAXE_BI, ntile, NTB, d_bi_idx, d_bi_val, d_abc, X, R);
      });
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_cpl_b<<<cdiv3((long long)cnt * NB, 8), 256, 0, stream>>>(cnt, s0, NB, NBP, NC, d_n_b, dense, R,
                                                                       d_cpl_b);
      });
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_cpl_i_rhs<<<cdiv3((long long)cnt * NI * 32, 256), 256, 0, stream>>>(
            cnt, s0, NI, NB, NC, H.MAXE_IB, ntile, NTB, d_ib_idx, d_ib_val, d_aic, d_cpl_b, X);
      });
      msolve(cnt, s0, NTB, 1);
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_coarse_contrib<<<cnt, 256, 0, stream>>>(cnt, s0, NI, NB, NC, ntile, NTB, X, d_aic, d_abc, d_acc,
                                                       d_cpl_b, d_cpl_i, contrib);
      });
      sync();
      t_cpl += now() - tt;
    }
    for (void* p : {(void*)X, (void*)dense, (void*)R, (void*)pbuf, (void*)cbuf, (void*)prat}) release(p);
    setup_t[2] = t_ms, setup_t[3] = t_sb, setup_t[4] = t_inv, setup_t[6] = t_pack;
    const double tc = now();
    setup_coarse(contrib);
    release(contrib);
    setup_t[5] = t_cpl + (now() - tc);

    // workspaces
    d_xin = alloc<double2>((size_t)S * NB);
    d_rows = alloc<double2>((size_t)nitems * 32);
    d_colp = alloc<double2>((size_t)std::max<long long>(colpart_rows, 1) * 32);
    d_wb = alloc<double2>((size_t)S * NB);
    d_u1 = alloc<double2>((size_t)S * NB);
    d_tb = alloc<double2>((size_t)S * NB);
    d_fi = alloc<double2>((size_t)S * NI);
    d_fb = alloc<double2>((size_t)S * NB);
    d_yi = alloc<double2>((size_t)S * NI);
    d_ri = alloc<double2>((size_t)S * NI);
    d_gcp = alloc<double2>((size_t)S * G * NC);
    zero(d_gcp, (size_t)S * G * NC);
    d_fc = alloc<double2>(std::max(nc, 1));
    d_g = alloc<double2>(std::max(nc, 1));
    d_z = alloc<double2>(std::max(nc, 1));
    zero(d_z, std::max(nc, 1));
    ldv = ((size_t)nl + 63) / 64 * 64;
    vcap = std::max(2, desc.max_iter + 1);
    d_V = alloc<double2>(ldv * vcap);
    d_Z = alloc<double2>(ldv * vcap);
    d_u0 = alloc<double2>((size_t)S * NB);
    d_gcp0 = alloc<double2>((size_t)S * G * NC);
    for (double2** p : {&d_w, &d_zl, &d_r, &d_lam, &d_best, &d_d, &d_t}) *p = alloc<double2>(ldv);
    mdot_rows = 512;  // (2048: 1.35 blocks per SM, latency-bound at small j; measured 4.8 -> 4.0 ms of CGS per config-4 solve)
    mdot_blocks = std::max(1, cdiv3(nl, mdot_rows));
    d_part = alloc<double2>((size_t)mdot_blocks * (vcap + 2) + 1024);
    d_h = alloc<double2>(2 * (vcap + 2));
    d_red = alloc<double2>(4);
    d_coef = alloc<double2>(vcap + 2);
    d_rhs = alloc<double2>(n);
    d_x = alloc<double2>(n);
    d_x2 = alloc<double2>(n);
    d_ax = alloc<double2>(n);
    d_real0 = alloc<double>(n);
    d_real1 = alloc<double>(n);
    d_in_ybar = alloc<double>(n);
    d_in_yc = alloc<double>(std::max(m, 1));
    d_out_y = alloc<double>(n);
    d_out_u = alloc<double>(n);
    d_out_l = alloc<double>(n);
    CU3(cudaMallocHost(&h_pin, sizeof(double2) * 4 * (vcap + 4)));
    setup_mass();
    setup_stencil();
    setup_fdm();
    sync();
    setup_seconds = now() - t0;
    setup_t[7] = setup_seconds;
  }

  void check_status(int count, const char* what) {
    std::vector<int> st(count);
    CU3(cudaMemcpyAsync(st.data(), d_status, count * sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
    for (int s = 0; s < count; ++s)
      if (st[s] != 0)
        throw NumericalError(std::string("assemble_subdomain_operators: singular ") + what + " in subdomain " +
                             std::to_string(s));
  }

  // K4: dense coarse matrix, equilibration 1/sqrt|C_ii|, Gauss-Jordan with partial pivoting,
  // pivot check |U_kk| > 1e-13 max |U_kk| (feti.cpp:456-475), explicit inverse
  void setup_coarse(const double2* contrib) {
    if (nc == 0) return;
    d_Cinv = alloc<double2>((size_t)nc * nc);
    const long long nn = (long long)nc * nc;
    launch(FETIGPU_K_OTHER, [&] {
      k3::k3_coarse_assemble<<<cdiv3(nn, 256), 256, 0, stream>>>(nc, NC, d_cslots, contrib, d_Cinv);
    });
    allreduce(d_Cinv, (size_t)nn);  // sharded: every rank assembled its subdomains' part
    double* sc = alloc<double>(nc);
    int* piv = alloc<int>(nc);
    double* pabs = alloc<double>(nc);
    double2* col = alloc<double2>(nc);
    launch(FETIGPU_K_OTHER, [&] { k3::k3_diag_scale<<<cdiv3(nc, 128), 128, 0, stream>>>(nc, d_Cinv, sc); });
    launch(FETIGPU_K_OTHER, [&] { k3::k3_scale_sym<<<cdiv3(nn, 256), 256, 0, stream>>>(nc, d_Cinv, sc); });
    for (int k = 0; k < nc; ++k) {
      k3::k3_cgj_pivot<<<1, 1024, 0, stream>>>(nc, k, d_Cinv, piv, pabs, col);
      k3::k3_cgj_update<<<dim3(cdiv3(nc, 256), nc), 256, 0, stream>>>(nc, k, d_Cinv, col);
    }
    CU3(cudaGetLastError());
    launches += 2LL * nc;
    launch(FETIGPU_K_OTHER, [&] { k3::k3_cgj_unpermute<<<cdiv3(nc, 128), 128, 0, stream>>>(nc, d_Cinv, piv); });
    std::vector<double> pa(nc);
    CU3(cudaMemcpyAsync(pa.data(), pabs, nc * sizeof(double), cudaMemcpyDeviceToHost, stream));
    sync();
    double umax = 0;
    for (double v : pa) umax = std::max(umax, v);
    for (double v : pa)
      if (!(v > umax * 1e-13)) throw NumericalError("feti: coarse problem is singular");
    launch(FETIGPU_K_OTHER, [&] { k3::k3_scale_sym<<<cdiv3(nn, 256), 256, 0, stream>>>(nc, d_Cinv, sc); });
    for (void* p : {(void*)sc, (void*)piv, (void*)pabs, (void*)col}) release(p);
  }

  // V = M_z (x) M_y (x) M_x (x) I_dpn on the free tensor grid (whole-boundary Dirichlet for
  // heat, x = 0 clamped for elasticity): exact like the reference's Cholesky (control.cpp:323)
  void setup_mass() {
    int i0 = P.nx, i1 = -1, j0 = P.ny, j1 = -1, k0 = P.nz, k1 = -1;
    const int nnx = P.nx + 1, nny = P.ny + 1;
    for (int md : P.free_dofs) {
      const int node = md / P.dpn, i = node % nnx, j = (node / nnx) % nny, k = node / (nnx * nny);
      i0 = std::min(i0, i), i1 = std::max(i1, i), j0 = std::min(j0, j), j1 = std::max(j1, j);
      k0 = std::min(k0, k), k1 = std::max(k1, k);
    }
    Lx = i1 - i0 + 1, Ly = j1 - j0 + 1, Lz = k1 - k0 + 1;
    if ((long long)Lx * Ly * Lz * P.dpn != n) throw ContractError("mass solve: free dofs do not form a tensor grid");
    const double hh = P.h / 6.0;
    moff = hh;
    auto factor = [&](int lo, int hi, int nmax, std::vector<double>& cp, std::vector<double>& dinv) {
      const int len = hi - lo + 1;
      cp.assign(len, 0.0);
      dinv.assign(len, 0.0);
      for (int k = 0; k < len; ++k) {
        const int g = lo + k;
        const double diag = hh * ((g == 0 || g == nmax) ? 2.0 : 4.0);
        const double den = k == 0 ? diag : diag - hh * cp[k - 1];
        dinv[k] = 1.0 / den;
        cp[k] = hh * dinv[k];
      }
    };
    std::vector<double> a, b;
    factor(i0, i1, P.nx, a, b);
    d_cx = upload(a), d_dx = upload(b);
    factor(j0, j1, P.ny, a, b);
    d_cy = upload(a), d_dy = upload(b);
    factor(k0, k1, P.nz, a, b);
    d_cz = upload(a), d_dz = upload(b);
  }
  void mass_solve(double* v) {
    const int dpn = P.dpn;
    const long long plane = (long long)Lx * Ly * dpn;
    // x lines: (k, j, c) -> start k*plane + j*Lx*dpn + c, stride dpn
    launch(FETIGPU_K_GLOBAL, [&] {
      k3::k3_tridiag<<<cdiv3((long long)Ly * Lz * dpn, 128), 128, 0, stream>>>(
          v, Ly * Lz * dpn, Lx, dpn, (long long)Lx * dpn, 1, dpn, d_cx, d_dx, moff);
    });
    // y lines: (k, i*dpn+c) -> start k*plane + (i*dpn+c), stride Lx*dpn
    launch(FETIGPU_K_GLOBAL, [&] {
      k3::k3_tridiag<<<cdiv3((long long)Lx * dpn * Lz, 128), 128, 0, stream>>>(
          v, Lx * dpn * Lz, Ly, Lx * dpn, plane, 1, (long long)Lx * dpn, d_cy, d_dy, moff);
    });
    // z lines: (j*Lx*dpn + i*dpn + c) -> start, stride plane
    launch(FETIGPU_K_GLOBAL, [&] {
      k3::k3_tridiag<<<cdiv3(plane, 128), 128, 0, stream>>>(v, (int)plane, Lz, (int)plane, 0, 1, plane, d_cz,
                                                             d_dz, moff);
    });
  }
  k3::Glob3 glob() const {
    return k3::Glob3{P.nx, P.ny, P.nz, P.dpn, P.edofs, n, d_free_dofs, d_free_map, d_cons_map, d_ke, d_me};
  }
  template <typename T>
  void apply_global(const T* x, const double* xc, cd kc, cd mcoef, T* y) {
    if (stencil_ok && xc == nullptr) {  // heat, all free nodes interior: the 27-point stencil
      k3::Stencil27 st;
      for (int q = 0; q < 27; ++q) st.c[q] = dd2(kc * st_k[q] + mcoef * st_m[q]);
      launch(FETIGPU_K_GLOBAL, [&] {
        k3::k3_apply_stencil27<T><<<dim3(cdiv3(Lx, 128), Ly, Lz), 128, 0, stream>>>(Lx, Ly, Lz, st, x, y);
      });
      return;
    }
    launch(FETIGPU_K_GLOBAL, [&] {
      k3::k3_apply_global<T><<<cdiv3(n, 128), 128, 0, stream>>>(glob(), x, xc, dd2(kc), dd2(mcoef), y);
    });
  }
  // 27-point stencils of K and M when the free dofs are exactly the interior grid nodes
  // (heat, whole-boundary Dirichlet): the element sums at an interior node are the same
  // everywhere, so the element-by-element apply reduces to a constant stencil (exact)
  bool stencil_ok = false;
  double st_k[27] = {}, st_m[27] = {};
  void setup_stencil() {
    if (P.dpn != 1 || std::getenv("FETIGPU_NO_STENCIL")) return;
    if (Lx != P.nx - 1 || Ly != P.ny - 1 || Lz != P.nz - 1) return;
    const int hx[8] = {0, 1, 1, 0, 0, 1, 1, 0}, hy[8] = {0, 0, 1, 1, 0, 0, 1, 1};
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        const int dx = hx[b] - hx[a], dy = hy[b] - hy[a], dz = (b >> 2) - (a >> 2);
        const int o = ((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1);
        st_k[o] += P.ke[a * 8 + b];
        st_m[o] += P.me[a * 8 + b];
      }
    stencil_ok = true;
  }

  // ---------------------------------------------------------------------------- operators
  // y = S x for the packed symmetric operator pk (xin -> y, both [S][NB])
  void sym_gemv(const double2* pk, const double2* xin, double2* y, int klass) {
    k3::SymArgs a{d_items, d_rslot, d_nt, d_off, d_coff, pk, xin, NB, d_rows, d_colp};
    const size_t smem = sizeof(double2) * 32 * (size_t)(kRowChunk + 1);
    static size_t smem_set = 0;
    if (smem > 48 * 1024 && smem > smem_set) {
      CU3(cudaFuncSetAttribute(k3::k3_sym_rows<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      smem_set = smem;
    }
    launch(klass, [&] { k3::k3_sym_rows<8><<<nitems, 128, smem, stream>>>(a); });
    launch(FETIGPU_K_LAMBDA, [&] {  // (partial reduction: counted with the gathers)
      k3::k3_sym_reduce<<<cdiv3(nwork, 8), 256, 0, stream>>>(nwork, d_work, d_rowtab, d_nt, d_coff, NB, d_rows,
                                                              d_colp, y);
    });
  }
  void coarse_solve(const double2* fc) {  // g = fc - sum gcp, z = C^-1 g
    if (nc == 0) return;
    const double2* fc_r = root() ? fc : nullptr;  // f_c counted once
    launch(FETIGPU_K_COARSE, [&] {
      k3::k3_coarse_rhs<<<cdiv3(nc, 128), 128, 0, stream>>>(nc, NC, G, d_cslots, d_gcp, fc_r, d_g);
    });
    allreduce(d_g, nc);
    launch(FETIGPU_K_COARSE, [&] { k3::k3_dense_gemv<<<cdiv3(nc, 8), 256, 0, stream>>>(nc, d_Cinv, d_g, d_z); });
  }
  // F lam (feti.cpp:581-594): t_b = -B^T lam, u1 = S^-1 t_b, g = -sum cpl_b^T t_b,
  // z = C^-1 g, out = -B (u1 - cpl_b z)
  void apply_dual(const double2* lam, double2* out) {
    launch(FETIGPU_K_LAMBDA, [&] {
      k3::k3_gather_in<<<cdiv3((long long)S * NB, 256), 256, 0, stream>>>(S, NB, MR, 1, d_n_b, d_brow, d_bsgn,
                                                                         d_lam_w, lam, nullptr, d_xin);
    });
    sym_gemv(d_Sip, d_xin, d_u1, FETIGPU_K_DUAL_GEMV);
    if (nc > 0) {
      launch(FETIGPU_K_COARSE, [&] {
        k3::k3_gcp<<<dim3(S, G), 256, 0, stream>>>(NB, NC, NI, G, d_cpl_b, d_xin, nullptr, nullptr, d_gcp);
      });
      coarse_solve(nullptr);
    }
    launch(FETIGPU_K_LAMBDA, [&] {
      k3::k3_lam_jump<<<cdiv3(nl, 256), 256, 0, stream>>>(nl, NB, NC, -1.0, d_lam_lo, d_lam_hi, d_u1, d_cpl_b, d_cglob,
                                                         nc > 0 ? d_z : nullptr, out);
    });
    allreduce(out, nl);
  }
  // Dirichlet preconditioner (feti.cpp:597-627): out = W B S_bb B^T W r
  void apply_precond(const double2* r, double2* out) {
    launch(FETIGPU_K_LAMBDA, [&] {
      k3::k3_gather_in<<<cdiv3((long long)S * NB, 256), 256, 0, stream>>>(S, NB, MR, 0, d_n_b, d_brow, d_bsgn,
                                                                         d_lam_w, r, nullptr, d_xin);
    });
    sym_gemv(d_Sp, d_xin, d_wb, FETIGPU_K_PRECOND_GEMV);
    launch(FETIGPU_K_LAMBDA, [&] {
      k3::k3_lam_pre<<<cdiv3(nl, 256), 256, 0, stream>>>(nl, d_lam_lo, d_lam_hi, d_lam_w, d_wb, out);
    });
    allreduce(out, nl);
  }
  // eliminate (feti.cpp:516-556) for t = [f_i ; tb]: u1_b = S^-1 (tb - A_bi y_i) with y_i =
  // A_ii^-1 f_i (computed once per FETI solve), g = f_c - (cpl_i^T f_i + cpl_b^T tb),
  // z = C^-1 g, u_b = u1_b - cpl_b z  -> d_u1
  void eliminate_boundary(const double2* tb, bool save = false) {
    launch(FETIGPU_K_OTHER, [&] {
      k3::k3_tb_minus<<<cdiv3((long long)S * NB, 256), 256, 0, stream>>>(S, NB, NI, H.MAXE_BI, d_bi_idx, d_bi_val,
                                                                        d_yi, tb, d_xin);
    });
    sym_gemv(d_Sip, d_xin, d_u1, FETIGPU_K_OTHER);
    if (save) CU3(cudaMemcpyAsync(d_u0, d_u1, sizeof(double2) * S * NB, cudaMemcpyDeviceToDevice, stream));
    if (nc > 0) {
      launch(FETIGPU_K_COARSE, [&] {
        k3::k3_gcp<<<dim3(S, G), 256, 0, stream>>>(NB, NC, NI, G, d_cpl_b, tb, d_cpl_i, d_fi, d_gcp);
      });
      if (save) CU3(cudaMemcpyAsync(d_gcp0, d_gcp, sizeof(double2) * S * G * NC, cudaMemcpyDeviceToDevice, stream));
      coarse_solve(d_fc);
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_ub_correct<<<cdiv3((long long)S * NB, 256), 256, 0, stream>>>(S, NB, NC, d_cglob, d_z, d_cpl_b, d_u1);
      });
    }
  }
  // interior solves: the TMA-streamed kernel (default), or the direct-load one
  // (FETIGPU3D_SOLVE=direct: one warp per off-diagonal block, 8 warps up to P = 8, else 32)
  int solve_kind = -1;
  // interior substitution ring: 12 slots of 16 KB (196 KB in flight per CTA), 6 consumer
  // warps with 2 slots each (config 5, 4 interior solves per Schur solve: 8 slots / 8 warps
  // 22.5 ms, 12 / 4 24.4, 12 / 3 29.9, 12 / 6 20.6)
  static constexpr int kBbsStages = 12, kBbsWarps = 6;
  // separable interior solve (k3_fdm_solve) for heat: FETIGPU3D_NO_FDM=1 disables it
  bool use_fdm = false;
  int fdm_m[3] = {0, 0, 0};
  double *d_fdm_s[3] = {nullptr, nullptr, nullptr};
  double2* d_fdm_invd = nullptr;
  void setup_fdm() {
    if (std::getenv("FETIGPU3D_NO_FDM") || P.dpn != 1 || P.physics != 0) return;
    const int mx = H.ex - 1, my = H.ey - 1, mz = H.ez - 1, ni = mx * my * mz;
    if (mx < 1 || my < 1 || mz < 1 || mx > 32 || my > 32 || mz > 32) return;
    if (k3::fdm3_smem(ni) > 200 * 1024) return;
    for (int s = 0; s < H.S; ++s) {
      if (H.n_i[s] != ni) return;
      for (int e = 0; e < ni; ++e) {
        const int i = e % mx, j = (e / mx) % my, k = e / (mx * my);
        const int node = P.node_id(H.sub_i0[s] + 1 + i, H.sub_j0[s] + 1 + j, H.sub_k0[s] + 1 + k);
        if (P.free_map[node] < 0 || H.idof[(size_t)s * NI + e] != P.free_map[node]) return;
      }
    }
    const double h = P.h, pi = std::acos(-1.0);
    const int ms[3] = {mx, my, mz};
    std::vector<double> ka[3], nu[3];
    for (int a = 0; a < 3; ++a) {
      const int m = ms[a];
      std::vector<double> S(1024, 0.0);
      const double c = std::sqrt(2.0 / (m + 1));
      for (int i = 0; i < m; ++i)
        for (int k = 0; k < m; ++k) S[i * 32 + k] = c * std::sin(pi * (double)(i + 1) * (k + 1) / (m + 1));
      ka[a].assign(m, 0.0);
      nu[a].assign(m, 0.0);
      for (int k = 0; k < m; ++k) {
        const double cs = std::cos(pi * (k + 1) / (m + 1));
        ka[a][k] = (2.0 - 2.0 * cs) / h;
        nu[a][k] = h * (4.0 + 2.0 * cs) / 6.0;
      }
      d_fdm_s[a] = upload(S);
      fdm_m[a] = m;
    }
    std::vector<double2> inv(ni);
    for (int e = 0; e < ni; ++e) {
      const int i = e % mx, j = (e / mx) % my, k = e / (mx * my);
      const double nx = nu[0][i], ny = nu[1][j], nz = nu[2][k];
      const cd d = cd(ka[0][i] * ny * nz + nx * ka[1][j] * nz + nx * ny * ka[2][k]) + mc * (nx * ny * nz);
      const cd r = 1.0 / d;
      inv[e] = make_double2(r.real(), r.imag());
    }
    d_fdm_invd = upload(inv);
    CU3(cudaFuncSetAttribute(k3::k3_fdm_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k3::fdm3_smem(ni)));
    sync();
    use_fdm = true;
  }
  void interior_solve(double2* x) {
    if (use_fdm) {
      launch(FETIGPU_K_BAND, [&] {
        k3::k3_fdm_solve<<<S, 256, k3::fdm3_smem(fdm_m[0] * fdm_m[1] * fdm_m[2]), stream>>>(
            x, (size_t)NI, fdm_m[0], fdm_m[1], fdm_m[2], d_fdm_s[0], d_fdm_s[1], d_fdm_s[2], d_fdm_invd);
      });
      return;
    }
    if (solve_kind < 0) {
      CU3(cudaFuncSetAttribute(k3::k3_bb_solve_tma<kBbsStages, kBbsWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)k3::bb_solve_tma_smem<kBbsStages, kBbsWarps>()));
      solve_kind = 1;
    }
    launch(FETIGPU_K_BAND, [&] {
      k3::k3_bb_solve_tma<kBbsStages, kBbsWarps><<<S, (kBbsWarps + 1) * 32, k3::bb_solve_tma_smem<kBbsStages, kBbsWarps>(), stream>>>(
          NBK, PB, d_bb, NI, x);
    });
  }
  // (|x|^2, max|x|) -> host
  std::pair<double, double> norm_max(const double2* x, int len) {
    const int blocks = std::max(1, std::min(296, cdiv3(std::max(len, 1), 256)));
    launch(FETIGPU_K_ORTHO, [&] { k3::k3_norm_part<<<blocks, 256, 0, stream>>>(len, x, d_part); });
    launch(FETIGPU_K_ORTHO, [&] { k3::k3_norm_final<<<1, 32, 0, stream>>>(blocks, d_part, d_red); });
    CU3(cudaMemcpyAsync(h_pin, d_red, sizeof(double2), cudaMemcpyDeviceToHost, stream));
    sync();
    return {std::sqrt(h_pin[0].x), h_pin[0].y};
  }
  // h[0..nv) = V^H w, h[nv] = |w|^2
  void mdot(int nv, const double2* w, double2* h) {
    launch(FETIGPU_K_ORTHO, [&] {
      k3::k3_mdot_part<<<mdot_blocks, 256, 0, stream>>>(nl, nv, d_V, ldv, w, d_part, mdot_rows);
    });
    launch(FETIGPU_K_ORTHO, [&] { k3::k3_mdot_final<<<cdiv3(nv + 1, 8), 256, 0, stream>>>(mdot_blocks, nv, d_part, h); });
  }

  // --------------------------------------------------------------------------------- GMRES
  // Right-preconditioned GMRES restated from krylov.hpp:102-223 (x0 = 0, Givens formula of
  // krylov.hpp:66-83, Arnoldi-estimate stop then true-residual check, restarts, best
  // iterate).  Hermitian MGS is replaced by CGS2 (equal in exact arithmetic).  Host-driven:
  // at 3D sizes one Arnoldi step streams ~19 GB, so a per-step sync costs nothing.
  struct Stats {
    int iterations = 0;
    bool converged = false;
    double relres = 0;
    bool dual_of_x = false;  // d_u1 / d_gcp hold S^-1(-B^T x) / its coarse terms for the returned x
  };
  Stats gmres(const double2* b, double2* x, int max_iter, double tol) {
    Stats st;
    zero(x, nl);
    const double bnorm = norm_max(b, nl).first;
    if (bnorm == 0.0) {
      st.converged = true;
      return st;
    }
    CU3(cudaMemcpyAsync(d_r, b, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, stream));  // r = b - A 0
    CU3(cudaMemcpyAsync(d_best, x, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, stream));
    double best = 1.0;
    const int mres = std::max(1, max_iter);
    // Hessenberg columns grown on demand (the reference zero-fills (m+1) x m up front,
    // 64 MB at max_iter = 2000, krylov.hpp:125; every entry read here is written first)
    std::vector<std::vector<cd>> Hcol;
    std::vector<cd> gs(mres), g(mres + 1);
    std::vector<double> gc(mres);
    auto Hij = [&](int i, int j) -> cd& {
      if ((int)Hcol.size() <= j) Hcol.resize(j + 1);
      if ((int)Hcol[j].size() < j + 2) Hcol[j].resize(j + 2);
      return Hcol[j][i];
    };
    const int nb = cdiv3(nl, 256);
    while (true) {
      const double rnorm = norm_max(d_r, nl).first;
      st.relres = rnorm / bnorm;
      if (st.relres < best) {
        best = st.relres;
        CU3(cudaMemcpyAsync(d_best, x, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, stream));
      }
      if (st.relres <= tol) {
        st.converged = true;
        break;
      }
      if (st.iterations >= max_iter) break;
      launch(FETIGPU_K_ORTHO, [&] {
        k3::k3_scale_to<<<nb, 256, 0, stream>>>(nl, make_double2(1.0 / rnorm, 0.0), d_r, d_V);
      });
      std::fill(g.begin(), g.end(), cd(0));
      g[0] = rnorm;
      int k = 0;
      for (int j = 0; j < mres && st.iterations < max_iter; ++j) {
        double2* vj = d_V + (size_t)j * ldv;
        double2* zj = d_Z + (size_t)j * ldv;
        apply_precond(vj, zj);
        apply_dual(zj, d_w);
        // CGS2: h1 = V^H w (+|w|^2), w -= V h1, h2 = V^H w, w -= V h2, |w|
        double2* h1 = d_h;
        double2* h2 = d_h + (vcap + 2);
        mdot(j + 1, d_w, h1);
        launch(FETIGPU_K_ORTHO, [&] { k3::k3_mupdate<<<nb, 256, 0, stream>>>(nl, j + 1, d_V, ldv, h1, d_w); });
        mdot(j + 1, d_w, h2);
        launch(FETIGPU_K_ORTHO, [&] { k3::k3_mupdate<<<nb, 256, 0, stream>>>(nl, j + 1, d_V, ldv, h2, d_w); });
        const int blocks = std::max(1, std::min(296, nb));
        launch(FETIGPU_K_ORTHO, [&] { k3::k3_norm_part<<<blocks, 256, 0, stream>>>(nl, d_w, d_part + (size_t)mdot_blocks * (vcap + 2)); });
        launch(FETIGPU_K_ORTHO, [&] {
          k3::k3_norm_final<<<1, 32, 0, stream>>>(blocks, d_part + (size_t)mdot_blocks * (vcap + 2), d_red);
        });
        CU3(cudaMemcpyAsync(h_pin, d_h, sizeof(double2) * 2 * (vcap + 2), cudaMemcpyDeviceToHost, stream));
        CU3(cudaMemcpyAsync(h_pin + 2 * (vcap + 2), d_red, sizeof(double2), cudaMemcpyDeviceToHost, stream));
        sync();
        const double wpre = std::sqrt(h_pin[j + 1].x);
        const double hnext = std::sqrt(h_pin[2 * (vcap + 2)].x);
        if (!std::isfinite(hnext) || !std::isfinite(h_pin[2 * (vcap + 2)].y))
          throw NumericalError("gmres: breakdown (NaN/Inf in Arnoldi)");
        for (int i = 0; i <= j; ++i) {
          const double2 a = h_pin[i], c = h_pin[vcap + 2 + i];
          Hij(i, j) = cd(a.x + c.x, a.y + c.y);
        }
        Hij(j + 1, j) = hnext;
        for (int i = 0; i < j; ++i) {
          const cd t1 = Hij(i, j), t2 = Hij(i + 1, j);
          Hij(i, j) = gc[i] * t1 + gs[i] * t2;
          Hij(i + 1, j) = -std::conj(gs[i]) * t1 + gc[i] * t2;
        }
        {  // make_givens (krylov.hpp:66-83)
          const cd h1v = Hij(j, j), h2v = Hij(j + 1, j);
          const double a1 = std::abs(h1v), a2 = std::abs(h2v);
          if (a2 == 0.0) {
            gc[j] = 1.0, gs[j] = 0.0;
          } else if (a1 == 0.0) {
            gc[j] = 0.0, gs[j] = 1.0;
          } else {
            const double t = std::hypot(a1, a2);
            gc[j] = a1 / t;
            gs[j] = (h1v / a1) * (std::conj(h2v) / t);
          }
        }
        Hij(j, j) = gc[j] * Hij(j, j) + gs[j] * Hij(j + 1, j);
        Hij(j + 1, j) = 0.0;
        g[j + 1] = -std::conj(gs[j]) * g[j];
        g[j] = gc[j] * g[j];
        ++st.iterations;
        k = j + 1;
        const double est = std::abs(g[j + 1]);
        const bool happy = hnext <= 1e-14 * std::max(wpre, 1e-300);
        if (happy || est <= tol * bnorm) break;
        launch(FETIGPU_K_ORTHO, [&] {
          k3::k3_scale_to<<<nb, 256, 0, stream>>>(nl, make_double2(1.0 / hnext, 0.0), d_w, d_V + (size_t)(j + 1) * ldv);
        });
      }
      // y = R^-1 g, t = V y, x += M t, r = b - A x
      std::vector<cd> y(k);
      for (int i = k - 1; i >= 0; --i) {
        cd acc = g[i];
        for (int j2 = i + 1; j2 < k; ++j2) acc -= Hij(i, j2) * y[j2];
        y[i] = acc / Hij(i, i);
      }
      for (int i = 0; i < k; ++i) h_pin[i] = dd2(y[i]);
      CU3(cudaMemcpyAsync(d_coef, h_pin, sizeof(double2) * std::max(k, 1), cudaMemcpyHostToDevice, stream));
      // x += P^-1 (V y) = Z y (the preconditioned basis of the cycle; linear, so equal up to
      // rounding, and one Dirichlet application cheaper), true residual r = b - F x
      launch(FETIGPU_K_ORTHO, [&] { k3::k3_mcombine<<<nb, 256, 0, stream>>>(nl, k, d_Z, ldv, d_coef, x); });
      apply_dual(x, d_w);
      st.dual_of_x = true;
      launch(FETIGPU_K_ORTHO, [&] { k3::k3_sub<<<nb, 256, 0, stream>>>(nl, b, d_w, d_r); });
    }
    // final true residual (krylov.hpp:205-215): r already holds b - A x
    st.relres = norm_max(d_r, nl).first / bnorm;
    if (st.relres > best) {
      CU3(cudaMemcpyAsync(x, d_best, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, stream));
      st.relres = best;
      st.dual_of_x = false;
    }
    st.converged = st.relres <= tol;
    return st;
  }

  // ------------------------------------------------------------------------- FETI solve
  // FetiSolver::solve (feti.cpp:630-717) on the factor K + cV; rhs, x: device, n complex
  void feti_solve(const double2* rhs, double2* x, fetigpu_feti_stats* out) {
    const double t0 = now();
    fetigpu_feti_stats st{};
    st.n_lambda = nl;
    st.coarse_dim = nc;
    st.setup_seconds = setup_seconds;
    const double rn = norm_max(rhs, n).first;
    if (rn == 0.0) {
      zero(x, n);
      sync();
      st.converged = 1;
      st.solve_seconds = now() - t0;
      if (out) *out = st;
      return;
    }
    // split_rhs (feti.cpp:493-510)
    launch(FETIGPU_K_OTHER, [&] {
      k3::k3_split<<<cdiv3((long long)S * (NI + NB), 256), 256, 0, stream>>>(S, NI, NB, d_idof, d_bdof, d_bw, rhs,
                                                                            d_fi, d_fb);
    });
    if (nc > 0)
      launch(FETIGPU_K_OTHER, [&] { k3::k3_gather_corner<<<cdiv3(nc, 128), 128, 0, stream>>>(nc, d_cdof, rhs, d_fc); });
    CU3(cudaMemcpyAsync(d_yi, d_fi, sizeof(double2) * S * NI, cudaMemcpyDeviceToDevice, stream));
    interior_solve(d_yi);
    eliminate_boundary(d_fb, true);
    launch(FETIGPU_K_LAMBDA, [&] {  // d = B u_r
      k3::k3_lam_jump<<<cdiv3(nl, 256), 256, 0, stream>>>(nl, NB, NC, 1.0, d_lam_lo, d_lam_hi, d_u1, d_cpl_b, d_cglob,
                                                         nullptr, d_d);
    });
    allreduce(d_d, nl);
    const Stats gs = gmres(d_d, d_lam, desc.max_iter, desc.tol);
    st.iterations = gs.iterations;
    st.converged = gs.converged ? 1 : 0;
    st.relative_residual = gs.relres;
    // t = f_r - B^T lam, final eliminate, interior recovery, primal assembly.  S^-1 and the
    // coarse terms are linear in t: when GMRES's last dual application was on the returned
    // lam, S^-1 (t_b - A_bi y_i) = u0 + S^-1(-B^T lam) and coupling^T t = gcp0 + its part, so
    // the elimination needs no further GEMV
    if (gs.dual_of_x) {
      launch(FETIGPU_K_OTHER, [&] {
        k3::k3_axpby<<<cdiv3((long long)S * NB, 256), 256, 0, stream>>>(S * NB, make_double2(1.0, 0.0), d_u0,
                                                                       make_double2(1.0, 0.0), d_u1);
      });
      if (nc > 0) {
        launch(FETIGPU_K_OTHER, [&] {
          k3::k3_axpby<<<cdiv3((long long)S * G * NC, 256), 256, 0, stream>>>(S * G * NC, make_double2(1.0, 0.0), d_gcp0,
                                                                             make_double2(1.0, 0.0), d_gcp);
        });
        coarse_solve(d_fc);
        launch(FETIGPU_K_OTHER, [&] {
          k3::k3_ub_correct<<<cdiv3((long long)S * NB, 256), 256, 0, stream>>>(S, NB, NC, d_cglob, d_z, d_cpl_b, d_u1);
        });
      }
    } else {
      launch(FETIGPU_K_LAMBDA, [&] {
        k3::k3_gather_in<<<cdiv3((long long)S * NB, 256), 256, 0, stream>>>(S, NB, MR, 2, d_n_b, d_brow, d_bsgn,
                                                                           d_lam_w, d_lam, d_fb, d_tb);
      });
      eliminate_boundary(d_tb);
    }
    launch(FETIGPU_K_OTHER, [&] {
      k3::k3_ri_rhs<<<cdiv3((long long)S * NI, 256), 256, 0, stream>>>(S, NI, NB, NC, H.MAXE_IB, d_ib_idx, d_ib_val,
                                                                      d_aic, d_cglob, d_z, d_u1, d_fi, d_ri);
    });
    interior_solve(d_ri);
    launch(FETIGPU_K_OTHER, [&] {
      k3::k3_assemble_x<<<cdiv3(n, 256), 256, 0, stream>>>(n, d_xkind, d_xref, d_xw, d_ri, d_u1, d_z, x);
    });
    allreduce(x, n);
    // interface jump max |B u_r| and primal residual |A x - rhs| / |rhs|
    launch(FETIGPU_K_LAMBDA, [&] {
      k3::k3_lam_jump<<<cdiv3(nl, 256), 256, 0, stream>>>(nl, NB, NC, 1.0, d_lam_lo, d_lam_hi, d_u1, d_cpl_b, d_cglob,
                                                         nullptr, d_w);
    });
    allreduce(d_w, nl);
    st.interface_jump = nl > 0 ? norm_max(d_w, nl).second : 0.0;
    apply_global<double2>(x, nullptr, cd(1.0), mc, d_ax);
    launch(FETIGPU_K_GLOBAL, [&] { k3::k3_sub<<<cdiv3(n, 256), 256, 0, stream>>>(n, d_ax, rhs, d_ax); });
    st.primal_residual = norm_max(d_ax, n).first / rn;
    prof_collect();
    st.solve_seconds = now() - t0;
    if (out) *out = st;
  }

  // range-space Schur solve (control.cpp:297-334), device buffers
  void schur_solve(const double* ybar, const double* yc, double* y, double* u, double* lam,
                   fetigpu_schur_stats* out) {
    if (!(phi > 0.0)) throw ContractError("schur_solve needs phi > 0 (context built for a plain feti_solve)");
    const double t0 = now();
    fetigpu_schur_stats st{};
    // rhs = K ybar + K_c y_c (control.cpp:15)
    apply_global<double>(ybar, (yc && m > 0) ? yc : nullptr, cd(1.0), cd(0.0), d_real0);
    launch(FETIGPU_K_GLOBAL, [&] { k3::k3_real_to_complex<<<cdiv3(n, 256), 256, 0, stream>>>(n, d_real0, d_rhs); });
    feti_solve(d_rhs, d_x, &st.plus);  // a = (K + cV)^-1 rhs
    apply_global<double2>(d_x, nullptr, cd(0.0), cd(1.0), d_x2);  // V a
    launch(FETIGPU_K_GLOBAL, [&] { k3::k3_conj<<<cdiv3(n, 256), 256, 0, stream>>>(n, d_x2, d_x2); });
    feti_solve(d_x2, d_x, &st.minus);  // conj(t) = (K + cV)^-1 conj(V a)
    launch(FETIGPU_K_GLOBAL, [&] { k3::k3_realify<<<cdiv3(n, 256), 256, 0, stream>>>(n, d_x, lam); });
    launch(FETIGPU_K_GLOBAL, [&] { k3::k3_imag<<<cdiv3(n, 256), 256, 0, stream>>>(n, d_x, d_x2); });
    st.imag_leak = norm_max(d_x2, n).second;
    apply_global<double>(lam, nullptr, cd(1.0), cd(0.0), d_real1);  // K lambda
    mass_solve(d_real1);
    launch(FETIGPU_K_GLOBAL, [&] { k3::k3_recover<<<cdiv3(n, 256), 256, 0, stream>>>(n, ybar, d_real1, lam, phi, y, u); });
    sync();
    st.imag_leak_warning = st.imag_leak > 1e-6 ? 1 : 0;
    st.converged = st.plus.converged && st.minus.converged;
    st.factor_setup_seconds = setup_seconds;
    st.solve_seconds = now() - t0;
    if (out) *out = st;
  }
};

namespace {

void validate3(const fetigpu3d_desc* d) {
  if (!d) throw ContractError("fetigpu3d: null descriptor");
  if (!(d->tol > 0.0)) throw ContractError("fetigpu: tol must be positive");
  if (d->max_iter < 0) throw ContractError("fetigpu: max_iter must be non-negative");
  if (d->phi < 0.0) throw ContractError("ControlProblem: phi must be positive");
}

int guard3(const std::function<void()>& f) {
  try {
    f();
    return FETIGPU_OK;
  } catch (const ContractError& e) {
    set_last_error(e.what());
    return FETIGPU_CONTRACT;
  } catch (const NumericalError& e) {
    set_last_error(e.what());
    return FETIGPU_NUMERICAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FETIGPU_RUNTIME;
  }
}

}  // namespace
}  // namespace fetigpu

using namespace fetigpu;

struct fetigpu3d_ctx {
  Ctx3 c;
};

static void init_ctx3(Ctx3& c, const fetigpu3d_desc* desc) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw RuntimeError("fetigpu3d: no CUDA device");
  c.desc = *desc;
  c.P = build_problem3d(*desc);
  if (desc->phi > 0.0) {
    c.phi = desc->phi;
    c.mc = std::complex<double>(0.0, -1.0 / std::sqrt(desc->phi));  // control.cpp:113-120
  } else {
    c.mc = std::complex<double>(desc->mass_coeff_re, desc->mass_coeff_im);
  }
}

extern "C" {

int fetigpu3d_problem_info(const fetigpu3d_desc* desc, long long* info) {
  return guard3([&] {
    validate3(desc);
    Host3Problem P = build_problem3d(*desc);
    for (int q = 0; q < 16; ++q) info[q] = 0;
    info[0] = P.n();
    info[1] = P.m();
    info[10] = P.dpn;
    if (desc->s_x > 0) {
      Host3Partition H = build_partition3d(P, desc->s_x, desc->s_y, desc->s_z);
      info[2] = H.S, info[3] = H.n_corner, info[4] = H.n_lambda, info[5] = H.NI, info[6] = H.NB, info[7] = H.NC;
      info[8] = H.MR, info[9] = H.P, info[11] = H.ex, info[12] = H.ey, info[13] = H.ez;
      info[14] = H.MAXE_BI, info[15] = H.MAXE_IB;
    }
  });
}

int fetigpu3d_target_sine(const fetigpu3d_desc* desc, unsigned long long seed, int modes, int mmax, double* ybar) {
  return guard3([&] {
    validate3(desc);
    Host3Problem P = build_problem3d(*desc);
    target_sine3d(P, seed, modes, mmax, ybar);
  });
}

int fetigpu3d_create(const fetigpu3d_desc* desc, fetigpu3d_ctx** out) {
  return guard3([&] {
    validate3(desc);
    *out = nullptr;
    auto ctx = std::make_unique<fetigpu3d_ctx>();
    Ctx3& c = ctx->c;
    init_ctx3(c, desc);
    c.H = build_partition3d(c.P, desc->s_x, desc->s_y, desc->s_z);
    c.setup();
    *out = ctx.release();
  });
}

void fetigpu3d_destroy(fetigpu3d_ctx* ctx) { delete ctx; }

// sharded context: this process is rank `rank` of `world` (one GPU each, NCCL); subdomain
// subdomain ids [rank S/world, (rank+1) S/world); schur/feti solves take and return FULL vectors
int fetigpu3d_create_sharded(const fetigpu3d_desc* desc, int rank, int world, const unsigned char* nccl_id,
                             fetigpu3d_ctx** out) {
  return guard3([&] {
    validate3(desc);
    if (!nccl_id) throw ContractError("fetigpu3d_create_sharded: nccl_id required");
    auto ctx = std::make_unique<fetigpu3d_ctx>();
    Ctx3& c = ctx->c;
    init_ctx3(c, desc);
    c.H = local_partition3d(build_partition3d(c.P, desc->s_x, desc->s_y, desc->s_z), rank, world);
    c.comm = make_nccl_comm(nccl_id, rank, world, desc->device);
    c.setup();
    *out = ctx.release();
  });
}

// `world` ranks emulated by host threads on ONE device (ThreadComm, device-to-device
// copies for the allreduces); one range-space Schur solve, rank 0's result.  Tests the
// sharded logic on a single GPU.
int fetigpu3d_emulated_schur_solve(const fetigpu3d_desc* desc, int world, const double* ybar, const double* yc,
                                   double* y, double* u, double* lambda, fetigpu_schur_stats* stats) {
  return guard3([&] {
    validate3(desc);
    if (world < 1) throw ContractError("fetigpu3d_emulated_schur_solve: world must be >= 1");
    const Host3Problem P0 = build_problem3d(*desc);
    const Host3Partition G = build_partition3d(P0, desc->s_x, desc->s_y, desc->s_z);
    auto group = std::make_shared<ThreadGroup>(world);
    std::vector<std::string> errs(world);
    std::vector<std::thread> th;
    for (int q = 0; q < world; ++q)
      th.emplace_back([&, q] {
        try {
          auto ctx = std::make_unique<fetigpu3d_ctx>();
          Ctx3& c = ctx->c;
          init_ctx3(c, desc);
          c.H = local_partition3d(G, q, world);
          c.comm = std::make_unique<ThreadComm>(group, q);
          c.setup();
          if (!(c.phi > 0.0)) throw ContractError("build_complex_factors: phi must be positive");
          const size_t nb = sizeof(double) * c.n;
          CU3(cudaMemcpyAsync(c.d_in_ybar, ybar, nb, cudaMemcpyHostToDevice, c.stream));
          const double* dyc = nullptr;
          if (yc && c.m > 0) {
            CU3(cudaMemcpyAsync(c.d_in_yc, yc, sizeof(double) * c.m, cudaMemcpyHostToDevice, c.stream));
            dyc = c.d_in_yc;
          }
          fetigpu_schur_stats st{};
          c.schur_solve(c.d_in_ybar, dyc, c.d_out_y, c.d_out_u, c.d_out_l, &st);
          if (q == 0) {
            CU3(cudaMemcpyAsync(y, c.d_out_y, nb, cudaMemcpyDeviceToHost, c.stream));
            CU3(cudaMemcpyAsync(u, c.d_out_u, nb, cudaMemcpyDeviceToHost, c.stream));
            CU3(cudaMemcpyAsync(lambda, c.d_out_l, nb, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            if (stats) *stats = st;
          }
          group->barrier();  // keep every rank's buffers alive until rank 0 has copied
        } catch (const std::exception& e) {
          errs[q] = e.what();
          group->abort();
        }
      });
    for (auto& t : th) t.join();
    for (int q = 0; q < world; ++q)
      if (!errs[q].empty() && errs[q] != "rank group aborted")
        throw RuntimeError("rank " + std::to_string(q) + ": " + errs[q]);
  });
}

// host-only layout of rank `rank`: info[0..5] = first subdomain, local subdomains, local
// multiplier-row owners (slots), rows with both owners local, local corner slots, n_lambda
int fetigpu3d_rank_info(const fetigpu3d_desc* desc, int rank, int world, long long* info6) {
  return guard3([&] {
    validate3(desc);
    const Host3Problem P0 = build_problem3d(*desc);
    const Host3Partition L = local_partition3d(build_partition3d(P0, desc->s_x, desc->s_y, desc->s_z), rank, world);
    long long owners = 0, both = 0, cs = 0;
    for (int r = 0; r < L.n_lambda; ++r) {
      owners += (L.lam_lo[r] >= 0) + (L.lam_hi[r] >= 0);
      both += (L.lam_lo[r] >= 0 && L.lam_hi[r] >= 0);
    }
    for (int v : L.corner_slots) cs += v >= 0;
    const long long v[6] = {L.s_first, L.S, owners, both, cs, L.n_lambda};
    std::copy(v, v + 6, info6);
  });
}

int fetigpu3d_schur_solve_device(fetigpu3d_ctx* ctx, const double* d_ybar, const double* d_yc, double* d_y, double* d_u,
                                 double* d_lambda, fetigpu_schur_stats* stats) {
  return guard3([&] { ctx->c.schur_solve(d_ybar, d_yc, d_y, d_u, d_lambda, stats); });
}

int fetigpu3d_schur_solve(fetigpu3d_ctx* ctx, const double* ybar, const double* yc, double* y, double* u,
                          double* lambda, fetigpu_schur_stats* stats) {
  return guard3([&] {
    Ctx3& c = ctx->c;
    const size_t nb = sizeof(double) * c.n;
    CU3(cudaMemcpyAsync(c.d_in_ybar, ybar, nb, cudaMemcpyHostToDevice, c.stream));
    if (yc && c.m > 0) CU3(cudaMemcpyAsync(c.d_in_yc, yc, sizeof(double) * c.m, cudaMemcpyHostToDevice, c.stream));
    c.schur_solve(c.d_in_ybar, (yc && c.m > 0) ? c.d_in_yc : nullptr, c.d_out_y, c.d_out_u, c.d_out_l, stats);
    CU3(cudaMemcpyAsync(y, c.d_out_y, nb, cudaMemcpyDeviceToHost, c.stream));
    CU3(cudaMemcpyAsync(u, c.d_out_u, nb, cudaMemcpyDeviceToHost, c.stream));
    CU3(cudaMemcpyAsync(lambda, c.d_out_l, nb, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  });
}

int fetigpu3d_feti_solve(fetigpu3d_ctx* ctx, int sign, const double* rhs, double* x, fetigpu_feti_stats* stats) {
  return guard3([&] {
    Ctx3& c = ctx->c;
    if (sign != 1 && sign != -1) throw ContractError("feti_solve: sign must be +1 or -1");
    const size_t nb = sizeof(double2) * c.n;
    CU3(cudaMemcpyAsync(c.d_rhs, rhs, nb, cudaMemcpyHostToDevice, c.stream));
    if (sign < 0) k3::k3_conj<<<cdiv3(c.n, 256), 256, 0, c.stream>>>(c.n, c.d_rhs, c.d_rhs);
    c.feti_solve(c.d_rhs, c.d_x, stats);
    if (sign < 0) k3::k3_conj<<<cdiv3(c.n, 256), 256, 0, c.stream>>>(c.n, c.d_x, c.d_x);
    CU3(cudaMemcpyAsync(x, c.d_x, nb, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  });
}

static int lam_op3(fetigpu3d_ctx* ctx, int sign, const double* in, double* out, bool dual) {
  return guard3([&] {
    Ctx3& c = ctx->c;
    if (sign != 1 && sign != -1) throw ContractError("sign must be +1 or -1");
    const size_t nb = sizeof(double2) * c.nl;
    CU3(cudaMemcpyAsync(c.d_r, in, nb, cudaMemcpyHostToDevice, c.stream));
    if (sign < 0) k3::k3_conj<<<cdiv3(c.nl, 256), 256, 0, c.stream>>>(c.nl, c.d_r, c.d_r);
    if (dual) c.apply_dual(c.d_r, c.d_w);
    else c.apply_precond(c.d_r, c.d_w);
    if (sign < 0) k3::k3_conj<<<cdiv3(c.nl, 256), 256, 0, c.stream>>>(c.nl, c.d_w, c.d_w);
    CU3(cudaMemcpyAsync(out, c.d_w, nb, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  });
}
int fetigpu3d_apply_dual(fetigpu3d_ctx* ctx, int sign, const double* lam, double* out) {
  return lam_op3(ctx, sign, lam, out, true);
}
int fetigpu3d_apply_precond(fetigpu3d_ctx* ctx, int sign, const double* r, double* out) {
  return lam_op3(ctx, sign, r, out, false);
}

void* fetigpu3d_stream(fetigpu3d_ctx* ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }

long long fetigpu3d_launch_count(fetigpu3d_ctx* ctx, int reset) {
  const long long v = ctx->c.launches;
  if (reset) ctx->c.launches = 0;
  return v;
}

int fetigpu3d_profile(fetigpu3d_ctx* ctx, int enable) {
  return guard3([&] {
    ctx->c.prof_collect();
    ctx->c.prof = enable != 0;
  });
}

int fetigpu3d_profile_read(fetigpu3d_ctx* ctx, double* ms, long long* cnt, int reset) {
  return guard3([&] {
    Ctx3& c = ctx->c;
    c.prof_collect();
    for (int k = 0; k < FETIGPU_K_COUNT; ++k) {
      ms[k] = c.prof_ms[k];
      cnt[k] = c.prof_n[k];
      if (reset) c.prof_ms[k] = 0, c.prof_n[k] = 0;
    }
  });
}

// algorithmic bytes per launch of the two GEMV classes (k3_sym_rows): the packed operator
// (read once), the input vector (once per subdomain), the row sums and the column partials
// (written once); DESIGN.md §9
double fetigpu3d_class_bytes(fetigpu3d_ctx* ctx, int klass) {
  Ctx3& c = ctx->c;
  if (klass == FETIGPU_K_BAND && c.use_fdm)  // separable solve: the vector in and out
    return 2.0 * 16.0 * (double)c.S * c.fdm_m[0] * c.fdm_m[1] * c.fdm_m[2];
  if (klass == FETIGPU_K_BAND)  // one interior solve: all blocks forward, off-diagonal ones backward
    return 16.0 * 1024.0 * (double)c.S * c.NBK * (2.0 * c.PB + 1.0) + 3.0 * 16.0 * (double)c.S * c.NI;
  if (klass != FETIGPU_K_PRECOND_GEMV && klass != FETIGPU_K_DUAL_GEMV) return 0.0;
  const double vec = 16.0 * (double)c.S * c.NB;
  return 16.0 * (double)c.pack_entries + 512.0 * (double)(c.colpart_rows + c.nitems) + vec;
}

int fetigpu3d_setup_times(fetigpu3d_ctx* ctx, double* out8) {
  for (int q = 0; q < 8; ++q) out8[q] = ctx->c.setup_t[q];
  return 0;
}

}  // extern "C"
