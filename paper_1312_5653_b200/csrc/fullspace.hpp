// fullspace.hpp — the full-space KKT method with the Murphy–Golub–Wathen block
// preconditioner, built on the B200 FETI-DP machinery.
//
// Restates (not copies) control.cpp:17-22 (kkt_rhs), 48-60 (KKT apply),
// 336-345 (solve_sp), 347-416 (PmgwPreconditioner), 418-476 (solve_full_space) and the
// outer Krylov methods of krylov.hpp:102-223 (GMRES, flexible when preconditioned) and
// 256-343 (preconditioned MINRES, Paige–Saunders, true-residual stopping).
//
//   KKT  [V 0 K; 0 phi V -V; K -V 0] [y; u; lambda] = [V ybar; 0; -K_c y_c]
//   P_mgw = blockdiag(V, phi V, S~):
//     "sc": S~^-1 = (K - cV)^-1 V (K + cV)^-1  (exact Schur inverse through the context's
//           complex FETI factor, the range-space solve without its recovery), outer GMRES
//     "sp": S~^-1 = (K + V/sqrt(phi))^-1 V (K + V/sqrt(phi))^-1 (Pearson–Wathen), through a
//           second, real-coefficient FETI context; outer MINRES or GMRES
// The outer Krylov loops are host-driven over device vectors (a handful of iterations with
// the exact-Schur preconditioner; each inner application is two FETI solves).
#pragma once

#include <memory>
#include <vector>

namespace fetigpu {

enum : int { FS_NONE = 0, FS_SP = 1, FS_SC = 2 };
enum : int { FS_MINRES = 0, FS_GMRES = 1 };

struct FullSpace {
  Ctx& c;
  std::unique_ptr<Ctx> spc;  // K + V/sqrt(phi) FETI context ("sp")
  int precond = FS_NONE;
  int n = 0;
  long long N = 0;
  double* part = nullptr;
  double* red = nullptr;
  std::vector<double*> pool;  // 3n work vectors
  int pool_used = 0;
  double last_leak = 0.0;
  long long inner_iters = 0;

  FullSpace(Ctx& ctx, int pc) : c(ctx), precond(pc), n(ctx.n), N(3LL * ctx.n) {
    part = c.alloc<double>(296);
    red = c.alloc<double>(2);
  }
  double* vec() {
    if (pool_used == (int)pool.size()) pool.push_back(c.alloc<double>((size_t)N));
    return pool[pool_used++];
  }
  int grid(long long m) const { return (int)std::min<long long>((m + 255) / 256, 1LL << 30); }

  double dot(const double* x, const double* y, long long m) {
    const int nb = (int)std::max<long long>(1, std::min<long long>(296, (m + 255) / 256));
    k_rdot_part<<<nb, 256, 0, c.stream>>>(m, x, y, part);
    k_rdot_final<<<1, 32, 0, c.stream>>>(nb, part, red);
    CU(cudaGetLastError());
    c.launches += 2;
    double h = 0;
    CU(cudaMemcpyAsync(&h, red, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return h;
  }
  double norm(const double* x) { return std::sqrt(std::max(0.0, dot(x, x, N))); }
  void axpby(double a, const double* x, double b, double* y, long long m) {
    k_axpby<<<grid(m), 256, 0, c.stream>>>(m, a, x, b, y);
    CU(cudaGetLastError());
    ++c.launches;
  }
  void copy(const double* x, double* y, long long m) {
    CU(cudaMemcpyAsync(y, x, sizeof(double) * m, cudaMemcpyDeviceToDevice, c.stream));
  }

  // KKT apply (control.cpp:48-60): y1 = V xy + K xl; y2 = phi V xu - V xl; y3 = K xy - V xu
  void kkt(const double* x, double* y) {
    const double *xy = x, *xu = x + n, *xl = x + 2LL * n;
    double *y1 = y, *y2 = y + n, *y3 = y + 2LL * n;
    double* t = c.d_real0;
    c.apply_global<double>(xy, nullptr, 0.0, 1.0, y1);
    c.apply_global<double>(xl, nullptr, 1.0, 0.0, t);
    axpby(1.0, t, 1.0, y1, n);
    c.apply_global<double>(xu, nullptr, 0.0, c.phi, y2);
    c.apply_global<double>(xl, nullptr, 0.0, 1.0, t);
    axpby(-1.0, t, 1.0, y2, n);
    c.apply_global<double>(xy, nullptr, 1.0, 0.0, y3);
    c.apply_global<double>(xu, nullptr, 0.0, 1.0, t);
    axpby(-1.0, t, 1.0, y3, n);
  }

  // z3 = S~^-1 r3 for the two Schur approximations
  void schur_inverse(const double* r3, double* z3) {
    const int g = (n + 255) / 256;
    if (precond == FS_SC) {  // (K - cV)^-1 V (K + cV)^-1 r3 = conj(F(conj(V F r3)))
      k_real_to_complex<<<g, 256, 0, c.stream>>>(n, r3, c.d_rhs);
      const auto s1 = c.feti_solve(c.d_rhs, c.d_x, 10);
      k_conj<<<g, 256, 0, c.stream>>>(n, c.d_x, c.d_x2);
      c.apply_global<double2>(c.d_x2, nullptr, 0.0, 1.0, c.d_rhs);
      const auto s2 = c.feti_solve(c.d_rhs, c.d_x, 10);
      k_realify<<<g, 256, 0, c.stream>>>(n, c.d_x, z3);  // Re conj(t') = Re t'
      const int nb = std::max(1, std::min(296, g));
      k_imag_max_part<<<nb, 256, 0, c.stream>>>(n, c.d_x, part);
      k_max_final<<<1, 32, 0, c.stream>>>(nb, part, c.d_stat + 15);
      CU(cudaGetLastError());
      c.launches += 5;
      inner_iters += s1.iterations + s2.iterations;
    } else {  // solve_sp (control.cpp:336-345) on the real-coefficient context
      c.sync();
      Ctx& s = *spc;
      k_real_to_complex<<<g, 256, 0, s.stream>>>(n, r3, s.d_rhs);
      const auto s1 = s.feti_solve(s.d_rhs, s.d_x, 10);
      s.apply_global<double2>(s.d_x, nullptr, 0.0, 1.0, s.d_rhs);
      const auto s2 = s.feti_solve(s.d_rhs, s.d_x, 10);
      k_realify<<<g, 256, 0, s.stream>>>(n, s.d_x, z3);
      CU(cudaGetLastError());
      s.launches += 3;
      s.sync();
      inner_iters += s1.iterations + s2.iterations;
    }
  }

  // P_mgw^-1 r (control.cpp:362-405)
  void pmgw(const double* r, double* z) {
    copy(r, z, n);
    c.mass_solve(z);
    copy(r + n, z + n, n);
    c.mass_solve(z + n);
    axpby(0.0, z + n, 1.0 / c.phi, z + n, n);
    schur_inverse(r + 2LL * n, z + 2LL * n);
  }
  void precondition(const double* r, double* z) {
    if (precond == FS_NONE)
      copy(r, z, N);
    else
      pmgw(r, z);
  }

  // krylov.hpp:102-223 over real 3n-vectors (Hermitian MGS, Givens, restarts, best iterate)
  fetigpu_feti_stats gmres(const double* b, double* x, double tol, int max_iter) {
    fetigpu_feti_stats st{};
    CU(cudaMemsetAsync(x, 0, sizeof(double) * N, c.stream));
    const double bnorm = norm(b);
    if (bnorm == 0.0) {
      st.converged = 1;
      return st;
    }
    double* r = vec();
    double* w = vec();
    double* best = vec();
    copy(b, r, N);  // x0 = 0
    copy(x, best, N);
    double best_res = 1.0;
    const bool pre = precond != FS_NONE;
    const int m = std::max(1, max_iter);
    std::vector<double*> V, Z;
    std::vector<double> giv_c(m + 1), giv_s(m + 1), g(m + 2);
    std::vector<std::vector<double>> H;  // column-major Hessenberg columns
    int iters = 0;
    double relres = 1.0;
    while (true) {
      const double rnorm = norm(r);
      relres = rnorm / bnorm;
      if (relres < best_res) {
        best_res = relres;
        copy(x, best, N);
      }
      if (relres <= tol) break;
      if (iters >= max_iter) break;
      if (V.empty()) V.push_back(vec());
      axpby(1.0 / rnorm, r, 0.0, V[0], N);
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = rnorm;
      H.clear();
      int k = 0;
      for (int j = 0; j < m && iters < max_iter; ++j) {
        double* zj;
        if (pre) {
          if ((int)Z.size() <= j) Z.push_back(vec());
          zj = Z[j];
          precondition(V[j], zj);
        } else {
          zj = V[j];
        }
        kkt(zj, w);
        const double wpre = norm(w);
        std::vector<double> h(j + 2, 0.0);
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
          h[i] = dot(V[i], w, N);
          axpby(-h[i], V[i], 1.0, w, N);
        }
        const double hnext = norm(w);
        if (!std::isfinite(hnext)) throw NumericalError("gmres: breakdown (NaN/Inf in Arnoldi)");
        h[j + 1] = hnext;
        for (int i = 0; i < j; ++i) {
          const double t1 = h[i], t2 = h[i + 1];
          h[i] = giv_c[i] * t1 + giv_s[i] * t2;
          h[i + 1] = -giv_s[i] * t1 + giv_c[i] * t2;
        }
        const double a1 = std::abs(h[j]), a2 = hnext;
        if (a2 == 0.0) {
          giv_c[j] = 1.0;
          giv_s[j] = 0.0;
        } else if (a1 == 0.0) {
          giv_c[j] = 0.0;
          giv_s[j] = 1.0;
        } else {
          const double t = std::hypot(a1, a2);
          giv_c[j] = a1 / t;
          giv_s[j] = (h[j] / a1) * a2 / t;
        }
        h[j] = giv_c[j] * h[j] + giv_s[j] * hnext;
        h[j + 1] = 0.0;
        g[j + 1] = -giv_s[j] * g[j];
        g[j] = giv_c[j] * g[j];
        H.push_back(h);
        ++iters;
        k = j + 1;
        const bool happy = hnext <= 1e-14 * std::max(wpre, 1e-300);
        if (happy || std::abs(g[j + 1]) <= tol * bnorm) break;
        if ((int)V.size() <= j + 1) V.push_back(vec());
        axpby(1.0 / hnext, w, 0.0, V[j + 1], N);
      }
      std::vector<double> y(k);
      for (int i = k - 1; i >= 0; --i) {
        double acc = g[i];
        for (int j2 = i + 1; j2 < k; ++j2) acc -= H[j2][i] * y[j2];
        y[i] = acc / H[i][i];
      }
      if (pre) {  // flexible: x += Z y
        for (int i = 0; i < k; ++i) axpby(y[i], Z[i], 1.0, x, N);
      } else {
        for (int i = 0; i < k; ++i) axpby(y[i], V[i], 1.0, x, N);
      }
      kkt(x, w);
      copy(b, r, N);
      axpby(-1.0, w, 1.0, r, N);
    }
    kkt(x, w);
    copy(b, r, N);
    axpby(-1.0, w, 1.0, r, N);
    relres = norm(r) / bnorm;
    if (relres > best_res) {
      copy(best, x, N);
      relres = best_res;
    }
    st.iterations = iters;
    st.relative_residual = relres;
    st.converged = relres <= tol;
    return st;
  }

  // krylov.hpp:256-343: preconditioned MINRES, convergence on the true residual
  fetigpu_feti_stats minres(const double* b, double* x, double tol, int max_iter) {
    fetigpu_feti_stats st{};
    CU(cudaMemsetAsync(x, 0, sizeof(double) * N, c.stream));
    const double bnorm = norm(b);
    if (bnorm == 0.0) {
      st.converged = 1;
      return st;
    }
    double *r1 = vec(), *r2 = vec(), *y = vec(), *w = vec(), *w1 = vec(), *w2 = vec(), *v = vec(), *tmp = vec(),
           *best = vec();
    copy(b, r1, N);
    copy(b, r2, N);
    precondition(b, y);
    double beta1 = dot(b, y, N);
    if (beta1 < 0.0) throw ContractError("minres: preconditioner is not positive definite");
    if (beta1 == 0.0) {
      st.converged = 1;
      return st;
    }
    beta1 = std::sqrt(beta1);
    double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0;
    CU(cudaMemsetAsync(w, 0, sizeof(double) * N, c.stream));
    CU(cudaMemsetAsync(w2, 0, sizeof(double) * N, c.stream));
    copy(x, best, N);
    double best_res = 1.0;
    int iters = 0;
    for (int itn = 1; itn <= max_iter; ++itn) {
      axpby(1.0 / beta, y, 0.0, v, N);
      kkt(v, y);
      if (itn >= 2) axpby(-beta / oldb, r1, 1.0, y, N);
      const double alfa = dot(v, y, N);
      axpby(-alfa / beta, r2, 1.0, y, N);
      copy(r2, r1, N);
      copy(y, r2, N);
      precondition(r2, y);
      oldb = beta;
      beta = dot(r2, y, N);
      if (beta < 0.0) throw ContractError("minres: preconditioner is not positive definite");
      beta = std::sqrt(beta);
      const bool exhausted = beta < 1e-300;
      const double oldeps = epsln;
      const double delta = cs * dbar + sn * alfa;
      const double gbar = sn * dbar - cs * alfa;
      epsln = sn * beta;
      dbar = -cs * beta;
      const double gamma = std::max(std::hypot(gbar, beta), 1e-300);
      cs = gbar / gamma;
      sn = beta / gamma;
      const double phi_k = cs * phibar;
      phibar = sn * phibar;
      // w1 = w2; w2 = w; w = (v - oldeps w1 - delta w2) / gamma
      std::swap(w1, w2);  // w1 <- old w2
      std::swap(w2, w);   // w2 <- old w, w <- old w1 (overwritten below)
      copy(v, w, N);
      axpby(-oldeps / gamma, w1, 1.0 / gamma, w, N);
      axpby(-delta / gamma, w2, 1.0, w, N);
      axpby(phi_k, w, 1.0, x, N);
      ++iters;
      kkt(x, tmp);
      axpby(1.0, b, -1.0, tmp, N);
      const double true_res = norm(tmp) / bnorm;
      if (true_res < best_res) {
        best_res = true_res;
        copy(x, best, N);
      }
      if (true_res <= tol || exhausted) break;
      if (!std::isfinite(true_res)) throw NumericalError("minres: breakdown (NaN/Inf residual)");
    }
    copy(best, x, N);
    st.iterations = iters;
    st.relative_residual = best_res;
    st.converged = best_res <= tol;
    return st;
  }
};

}  // namespace fetigpu
