"""Generates tests/golden/ref_golden.npz from the REFERENCE ITSELF: the unmodified pdeopt
sources (/root/reference/proj/src) compiled against the Eigen-API shim (oracle/_ref, see
oracle/Makefile `ref` and oracle/ref_driver.cpp), called through the reference's own public
API (solve_range_space with FactorMethod::FetiDp; FetiSolver<Complex>).

Run here (where /root/reference exists):  python tests/golden/make_ref_golden.py
The fixtures travel with the repo; the GPU box never needs the reference.

Cases (BASELINE.json target: seeded sine modes, y_c = 0, augment = false, tol 1e-10):
  cfg1_s{0,1,2}     config 1 (64^2, 4x4 subdomains, phi = 1e-4), y / u / lambda / iterations
  sweep_p{2,4,6,8}  config 2's phi sweep {1e-2,1e-4,1e-6,1e-8} on 128^2 with 4x4 subdomains
                    of 32x32 elements (config 2's subdomain shape): y / lambda / iterations
  thermal32         the reference's own thermal problem (target (2x-1)^2(2y-1)^2 on
                    [0,1/2]^2, y_c = target trace), 32^2, 4x4, phi = 1e-4
  aug_cfg1          config 1 seed 0 with edge-RBM augmentation (the reference default)
  cant8             plane-strain rubber cantilever 24x8 (reference target), 6x2, phi = 1e-4
  ops_cfg1          dual operator / Dirichlet preconditioner of K +- cV on a seeded lambda
  feti16            FetiSolver<Complex> on K + cV, n = 16, 2x2, phi = 2e-8, seeded rhs,
                    augment = true and false (test_feti.cpp:309-332)
  crit6_iters       acceptance criterion 6's sweep (verify.cpp:194-226; experiments.cpp:118-127,
                    244-283): thermal 64^2, 8x8, phi = 2e-2 .. 2e-12, augment false / true:
                    [phi][augment][plus, minus] iterations
  crit7_iters       criterion 7 (verify.cpp:228-246; experiments.cpp:285-322): thermal n = 16,
                    32, 64 at H/h = 8, phi = 2e-8, augment = true: [n][plus, minus]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refbind as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_golden.npz")
TOL, MAX_ITER = 1e-10, 2000


def seeded_target(n, seed):
    import paper_1312_5653_b200 as F  # host-side target generator (no GPU needed)

    return F.make_seeded_problem(n, 1e-4, seed=seed).target_state


def main():
    R.build()
    d = {}
    for seed in (0, 1, 2):
        ybar = seeded_target(64, seed)
        r = R.schur_solve(64, 4, 4, 1e-4, ybar, tol=TOL, max_iter=MAX_ITER)
        for k in ("y", "u", "lambda"):
            d[f"cfg1_s{seed}_{k}"] = r[k]
        d[f"cfg1_s{seed}_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
        d[f"cfg1_s{seed}_ybar"] = ybar
    ybar = seeded_target(128, 0)
    d["sweep_ybar"] = ybar
    for e in (2, 4, 6, 8):
        phi = 10.0 ** (-e)
        r = R.schur_solve(128, 4, 4, phi, ybar, tol=TOL, max_iter=MAX_ITER, threads=8)
        d[f"sweep_p{e}_y"] = r["y"]
        d[f"sweep_p{e}_lambda"] = r["lambda"]
        d[f"sweep_p{e}_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
    ybar, yc = R.problem_data(R.HEAT, 32)
    r = R.schur_solve(32, 4, 4, 1e-4, ybar, yc, tol=TOL, max_iter=MAX_ITER)
    for k in ("y", "u", "lambda"):
        d[f"thermal32_{k}"] = r[k]
    d["thermal32_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
    r = R.schur_solve(64, 4, 4, 1e-4, d["cfg1_s0_ybar"], tol=TOL, max_iter=MAX_ITER, augment=True)
    for k in ("y", "u", "lambda"):
        d[f"aug_cfg1_{k}"] = r[k]
    d["aug_cfg1_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
    ybar, yc = R.problem_data(R.CANTILEVER, 8)
    r = R.schur_solve(8, 6, 2, 1e-4, ybar, yc, tol=TOL, max_iter=MAX_ITER, kind=R.CANTILEVER)
    d["cant8_ybar"] = ybar
    for k in ("y", "u", "lambda"):
        d[f"cant8_{k}"] = r[k]
    d["cant8_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
    c = -1j / np.sqrt(1e-4)
    for sign, coeff in ((1, c), (-1, -c)):
        f = R.Feti(64, 4, 4, coeff)
        rng = np.random.default_rng(7)
        lam = rng.uniform(-1, 1, f.n_lambda) + 1j * rng.uniform(-1, 1, f.n_lambda)
        d[f"ops_cfg1_{'p' if sign > 0 else 'm'}_dual"] = f.apply_dual_operator(lam)
        d[f"ops_cfg1_{'p' if sign > 0 else 'm'}_precond"] = f.apply_dirichlet_preconditioner(lam)
        f.close()
    c = -1j / np.sqrt(2e-8)
    rng = np.random.default_rng(29)
    nf, _ = R.problem_size(R.HEAT, 16)
    rhs = rng.uniform(-1, 1, nf).astype(complex)
    d["feti16_rhs"] = rhs
    for aug in (True, False):
        f = R.Feti(16, 2, 2, c, augment=aug)
        x, st = f.solve(rhs)
        f.close()
        d[f"feti16_aug{int(aug)}_x"] = x
        d[f"feti16_aug{int(aug)}_iters"] = np.array([st["iterations"]])
    ybar, yc = R.problem_data(R.HEAT, 64)
    phis = [2.0 * 10.0 ** -e for e in range(2, 13)]
    d["crit6_phis"] = np.array(phis)
    d["crit6_iters"] = np.array([[[r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]]
                                  for r in (R.schur_solve(64, 8, 8, phi, ybar, yc, tol=TOL, max_iter=MAX_ITER,
                                                          augment=aug) for aug in (False, True))]
                                 for phi in phis])
    crit7 = []
    for n in (16, 32, 64):
        ybar, yc = R.problem_data(R.HEAT, n)
        r = R.schur_solve(n, n // 8, n // 8, 2e-8, ybar, yc, tol=TOL, max_iter=MAX_ITER, augment=True)
        crit7.append([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
    d["crit7_iters"] = np.array(crit7)
    np.savez_compressed(OUT, **d)
    print(f"wrote {OUT}: {len(d)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
