"""Experiment drivers / result schema (experiments.cpp)."""
import json

import numpy as np
import pytest


@pytest.fixture(scope="module")
def X(fetigpu):
    from paper_1312_5653_b200 import experiments
    return experiments


def test_default_configs_and_canonical_json(X):
    c = X.ExperimentConfig.defaults_for("phi_sweep")
    assert c.phi[0] == 2e-2 and c.phi[-1] == pytest.approx(2e-12) and len(c.phi) == 11
    j = c.to_json()
    assert j.startswith('{"augment":true,"deterministic":true,"feti_tol":1e-10,"inner_tol":1e-09,')
    assert '"kind":"phi_sweep"' in j and '"pressure":100000.0' in j and '"mesh_sizes":[]' in j
    assert len(c.hash()) == 16 and c.hash() == X.ExperimentConfig.from_json(j).hash()
    s = X.ExperimentConfig.defaults_for("scalability")
    assert s.mesh_sizes == [16, 32, 64] and s.ratio == 8 and s.phi == [2e-8]
    e = X.ExperimentConfig.defaults_for("precond_compare")
    assert (e.physics, e.n, e.s_x, e.s_y) == ("elasticity", 12, 6, 2)


def test_config_validation(X, fetigpu):
    with pytest.raises(fetigpu.ContractError):
        X.ExperimentConfig.from_json(json.dumps({"kind": "phi_sweep", "phi": [1e-4, 1e-2]}))
    with pytest.raises(fetigpu.ContractError):
        X.ExperimentConfig.from_json(json.dumps({"kind": "phi_sweep", "phi": [-1.0]}))
    with pytest.raises(fetigpu.ContractError):
        X.ExperimentConfig.from_json(json.dumps({"kind": "nope"}))
    with pytest.raises(fetigpu.ContractError):
        X.ExperimentConfig.from_json(json.dumps({"kind": "phi_sweep", "physics": "fluid"}))


def test_rows_roundtrip_csv_json(X, tmp_path):
    r = X.ResultRow(experiment="phi_sweep", config_hash="0123456789abcdef", physics="heat", n=16, dofs=225,
                    elements=256, h=1 / 16, H=0.5, s_x=2, s_y=2, nsub=4, phi=1e-4, method="range_space",
                    backend="feti_aug", augment=True, iters_minus=7, iters_plus=7, converged=True,
                    relative_residual=3.2e-11, error="a, b\nc", total_seconds=0.5)
    r.error = "a; b;c"
    assert r.key() == "phi_sweep|heat|16|2x2|0.0001|range_space|feti_aug|1"
    for fmt, parse in (("csv", X.parse_rows_csv), ("json", X.parse_rows_json)):
        path = tmp_path / f"rows.{fmt}"
        X.emit_rows([r, r], fmt, str(path))
        back = parse(path.read_text())
        assert len(back) == 2 and all(b.equal_ignoring_wall_time(r) for b in back)
        assert X.parse_rows_file(str(path))[0].key() == r.key()
    assert X.rows_to_csv([r]).splitlines()[0] == "# pdeopt-results schema=1 config=0123456789abcdef"
    assert X.rows_to_csv([r]).splitlines()[1] == ",".join(X.COLUMNS)
    with pytest.raises(Exception):
        X.emit_rows([], "csv", str(tmp_path / "empty.csv"))


@pytest.mark.gpu
def test_phi_sweep_and_cache(X, tmp_path):
    cfg = X.ExperimentConfig.from_json(json.dumps({"kind": "phi_sweep", "n": 16, "s_x": 2, "s_y": 2,
                                                   "phi": [1e-2, 1e-5]}))
    rows = X.run_experiment(cfg)
    assert [(r.phi, r.backend) for r in rows] == [(1e-2, "feti"), (1e-2, "feti_aug"), (1e-5, "feti"), (1e-5, "feti_aug")]
    for r in rows:
        assert r.converged and not r.error and r.iters_plus > 0 and r.constraint_violation < 1e-6
        assert r.dofs == 15 * 15 and r.nsub == 4 and r.config_hash == cfg.hash()
    assert rows[1].iters_plus <= rows[0].iters_plus  # augmentation helps
    assert rows[2].target_mismatch < rows[0].target_mismatch  # smaller phi tracks the target better
    out = tmp_path / "sweep.csv"
    X.emit_rows(rows, "csv", str(out))
    again = X.run_experiment(cfg, str(out))  # every row comes from the cache
    assert all(a.equal_ignoring_wall_time(b) and a.total_seconds == b.total_seconds for a, b in zip(again, X.parse_rows_csv(out.read_text())))


@pytest.mark.gpu
def test_precond_compare_and_diagnostics(X, fetigpu):
    cfg = X.ExperimentConfig.from_json(json.dumps({"kind": "precond_compare", "physics": "heat", "n": 16, "s_x": 2,
                                                   "s_y": 2, "phi": [1e-4]}))
    rows = X.run_precond_compare(cfg)
    assert [r.backend for r in rows] == ["sp", "sc"]
    assert all(r.converged and r.method == "full_space" for r in rows)
    assert rows[0].cross_agreement == rows[1].cross_agreement < 1e-6
    assert rows[1].outer_iters <= 4


@pytest.mark.gpu
def test_device_diagnostics_match_host(fetigpu, oracle_mod):
    p = fetigpu.make_thermal_problem(16, 1e-4)
    out = fetigpu.solve_range_space(p, tol=1e-12)
    op = oracle_mod.Problem(16)
    K, V, Kc = op.dense(0), op.dense(1), op.dense(2)
    dev = fetigpu.diagnostics(p, out["y"], out["u"], out["lambda"])
    host = fetigpu.diagnostics(p, out["y"], out["u"], out["lambda"], K=K, V=V, Kc=Kc)
    for k in ("constraint_violation", "target_mismatch", "control_norm", "objective"):
        assert abs(dev[k] - host[k]) <= 1e-10 * max(abs(host[k]), 1e-3), k


@pytest.mark.gpu
def test_cantilever_target_is_the_pressure_displacement(fetigpu, oracle_mod):
    p = fetigpu.make_cantilever_problem(4, 1e-4)
    op = oracle_mod.Problem(12, 4, len_x=3.0, len_y=1.0, physics=1, young=20.7e6, poisson=0.45)
    K = op.dense(0)
    f = K @ p.target_state
    nodal = -100e3 * (1.0 / 4) / 2.0
    assert np.isclose(f.min(), 2 * nodal, rtol=1e-6) and np.all(f[::2] <= 1e-6 * abs(nodal))  # downward only
    # total pressure force on the bottom edge minus the clamped corner node's h/2 share
    assert abs(f.sum() - (-100e3 * 3.0 + 100e3 * 0.25 / 2)) <= 1e-6 * 100e3
