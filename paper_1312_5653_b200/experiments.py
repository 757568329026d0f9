"""Experiment drivers and the result-row schema on the B200 path.

Mirrors include/pdeopt/experiments.hpp + src/experiments.cpp of the reference:

    ExperimentConfig (JSON round trip, FNV-1a 64 hash of the canonical JSON)  :20-44, 158-232
    ResultRow (schema_version 1, stable CSV column order, key())              :46-84, 234-240
    run_phi_sweep / run_scalability / run_precond_compare / run_accuracy_cliff :244-460
    run_experiment (row cache keyed by ResultRow.key() for the same config)    :462-488
    emit_rows / rows_to_csv / rows_to_json / parse_rows_*                      :490-720

Every solve runs on the GPU (range space through ``SchurSolver``, full space through
``solve_full_space``, diagnostics on the device).  Differences, all reported in the rows:
the reference's ``direct`` backend (sparse LU on the CPU) has no counterpart here, so
accuracy_cliff's range-space row carries ``error = "backend 'direct' not provided"``; its
full-space row uses FETI-DP inner solves instead of LU and no refinement sweeps.
"""
from __future__ import annotations

import csv
import io
import json
import os
import time
from dataclasses import dataclass, field, fields

import numpy as np

from . import (ContractError, NumericalError, SchurSolver, diagnostics, make_cantilever_problem,
               make_thermal_problem, solve_full_space)

KINDS = ("phi_sweep", "scalability", "precond_compare", "accuracy_cliff")


def _fnv1a(text: str) -> int:
    h = 1469598103934665603
    for c in text.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _jnum(v):
    """nlohmann::json number formatting: shortest round trip, doubles keep a '.0'."""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    r = repr(float(v))
    if r in ("inf", "-inf", "nan"):
        return "null"
    if "e" not in r and "." not in r:
        r += ".0"
    return r


def _jdump(obj) -> str:
    """Compact JSON with sorted keys (nlohmann's default object ordering)."""
    if isinstance(obj, dict):
        return "{" + ",".join(json.dumps(k) + ":" + _jdump(obj[k]) for k in sorted(obj)) + "}"
    if isinstance(obj, (list, tuple)):
        return "[" + ",".join(_jdump(v) for v in obj) + "]"
    if isinstance(obj, str):
        return json.dumps(obj)
    return _jnum(obj)


@dataclass
class ExperimentConfig:
    kind: str = "phi_sweep"
    physics: str = "heat"  # heat | elasticity
    n: int = 64
    s_x: int = 8
    s_y: int = 8
    phi: list = field(default_factory=list)  # strictly positive, sorted descending
    feti_tol: float = 1e-10
    outer_tol: float = 1e-10
    inner_tol: float = 1e-9
    augment: bool = True
    deterministic: bool = True
    threads: int = 1
    seed: int = 0
    mesh_sizes: list = field(default_factory=list)
    ratio: int = 8
    pressure: float = 100e3

    @staticmethod
    def defaults_for(kind: str) -> "ExperimentConfig":  # experiments.cpp:118-156
        if kind not in KINDS:
            raise ContractError(f"unknown experiment kind '{kind}'")
        c = ExperimentConfig(kind=kind)
        if kind == "phi_sweep":
            c.physics, c.n, c.s_x, c.s_y = "heat", 64, 8, 8
            c.phi = [2.0 * 10.0 ** -e for e in range(2, 13)]
            c.feti_tol = 1e-10
        elif kind == "scalability":
            c.physics, c.mesh_sizes, c.ratio, c.phi, c.feti_tol = "heat", [16, 32, 64], 8, [2e-8], 1e-10
        elif kind == "precond_compare":
            c.physics, c.n, c.s_x, c.s_y = "elasticity", 12, 6, 2
            c.phi = [10.0 ** -e for e in range(7, 15)]
            c.outer_tol, c.inner_tol = 1e-10, 1e-9
        else:
            c.physics, c.n, c.s_x, c.s_y = "elasticity", 24, 6, 2
            c.phi = [10.0 ** -e for e in range(7, 17)]
            c.outer_tol, c.inner_tol = 1e-9, 1e-12
        return c

    def validate(self):  # experiments.cpp:158-167
        for p in self.phi:
            if not p > 0.0:
                raise ContractError("ExperimentConfig: phi values must be positive")
        for a, b in zip(self.phi, self.phi[1:]):
            if not b < a:
                raise ContractError("ExperimentConfig: phi list must be sorted strictly descending")
        if self.n < 2:
            raise ContractError("ExperimentConfig: n must be at least 2")
        if self.threads < 1:
            raise ContractError("ExperimentConfig: threads must be at least 1")

    def to_json(self) -> str:
        d = {f.name: getattr(self, f.name) for f in fields(self)}
        d["phi"] = [float(v) for v in self.phi]
        d["mesh_sizes"] = [int(v) for v in self.mesh_sizes]
        d["feti_tol"], d["outer_tol"] = float(self.feti_tol), float(self.outer_tol)
        d["inner_tol"], d["pressure"] = float(self.inner_tol), float(self.pressure)
        return _jdump(d)

    @staticmethod
    def from_json(text: str) -> "ExperimentConfig":  # experiments.cpp:190-225
        j = json.loads(text)
        c = ExperimentConfig.defaults_for(j["kind"])
        if "physics" in j:
            p = j["physics"]
            if p == "heat":
                c.physics = "heat"
            elif p in ("elasticity", "plane_strain_elasticity"):
                c.physics = "elasticity"
            else:
                raise ContractError(f"ExperimentConfig: unknown physics '{p}'")
        for k in ("n", "s_x", "s_y", "feti_tol", "outer_tol", "inner_tol", "augment", "deterministic", "threads",
                  "seed", "ratio", "pressure"):
            if k in j:
                setattr(c, k, type(getattr(c, k))(j[k]))
        if "phi" in j:
            c.phi = [float(v) for v in j["phi"]]
        if "mesh_sizes" in j:
            c.mesh_sizes = [int(v) for v in j["mesh_sizes"]]
        c.validate()
        return c

    def hash(self) -> str:
        return f"{_fnv1a(self.to_json()):016x}"


COLUMNS = ("schema_version", "experiment", "config_hash", "physics", "n", "dofs", "elements", "h", "H", "s_x", "s_y",
           "nsub", "phi", "method", "backend", "augment", "iters_minus", "iters_plus", "outer_iters", "converged",
           "relative_residual", "constraint_violation", "target_mismatch", "control_norm", "objective", "imag_leak",
           "cross_agreement", "error", "build_seconds", "per_solve_seconds", "total_seconds")
WALL_TIME_COLUMNS = ("build_seconds", "per_solve_seconds", "total_seconds")
_INT = {"schema_version", "n", "dofs", "elements", "s_x", "s_y", "nsub", "iters_minus", "iters_plus", "outer_iters"}
_BOOL = {"augment", "converged"}
_STR = {"experiment", "config_hash", "physics", "method", "backend", "error"}


@dataclass
class ResultRow:
    schema_version: int = 1
    experiment: str = ""
    config_hash: str = ""
    physics: str = ""
    n: int = 0
    dofs: int = 0
    elements: int = 0
    h: float = 0.0
    H: float = 0.0
    s_x: int = 0
    s_y: int = 0
    nsub: int = 0
    phi: float = 0.0
    method: str = ""   # range_space | full_space
    backend: str = ""  # feti | feti_aug | direct | sp | sc
    augment: bool = False
    iters_minus: int = 0
    iters_plus: int = 0
    outer_iters: int = 0
    converged: bool = False
    relative_residual: float = 0.0
    constraint_violation: float = 0.0
    target_mismatch: float = 0.0
    control_norm: float = 0.0
    objective: float = 0.0
    imag_leak: float = 0.0
    cross_agreement: float = 0.0
    error: str = ""
    build_seconds: float = 0.0
    per_solve_seconds: float = 0.0
    total_seconds: float = 0.0

    def key(self) -> str:  # experiments.cpp:234-240
        return (f"{self.experiment}|{self.physics}|{self.n}|{self.s_x}x{self.s_y}|{_fmt17(self.phi)}|{self.method}|"
                f"{self.backend}|{1 if self.augment else 0}")

    def equal_ignoring_wall_time(self, other: "ResultRow") -> bool:
        return all(getattr(self, c) == getattr(other, c) for c in COLUMNS if c not in WALL_TIME_COLUMNS)


def _fmt17(v) -> str:
    return "%.17g" % float(v)


def _sanitize(text: str) -> str:
    return "".join(";" if ch in ",\n\r" else ch for ch in text)


# ------------------------------------------------------------------------ problems and rows
def _build_problem(config: ExperimentConfig, n: int, phi: float):
    if config.physics == "heat":
        return make_thermal_problem(n, phi)
    return make_cantilever_problem(n, phi, config.pressure)


def _base_row(config: ExperimentConfig, p, phi: float) -> ResultRow:  # experiments.cpp:60-76
    r = ResultRow(experiment=config.kind, config_hash=config.hash(), physics=config.physics)
    r.n = p.n_y
    r.dofs = p.n
    r.elements = p.n_x * p.n_y
    r.h = p.len_x / p.n_x
    r.H = p.len_x / config.s_x
    r.s_x, r.s_y, r.nsub, r.phi = config.s_x, config.s_y, config.s_x * config.s_y, phi
    return r


def _fill_diagnostics(row: ResultRow, p, y, u, lam, imag_leak):
    rep = diagnostics(p, y, u, lam)
    row.constraint_violation = rep["constraint_violation"]
    row.target_mismatch = rep["target_mismatch"]
    row.control_norm = rep["control_norm"]
    row.objective = rep["objective"]
    row.imag_leak = imag_leak


def _range_space_row(config, p, phi, augment, tol, cache, rows):
    t0 = time.perf_counter()
    row = _base_row(config, p, phi)
    row.method, row.backend, row.augment = "range_space", "feti_aug" if augment else "feti", augment
    if cache and row.key() in cache:
        rows.append(cache[row.key()])
        return
    try:
        solver = SchurSolver(p, config.s_x, config.s_y, tol=tol, max_iter=2000, augment=augment)
        try:
            out = solver.solve()
        finally:
            solver.close()
        row.iters_plus = out["plus_stats"]["iterations"]
        row.iters_minus = out["minus_stats"]["iterations"]
        row.converged = out["converged"]
        row.relative_residual = max(out["plus_stats"]["relative_residual"], out["minus_stats"]["relative_residual"])
        row.build_seconds = out["factor_setup_seconds"]
        row.per_solve_seconds = out["solve_seconds"]
        _fill_diagnostics(row, p, out["y"], out["u"], out["lambda"], out["imag_leak"])
    except (ContractError, NumericalError, RuntimeError) as e:
        row.error, row.converged = _sanitize(str(e)), False
    row.total_seconds = time.perf_counter() - t0
    rows.append(row)


def run_phi_sweep(config: ExperimentConfig, cache=None):  # experiments.cpp:244-283
    config.validate()
    rows = []
    for phi in config.phi:
        p = _build_problem(config, config.n, phi)
        for augment in (False, True):
            _range_space_row(config, p, phi, augment, config.feti_tol, cache, rows)
    return rows


def run_scalability(config: ExperimentConfig, cache=None):  # experiments.cpp:285-322
    config.validate()
    if config.physics != "heat":
        raise ContractError("run_scalability: the scalability study runs on the thermal problem")
    phi = config.phi[0] if config.phi else 2e-8
    rows = []
    for n in config.mesh_sizes:
        if n % config.ratio != 0:
            raise ContractError("run_scalability: mesh size must be divisible by the H/h ratio")
        local = ExperimentConfig(**{f.name: getattr(config, f.name) for f in fields(config)})
        local.n, local.s_x, local.s_y = n, n // config.ratio, n // config.ratio
        p = _build_problem(local, n, phi)
        _range_space_row(local, p, phi, config.augment, config.feti_tol, cache, rows)
        rows[-1].config_hash = config.hash()  # the hash of the experiment, not of the derived config
    return rows


def _full_space_row(config, p, phi, backend, tol, inner_tol, max_iter, cache, rows):
    t0 = time.perf_counter()
    row = _base_row(config, p, phi)
    row.method, row.backend, row.augment = "full_space", backend, True
    if cache and row.key() in cache:
        rows.append(cache[row.key()])
        return None
    sol = None
    try:
        out = solve_full_space(p, precond=backend, outer="gmres", tol=tol, inner_tol=inner_tol, s_x=config.s_x,
                               s_y=config.s_y, augment=True, max_iter=max_iter)
        st = out["stats"]
        row.outer_iters, row.converged, row.relative_residual = st["iterations"], st["converged"], st["relative_residual"]
        row.build_seconds = out["precond_setup_seconds"]
        row.per_solve_seconds = st["wall_time"] / st["iterations"] if st["iterations"] > 0 else 0.0
        _fill_diagnostics(row, p, out["y"], out["u"], out["lambda"], out["imag_leak"])
        sol = np.concatenate([out["y"], out["u"], out["lambda"]])
    except (ContractError, NumericalError, RuntimeError) as e:
        row.error, row.converged = _sanitize(str(e)), False
    row.total_seconds = time.perf_counter() - t0
    rows.append(row)
    return sol


def run_precond_compare(config: ExperimentConfig, cache=None):  # experiments.cpp:324-381
    config.validate()
    rows = []
    for phi in config.phi:
        p = _build_problem(config, config.n, phi)
        sols = [_full_space_row(config, p, phi, b, config.outer_tol, config.inner_tol, 2000, cache, rows)
                for b in ("sp", "sc")]
        if sols[0] is not None and sols[1] is not None:
            gap = float(np.linalg.norm(sols[0] - sols[1]) / max(np.linalg.norm(sols[1]), 1e-300))
            rows[-1].cross_agreement = rows[-2].cross_agreement = gap
    return rows


def run_accuracy_cliff(config: ExperimentConfig, cache=None):  # experiments.cpp:383-460
    config.validate()
    rows = []
    for phi in config.phi:
        p = _build_problem(config, config.n, phi)
        row = _base_row(config, p, phi)
        row.method, row.backend = "range_space", "direct"
        if cache and row.key() in cache:
            rows.append(cache[row.key()])
        else:
            row.error = "backend 'direct' not provided by the B200 path (sparse LU on the CPU)"
            rows.append(row)
        _full_space_row(config, p, phi, "sc", config.outer_tol, config.inner_tol, 300, cache, rows)
        rows[-1].augment = False
    return rows


def parse_rows_file(path: str):
    with open(path) as f:
        text = f.read()
    return parse_rows_json(text) if text.lstrip().startswith("{") else parse_rows_csv(text)


def run_experiment(config: ExperimentConfig, out_path: str = ""):  # experiments.cpp:462-488
    config.validate()
    cache = None
    if out_path and os.path.exists(out_path):
        try:
            prev = parse_rows_file(out_path)
        except Exception:  # unreadable caches are recomputed
            prev = []
        h = config.hash()
        cache = {r.key(): r for r in prev if r.config_hash == h} or None
    return {"phi_sweep": run_phi_sweep, "scalability": run_scalability, "precond_compare": run_precond_compare,
            "accuracy_cliff": run_accuracy_cliff}[config.kind](config, cache)


# ------------------------------------------------------------------------ row I/O
def _cell(r: ResultRow, c: str) -> str:
    v = getattr(r, c)
    if c in _BOOL:
        return "1" if v else "0"
    if c in _INT or c in _STR:
        return str(v)
    return _fmt17(v)


def rows_to_csv(rows) -> str:  # experiments.cpp:538-560
    out = io.StringIO()
    out.write("# pdeopt-results schema=1" + (f" config={rows[0].config_hash}" if rows else "") + "\n")
    out.write(",".join(COLUMNS) + "\n")
    for r in rows:
        out.write(",".join(_cell(r, c) for c in COLUMNS) + "\n")
    return out.getvalue()


def parse_rows_csv(text: str):
    rows = []
    lines = [ln for ln in text.splitlines() if ln and not ln.startswith("#")]
    for ln in lines[1:]:
        cells = next(csv.reader([ln]))
        cells += [""] * (len(COLUMNS) - len(cells))
        if len(cells) != len(COLUMNS):
            raise NumericalError(f"parse_rows_csv: column count mismatch in line: {ln}")
        r = ResultRow()
        for c, v in zip(COLUMNS, cells):
            setattr(r, c, int(v) if c in _INT else (v == "1") if c in _BOOL else v if c in _STR else float(v))
        rows.append(r)
    return rows


def rows_to_json(rows) -> str:  # experiments.cpp:686-695
    obj = {"schema_version": 1, "config_hash": rows[0].config_hash if rows else "",
           "rows": [{c: getattr(r, c) for c in COLUMNS} for r in rows]}
    return json.dumps(obj, indent=2, sort_keys=True)


def parse_rows_json(text: str):
    rows = []
    for item in json.loads(text)["rows"]:
        r = ResultRow()
        for c in COLUMNS:
            v = item[c]
            setattr(r, c, int(v) if c in _INT else bool(v) if c in _BOOL else str(v) if c in _STR else float(v))
        rows.append(r)
    return rows


def emit_rows(rows, fmt: str, path: str, allow_empty: bool = False):  # experiments.cpp:490-505
    if not rows and not allow_empty:
        raise ContractError("emit_rows: refusing to write an empty result set (pass allow_empty)")
    if fmt == "csv":
        text = rows_to_csv(rows)
    elif fmt == "json":
        text = rows_to_json(rows)
    else:
        raise ContractError(f"emit_rows: unknown format '{fmt}'")
    with open(path, "w") as f:
        f.write(text)


def run_experiment_json(config_json: str, out_path: str = "") -> str:
    """bindings.cpp:187-195: run one experiment from a JSON config, rows back as JSON."""
    return rows_to_json(run_experiment(ExperimentConfig.from_json(config_json), out_path))


def default_config_json(kind: str) -> str:
    return ExperimentConfig.defaults_for(kind).to_json()


__all__ = ["ExperimentConfig", "ResultRow", "COLUMNS", "WALL_TIME_COLUMNS", "run_phi_sweep", "run_scalability",
           "run_precond_compare", "run_accuracy_cliff", "run_experiment", "run_experiment_json",
           "default_config_json", "rows_to_csv", "rows_to_json", "parse_rows_csv", "parse_rows_json",
           "parse_rows_file", "emit_rows"]
