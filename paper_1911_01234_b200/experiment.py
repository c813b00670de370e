"""Experiment runner on the B200 path (mirrors src/cli.py, src/config.py).

Same YAML config, seeds, substreams and artifacts as the reference CLI
(src/cli.py:40-164), with the reconstructions on the GPU: all VDAMP cells of
one experiment (one per undersampling factor, each with its own mask and
density) run as ONE batched ``run_batch``; FISTA (with its lambda grid tuned
as one batch) and SURE-IT run per cell through :mod:`.baselines`.

    python -m paper_1911_01234_b200.experiment run --config exp.yaml --device cuda
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
import traceback
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

from . import artifacts

QQ_ITERS = (0, 1, 2)


class ConfigError(ValueError):
    """Malformed or unparsable configuration (src/config.py:11-12)."""


@dataclass
class DensityConfig:
    degree: int = 8
    center_radius: float = 0.02
    p_min: float = 1e-3


@dataclass
class AlgorithmConfig:
    n_iters: int = 30
    lam: float | None = None
    lambda_grid: list = field(default_factory=list)
    tune_budget: int | None = None


@dataclass
class ExperimentConfig:
    """src/config.py:31-90 (same fields, defaults and validation messages)."""

    phantom_size: int = 64
    scales: int = 4
    snr_db: float | None = 40.0
    undersampling: list = field(default_factory=lambda: [4.0])
    density: DensityConfig = field(default_factory=DensityConfig)
    algorithms: dict = field(default_factory=lambda: {"vdamp": AlgorithmConfig()})
    seed: int = 0
    output_dir: str = "runs"

    def to_dict(self) -> dict:
        return asdict(self)

    def validate(self) -> list:
        out = []
        if self.phantom_size < 16:
            out.append(f"phantom_size {self.phantom_size} below minimum 16")
        if self.scales < 1:
            out.append(f"scales must be >= 1, got {self.scales}")
        elif self.phantom_size % (2 ** self.scales):
            out.append(f"phantom_size {self.phantom_size} not divisible by 2^{self.scales}")
        if not self.undersampling:
            out.append("no undersampling factors given")
        out += [f"undersampling factor {r} < 1" for r in self.undersampling if r < 1]
        d = self.density
        if d.degree < 1:
            out.append(f"density degree must be >= 1, got {d.degree}")
        if not 0 <= d.center_radius < 1:
            out.append(f"center_radius {d.center_radius} outside [0, 1)")
        if not 0 < d.p_min <= 1:
            out.append(f"p_min {d.p_min} outside (0, 1]")
        if not self.algorithms:
            out.append("no algorithms selected")
        for name, a in self.algorithms.items():
            if name not in ("vdamp", "fista", "sure_it"):
                out.append(f"unknown algorithm {name!r}")
                continue
            if a.n_iters < 1:
                out.append(f"{name}: n_iters must be >= 1")
            if name == "fista":
                if a.lam is None and not a.lambda_grid:
                    out.append("fista: needs lam or lambda_grid")
                if a.lam is not None and a.lam <= 0:
                    out.append(f"fista: lam must be > 0, got {a.lam}")
                if any(g <= 0 for g in a.lambda_grid):
                    out.append("fista: lambda_grid entries must be > 0")
        if self.snr_db is not None and self.snr_db <= 0:
            out.append(f"snr_db must be > 0 or null (noiseless), got {self.snr_db}")
        return out


def config_from_dict(raw: dict) -> ExperimentConfig:
    raw = dict(raw)
    try:
        dens = DensityConfig(**raw.pop("density", {}))
        algs = {k: AlgorithmConfig(**(v or {})) for k, v in raw.pop("algorithms", {"vdamp": {}}).items()}
        return ExperimentConfig(density=dens, algorithms=algs, **raw)
    except TypeError as exc:
        raise ConfigError(f"unrecognized config field: {exc}") from exc


def load_config(path) -> ExperimentConfig:
    import yaml
    path = Path(path)
    try:
        raw = yaml.safe_load(path.read_text())
    except yaml.YAMLError as exc:
        raise ConfigError(f"cannot parse {path}: {exc}") from exc
    if not isinstance(raw, dict):
        raise ConfigError(f"{path}: expected a mapping at top level")
    return config_from_dict(raw)


def validate_config(path) -> list:
    try:
        return load_config(path).validate()
    except ConfigError as exc:
        return [str(exc)]


def _substream(master: int, r_index: int, role: int) -> np.random.SeedSequence:
    return np.random.SeedSequence(entropy=master, spawn_key=(r_index, role))


def _rtag(r: float) -> str:
    return f"{r:g}"


def _vdamp_cells(config, out, cells, x0, w0, precision):
    """All VDAMP cells as one batch (src/cli.py:51-72 per cell)."""
    from . import vdamp
    a = config.algorithms["vdamp"]
    keep = tuple(k for k in QQ_ITERS if k < a.n_iters)
    xs, traces = vdamp.run_batch([c["y"] for c in cells], [c["mask"] for c in cells],
                                 [c["pmap"] for c in cells], [c["noise_var"] for c in cells],
                                 config.scales, a.n_iters, [x0] * len(cells), keep, precision=precision)
    infos = []
    for c, x_hat, trace in zip(cells, xs, traces):
        tag = _rtag(c["r"])
        entries = []
        for k, snap in sorted(trace.r_snapshots.items()):
            for j, b in enumerate(snap.layout.subbands):
                res = snap.subband(j) - w0.subband(j)
                if res.size < 16:
                    continue
                for qq in artifacts.qq_data(res, min(100, res.size)):
                    entries.append((k, j, qq))
            mosaic = np.abs(artifacts.coeff_mosaic(snap.values, snap.layout)
                            - artifacts.coeff_mosaic(w0.values, w0.layout))
            artifacts.save_array(out / f"resid_vdamp_R{tag}_k{k}.bin", mosaic,
                                 {"undersampling": c["r"], "iteration": k})
        run_id = f"vdamp_R{tag}"
        artifacts.write_qq_csv(out / f"qq_vdamp_R{tag}.csv", run_id, entries)
        infos.append(_finish(out, run_id, "vdamp", c["r"], a.n_iters, x_hat, trace,
                             {"precompute_time": trace.precompute_time}))
    return infos


def _finish(out, run_id, alg, r, n_iters, x_hat, trace, extra):
    artifacts.write_trace_csv(out / f"trace_{run_id}.csv", run_id, trace)
    artifacts.save_array(out / f"xhat_{run_id}.bin", x_hat, {"algorithm": alg, "undersampling": r})
    info = {"algorithm": alg, "undersampling": r, "n_iters": n_iters}
    info.update(extra)
    info["final_nmse_db"] = trace.records[-1].nmse_db
    info["mean_iteration_time"] = trace.mean_iteration_time()
    return info


def _baseline_cell(config, out, c, alg, x0, w0, precision):
    from . import baselines
    a = config.algorithms[alg]
    run_id = f"{alg}_R{_rtag(c['r'])}"
    if alg == "fista":
        lam = a.lam
        if lam is None:
            lam = baselines.tune_lambda(c["y"], c["mask"], x0, a.tune_budget or a.n_iters,
                                        np.array(a.lambda_grid), config.scales, precision=precision)
        x_hat, trace = baselines.fista(c["y"], c["mask"], lam, a.n_iters, config.scales, ground_truth=x0,
                                       precision=precision)
        return _finish(out, run_id, alg, c["r"], a.n_iters, x_hat, trace, {"lam": lam})
    x_hat, trace = baselines.sure_it(c["y"], c["mask"], w0, a.n_iters, config.scales, ground_truth=x0,
                                     precision=precision)
    return _finish(out, run_id, alg, c["r"], a.n_iters, x_hat, trace, {})


def run_experiment(config: ExperimentConfig, out_dir=None, threads: int = 1, *, precision="fp64") -> Path:
    """src/cli.py:104-164 on the GPU.  ``threads`` is accepted for CLI
    compatibility; the GPU batches the cells instead."""
    from .sampling import draw_mask, polynomial_pmap, shepp_logan, synthesize
    from .wavelet import dwt
    problems = config.validate()
    if problems:
        raise ConfigError("; ".join(problems))
    out = Path(out_dir if out_dir is not None else config.output_dir)
    out.mkdir(parents=True, exist_ok=True)
    n = config.phantom_size
    x0 = shepp_logan(n, n)
    w0 = dwt(x0, config.scales, precision="fp64")
    artifacts.save_array(out / "phantom.bin", x0, {"size": n})
    energies = [float(np.vdot(w0.subband(j), w0.subband(j)).real) for j in range(w0.layout.n_subbands)]
    cells = []
    for ri, r in enumerate(config.undersampling):
        d = config.density
        pmap = polynomial_pmap(n, n, d.degree, d.center_radius, r, d.p_min)
        mask = draw_mask(pmap, _substream(config.seed, ri, 0))
        kd = synthesize(x0, mask, config.snr_db, _substream(config.seed, ri, 1))
        tag = _rtag(r)
        artifacts.save_array(out / f"pmap_R{tag}.bin", pmap.probs,
                             {"undersampling": r, "degree": d.degree, "center_radius": d.center_radius,
                              "p_min": d.p_min, "seed": config.seed})
        artifacts.save_array(out / f"mask_R{tag}.bin", mask.sampled.astype(np.uint8),
                             {"undersampling": r, "n": mask.n, "seed": config.seed})
        artifacts.write_subband_csv(out / f"subbands_R{tag}.csv", w0.layout, energies)
        cells.append({"r": r, "y": kd.values, "mask": mask, "pmap": pmap, "noise_var": kd.noise_var})
    started = time.time()
    results = {}
    if "vdamp" in config.algorithms:
        for i, info in enumerate(_vdamp_cells(config, out, cells, x0, w0, precision)):
            results[(i, "vdamp")] = info
    for i, c in enumerate(cells):
        for alg in config.algorithms:
            if alg != "vdamp":
                results[(i, alg)] = _baseline_cell(config, out, c, alg, x0, w0, precision)
    ordered = [results[(i, alg)] for i in range(len(cells)) for alg in config.algorithms]
    cfg = config.to_dict()
    manifest = {
        "config": cfg,
        "config_sha256": hashlib.sha256(json.dumps(cfg, sort_keys=True).encode()).hexdigest(),
        "seed": config.seed,
        "substreams": {_rtag(r): {"mask": [config.seed, i, 0], "noise": [config.seed, i, 1]}
                       for i, r in enumerate(config.undersampling)},
        "cells": ordered,
        "elapsed_seconds": time.time() - started,
    }
    (out / "manifest.json").write_text(json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    return out


def list_outputs(root: Path) -> list:
    found = []
    for mp in sorted(Path(root).rglob("manifest.json")):
        try:
            m = json.loads(mp.read_text())
        except (OSError, json.JSONDecodeError):
            continue
        found.append({"directory": str(mp.parent), "seed": m.get("seed"),
                      "cells": [f"{c['algorithm']} R={c['undersampling']:g} "
                                f"NMSE={c.get('final_nmse_db') or float('nan'):.1f}dB"
                                for c in m.get("cells", [])]})
    return found


def _parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="csmri", description="Compressed-sensing MRI experiment runner (B200)")
    sub = p.add_subparsers(dest="verb", required=True)
    rp = sub.add_parser("run", help="run the configured experiment")
    rp.add_argument("--config", required=True, type=Path)
    rp.add_argument("--seed", type=int, default=None)
    rp.add_argument("--out", type=Path, default=None)
    rp.add_argument("--threads", type=int, default=1)
    rp.add_argument("--device", default="cuda", choices=["cuda"],
                    help="the reconstructions run on the GPU (no CPU path)")
    rp.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    vp = sub.add_parser("validate", help="check a config without running")
    vp.add_argument("--config", required=True, type=Path)
    lp = sub.add_parser("list-outputs", help="summarize completed runs")
    lp.add_argument("--out", type=Path, default=Path("runs"))
    return p


def main(argv=None) -> int:
    """Same verbs and exit codes as src/cli.py:167-237."""
    args = _parser().parse_args(argv)
    if args.verb == "validate":
        try:
            problems = validate_config(args.config)
        except OSError as exc:
            print(f"error: {exc}", file=sys.stderr)
            return 2
        for pr in problems:
            print(f"violation: {pr}")
        return 2 if problems else 0
    if args.verb == "list-outputs":
        for e in list_outputs(args.out):
            print(e["directory"])
            for c in e["cells"]:
                print(f"  {c}")
        return 0
    try:
        config = load_config(args.config)
        problems = config.validate()
        if problems:
            for pr in problems:
                print(f"invalid config: {pr}", file=sys.stderr)
            return 2
        if args.seed is not None:
            config.seed = args.seed
        out = run_experiment(config, args.out, threads=args.threads, precision=args.precision)
    except (ConfigError, OSError) as exc:
        print(f"invalid config: {exc}", file=sys.stderr)
        return 2
    except Exception:
        traceback.print_exc()
        return 1
    print(out)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
