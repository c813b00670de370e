"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (it imports csmri from /root/reference):

    python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  The fixtures pin ``oracle/vdamp_oracle.py``
(tests/test_oracle.py) and are also compared directly against the CUDA path
(tests/test_gpu_*.py).  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from csmri import vdamp
    from csmri.denoise import SubbandVector, _threshold_scan, denoise_colored
    from csmri.fourier import adjoint, fft2c, forward, ifft2c
    from csmri.sampling import draw_mask, polynomial_pmap, shepp_logan, synthesize
    from csmri.wavelet import SubbandLayout, WaveletCoeffs, dwt, idwt

    rng = np.random.default_rng(20261020)

    # ---- operators: dwt / idwt / fft2c / ifft2c ------------------------
    ops = {}
    for (h, w, s) in [(2, 2, 1), (8, 8, 2), (16, 32, 3), (32, 16, 2), (64, 64, 4), (64, 64, 6)]:
        x = rng.normal(size=(h, w)) + 1j * rng.normal(size=(h, w))
        c = rng.normal(size=h * w) + 1j * rng.normal(size=h * w)
        layout = SubbandLayout.create(h, w, s)
        key = f"{h}x{w}s{s}"
        ops[f"dwt_in_{key}"] = x
        ops[f"dwt_out_{key}"] = dwt(x, s).values
        ops[f"idwt_in_{key}"] = c
        ops[f"idwt_out_{key}"] = idwt(WaveletCoeffs(c, layout))
        ops[f"offsets_{key}"] = np.array([b.offset for b in layout.subbands])
        ops[f"fft_out_{key}"] = fft2c(x)
        ops[f"ifft_out_{key}"] = ifft2c(x)
    # unit-atom spectra (the reference's own construction)
    for (h, w, s) in [(16, 16, 2), (32, 64, 3)]:
        sp = vdamp.compute_spectra(SubbandLayout.create(h, w, s))
        ops[f"spectra_{h}x{w}s{s}"] = sp.profiles
    np.savez_compressed(os.path.join(OUT, "operators.npz"), **ops)

    # ---- threshold scan known answers ----------------------------------
    scan = {}
    cases = [
        np.array([0.0, 0.0, 1.0, 1.0, 1.0, 2.0]),
        np.array([0.5]),
        np.array([0.0]),
        np.array([3.0, 3.0, 3.0, 3.0]),
        np.array([1e-12, 1.0, 1.0 + 1e-15, 2.0, 50.0]),
    ]
    taus = [0.5, 1.0, 0.3, 2.0, 0.7]
    for _ in range(24):
        n = int(rng.choice([4, 16, 64, 256, 1024, 4096]))
        sig = np.abs(rng.normal(size=n) + 1j * rng.normal(size=n))
        sparse = np.where(rng.random(n) < 0.1, rng.exponential(5.0, n), 0.0)
        mags = np.abs(sig * rng.uniform(0.2, 2.0) + sparse)
        if rng.random() < 0.3:
            mags[: n // 8] = 0.0
        if rng.random() < 0.3:
            mags = np.round(mags, 1)        # many ties
        cases.append(mags)
        taus.append(float(rng.uniform(0.05, 3.0)))
    for i, (m, tau) in enumerate(zip(cases, taus)):
        ms = np.sort(m)
        t, cnt, inv = _threshold_scan(ms, tau)
        scan[f"mag_{i}"] = ms
        scan[f"tau_{i}"] = np.array(tau)
        scan[f"out_{i}"] = np.array([t, cnt, inv])
        ms32 = np.sort(m.astype(np.float32)).astype(np.float64)
        scan[f"out32_{i}"] = np.array(_threshold_scan(ms32, tau))
    scan["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "threshold_scan.npz"), **scan)

    # ---- denoise_colored ----------------------------------------------
    den = {}
    for (h, w, s) in [(32, 32, 2), (64, 32, 3)]:
        layout = SubbandLayout.create(h, w, s)
        r = rng.normal(size=h * w) + 1j * rng.normal(size=h * w)
        r[: layout.subbands[0].length] *= 20.0
        tau = rng.uniform(0.2, 2.0, layout.n_subbands)
        wh, al, lam = denoise_colored(WaveletCoeffs(r, layout), SubbandVector(tau))
        key = f"{h}x{w}s{s}"
        den[f"r_{key}"] = r
        den[f"tau_{key}"] = tau
        den[f"what_{key}"] = wh.values
        den[f"alpha_{key}"] = al.values
        den[f"lambda_{key}"] = lam.values
    np.savez_compressed(os.path.join(OUT, "denoise.npz"), **den)

    # ---- full runs ------------------------------------------------------
    def record_run(name, x0, pmap, mask, kdata, scales, n_iters, gt=True, keep=(), steps=0):
        x_hat, trace = vdamp.run(kdata.values, mask, pmap, kdata.noise_var, scales, n_iters,
                                 ground_truth=x0 if gt else None, keep_r_iters=keep)
        d = dict(
            x0=x0, probs=pmap.probs, sampled=mask.sampled, y=kdata.values,
            noise_var=np.array(kdata.noise_var), scales=np.array(scales),
            n_iters=np.array(n_iters), x_hat=x_hat,
            tau=np.array([r.tau for r in trace.records]),
            thresholds=np.array([r.thresholds for r in trace.records]),
            lambdas=np.array([r.lambdas for r in trace.records]),
            alphas=np.array([r.alphas for r in trace.records]),
            clamped=np.array([r.alpha_clamped for r in trace.records]),
        )
        if gt:
            d["nmse_db"] = trace.nmse_curve()
            d["subband_nmse_db"] = np.array([r.subband_nmse_db for r in trace.records])
        for k in keep:
            d[f"snap_{k}"] = trace.r_snapshots[k].values
        # teacher-forcing fixtures: the first `steps` iterate() states
        layout = SubbandLayout.create(x0.shape[0], x0.shape[1], scales)
        spectra = vdamp.compute_spectra(layout)
        st = vdamp.initial_state(layout)
        for k in range(steps):
            d[f"step{k}_rtilde_in"] = st.r_tilde.values.copy()
            st = vdamp.iterate(st, kdata.values, mask, pmap, kdata.noise_var, spectra)
            d[f"step{k}_r"] = st.r.values
            d[f"step{k}_z"] = st.z
            d[f"step{k}_tau"] = st.tau.values
            d[f"step{k}_thr"] = st.thresholds
            d[f"step{k}_alpha"] = st.alpha.values
            d[f"step{k}_what"] = st.w_hat.values
            d[f"step{k}_rtilde_out"] = st.r_tilde.values
        d["steps"] = np.array(steps)
        np.savez_compressed(os.path.join(OUT, f"run_{name}.npz"), **d)

    x0 = shepp_logan(32, 32)
    pmap = polynomial_pmap(32, 32, 8, 0.02, 3.0)
    mask = draw_mask(pmap, 0)
    record_run("shepp32", x0, pmap, mask, synthesize(x0, mask, 40.0, 1), 2, 6,
               keep=(0, 2), steps=2)

    x0 = shepp_logan(64, 64)
    pmap = polynomial_pmap(64, 64, 8, 0.02, 4.0)
    mask = draw_mask(pmap, 5)
    record_run("shepp64", x0, pmap, mask, synthesize(x0, mask, 40.0, 6), 4, 10, steps=3)

    x0 = shepp_logan(64, 32) * np.exp(1j * np.linspace(0, 1, 32))[None, :]
    pmap = polynomial_pmap(64, 32, 8, 0.02, 2.5)
    mask = draw_mask(pmap, 9)
    record_run("rect64x32", x0, pmap, mask, synthesize(x0, mask, 35.0, 10), 3, 8, steps=2)

    x0 = shepp_logan(128, 128)
    pmap = polynomial_pmap(128, 128, 8, 0.02, 6.0)
    mask = draw_mask(pmap, 11)
    record_run("shepp128", x0, pmap, mask, synthesize(x0, mask, 40.0, 12), 4, 12, gt=True)

    # full sampling, noiseless: one iteration recovers x0 exactly
    x0 = shepp_logan(64, 64)
    pmap = polynomial_pmap(64, 64, 8, 0.02, 1.0)
    mask = draw_mask(pmap, 0)
    record_run("full64", x0, pmap, mask, synthesize(x0, mask, None), 4, 1)

    # baselines on the same operators (src/baselines.py)
    from csmri import baselines
    x0 = shepp_logan(64, 64)
    pmap = polynomial_pmap(64, 64, 8, 0.02, 4.0)
    mask = draw_mask(pmap, 5)
    kd = synthesize(x0, mask, 40.0, 6)
    xf, trf = baselines.fista(kd.values, mask, 0.01, 12, 4, ground_truth=x0)
    w0 = dwt(x0, 4)
    xs, trs = baselines.sure_it(kd.values, mask, w0, 10, 4, ground_truth=x0)
    grid = np.geomspace(1e-4, 1e-1, 6)
    lam = baselines.tune_lambda(kd.values, mask, x0, 8, grid, 4)
    np.savez_compressed(
        os.path.join(OUT, "baselines.npz"),
        x0=x0, sampled=mask.sampled, y=kd.values, noise_var=np.array(kd.noise_var),
        fista_x=xf, fista_nmse=trf.nmse_curve(), fista_sbn=np.array([r.subband_nmse_db for r in trf.records]),
        sure_x=xs, sure_nmse=trs.nmse_curve(), sure_tau=np.array([r.tau for r in trs.records]),
        sure_thr=np.array([r.thresholds for r in trs.records]),
        sure_sbn=np.array([r.subband_nmse_db for r in trs.records]),
        grid=grid, lam=np.array(lam),
    )

    # density + mask pin for the workload generator (reference disc centre)
    pm = polynomial_pmap(64, 48, 8, 0.02, 4.0)
    pm6 = polynomial_pmap(96, 96, 6, 0.1, 5.0)
    np.savez_compressed(
        os.path.join(OUT, "sampling.npz"),
        probs_64x48=pm.probs, mask_64x48_seed7=draw_mask(pm, 7).sampled,
        probs_96_d6=pm6.probs,
    )
    cli_golden()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


CLI_CONFIG = {
    "phantom_size": 32, "scales": 3, "snr_db": 40.0, "undersampling": [3.0, 5.0],
    "density": {"degree": 8, "center_radius": 0.02, "p_min": 1e-3},
    "algorithms": {"vdamp": {"n_iters": 8},
                   "fista": {"n_iters": 6, "lambda_grid": [1e-3, 1e-2, 1e-1], "tune_budget": 4},
                   "sure_it": {"n_iters": 6}},
    "seed": 11,
}


def cli_golden():
    """Every artifact of one reference ``run_experiment`` (src/cli.py:104-164),
    packed as text (CSV/JSON) and arrays (.bin) into cli.npz."""
    import json
    import tempfile
    sys.path.insert(0, REF)
    from csmri import cli, io
    from csmri.config import config_from_dict
    d = {"config_json": np.array(json.dumps(CLI_CONFIG))}
    with tempfile.TemporaryDirectory() as tmp:
        cli.run_experiment(config_from_dict(json.loads(json.dumps(CLI_CONFIG))), tmp)
        names = sorted(os.listdir(tmp))
        d["files"] = np.array(names)
        for f in names:
            path = os.path.join(tmp, f)
            if f.endswith(".bin"):
                arr, _ = io.load_array(path)
                d["bin:" + f] = arr
            else:
                with open(path) as fh:
                    d["txt:" + f] = np.array(fh.read())
    np.savez_compressed(os.path.join(OUT, "cli.npz"), **d)


def bench512_golden():
    """The reference's own benchmark fixture (tests/conftest.py:101-132 of the
    reference): Shepp-Logan 512^2, Haar s=4, polynomial density (d=8, centre
    0.02, R=8), mask seed 3, noise seed 103, 40 dB, 30 iterations with ground
    truth.  Its recorded result is -35.5 dB at iteration 30 (test_output.txt).
    The inputs are regenerated at test time by paper_1911_01234_b200.sampling
    (pinned bit-exact here through the mask bits, y checksums and noise_var);
    x_hat is stored on a stride-8 grid plus 16 random projections."""
    sys.path.insert(0, REF)
    from csmri import vdamp
    from csmri.sampling import draw_mask, polynomial_pmap, shepp_logan, synthesize
    size, scales, n_iters = 512, 4, 30
    x0 = shepp_logan(size, size)
    pmap = polynomial_pmap(size, size, 8, 0.02, 8.0)
    mask = draw_mask(pmap, 3)
    kd = synthesize(x0, mask, 40.0, 103)
    x_hat, trace = vdamp.run(kd.values, mask, pmap, kd.noise_var, scales, n_iters, ground_truth=x0)
    proj = np.random.default_rng(512).normal(size=(16, size * size))
    np.savez_compressed(
        os.path.join(OUT, "bench512.npz"),
        mask_bits=np.packbits(mask.sampled.ravel()), n=np.array(mask.n),
        y_sum=np.array([kd.values.real.sum(), kd.values.imag.sum()]), y_norm=np.array(np.linalg.norm(kd.values)),
        noise_var=np.array(kd.noise_var), scales=np.array(scales), n_iters=np.array(n_iters),
        x_hat_grid=x_hat[::8, ::8], x_hat_norm=np.array(np.linalg.norm(x_hat)),
        x_hat_proj=proj @ x_hat.ravel(), proj_seed=np.array(512),
        nmse_db=trace.nmse_curve(),
        tau=np.array([r.tau for r in trace.records]),
        thresholds=np.array([r.thresholds for r in trace.records]),
        alphas=np.array([r.alphas for r in trace.records]),
        clamped=np.array([r.alpha_clamped for r in trace.records]),
        subband_nmse_db=np.array([r.subband_nmse_db for r in trace.records]),
    )
    print("bench512: nmse at iteration 30 =", trace.nmse_curve()[-1])


if __name__ == "__main__":
    if sys.argv[1:] == ["cli"]:
        cli_golden()
    elif sys.argv[1:] == ["bench512"]:
        bench512_golden()
    else:
        main()
