"""Generate the golden parity fixtures from the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``pauli_lre`` from ``/root/reference/pkg/src`` (numba cache
redirected to /tmp so nothing is written into the read-only tree), runs the
reference's own step (i)/(ii)/(iii) on seeded inputs and writes the inputs and
outputs under ``tests/golden/``.  The GPU box never reads /root/reference: the
tests there only read these committed fixtures.

Cases:
  kat.npz          SPEC known-answer tests KAT1/2/4/5/8
  blocks_n3.npz    index-map building blocks (pauli.py:153-297) at n=3
  c1_*.npz         n=4 GHZ exact (shots 16) and sampled (1000 shots, seed 1602)
  small_*.npz      n=1..6 random/productz/maxmixed records (KAT10-style)
  c2_w8.npz        n=8 W state, 1000 shots, seed 1602 (counts stored as uint16)
  c3_random10.npz  n=10 Ginibre state (_random_density(10, 8604)), 1000 shots,
                   seed 1602 — counts are NOT stored (120 MB); the fixture
                   holds their sha256 and strided samples of theta/mu; the
                   tests regenerate the counts with the oracle's restatement
                   of simulate.sample_counts and check the hash first.
  validate.npz     MeasurementRecord.validate error messages.
  files/           file formats written by the reference itself: a
                   pauli-lre/1 text record (records.py:67-84), a PLRE v1
                   state file (statefile.py:19-29), and the messages its
                   readers raise on the perturbations tests/test_recordio.py
                   applies (files/messages.json).

  metrics.npz      reference metrics.py on reference reconstructions:
                   evaluate_errors reports (ghz4 sampled, maxmixed4 sampled,
                   productz3 sampled), predicted_mse_dense for dense states
                   n <= 4, fidelity (auto and general) on random pairs.

Run a subset with `python tests/golden/make_golden.py files`.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_golden"))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from pauli_lre import pauli, pipeline, simulate  # noqa: E402  (the reference)
from pauli_lre.records import MeasurementRecord  # noqa: E402

from oracle import lre_oracle as O  # noqa: E402
from perturb import record_perturbations, state_perturbations  # noqa: E402

SEED = 1602


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.1f} KiB)")


def _run_reference(counts, n, shots, with_step3=True):
    rec = MeasurementRecord(n=n, shots=shots, counts=np.asarray(counts, dtype=np.int64))
    theta = pipeline.step_one_least_squares(rec, workers=1)
    mu = pipeline.step_two_assemble(theta, workers=1)
    out = dict(counts=np.asarray(counts), n=n, shots=shots, theta=theta, mu=mu)
    if with_step3:
        rho, ev = pipeline.step_three_project(mu)
        out.update(rho=rho, eigenvalues=ev)
    return out


def _reference_sample_from_rho(rho, n, shots, seed):
    """Reference primitives: dense_to_theta (complex) -> _theta_probability_block
    -> _setting_rng(seed, w).multinomial (simulate.py:114-151, 216-242)."""
    theta = simulate.dense_to_theta(np.asarray(rho, dtype=np.complex128))
    settings = 3**n
    counts = np.empty((settings, 1 << n), dtype=np.int64)
    block = max(1, (1 << 18) >> n)
    for start in range(0, settings, block):
        stop = min(settings, start + block)
        probs = np.clip(simulate._theta_probability_block(theta, start, stop, n), 0.0, 1.0)
        for row, w in enumerate(range(start, stop)):
            p = np.clip(probs[row], 0.0, None)
            counts[w] = simulate._setting_rng(seed, w).multinomial(shots, p / p.sum())
    return counts


def kat():
    sq2 = 1.0 / np.sqrt(2.0)
    kat1_counts = np.array([[1, 1], [1, 1], [2, 0]], dtype=np.int64)
    kat2_counts = np.array([[1, 1], [1, 1], [1, 1]], dtype=np.int64)
    t1 = pipeline.step_one_least_squares(MeasurementRecord(1, 2, kat1_counts))
    t2 = pipeline.step_one_least_squares(MeasurementRecord(1, 2, kat2_counts))
    assert np.allclose(t1, [sq2, 0, 0, sq2]) and np.allclose(t2, [sq2, 0, 0, 0])
    mu4 = pipeline.step_two_assemble(np.array([sq2, 0, 0, sq2]))
    mu5 = pipeline.step_two_assemble(np.array([sq2, 0, 0, 0]))
    p8a = pipeline.project_spectrum_to_simplex(np.array([1.02, 0.04, -0.03, -0.03]))
    p8b = pipeline.project_spectrum_to_simplex(np.array([0.6, 0.5, -0.1]))
    _save("kat.npz", kat1_counts=kat1_counts, kat1_theta=t1, kat2_counts=kat2_counts, kat2_theta=t2,
          kat4_mu=mu4, kat5_mu=mu5, kat8a=p8a, kat8b=p8b)


def blocks():
    n = 3
    locs = pauli.nonzero_locations_block(pauli.setting_digit_rows(0, 3**n, n), n)
    gather = np.stack([pauli.omega_gather_indices(m, n) for m in range(1 << n)])
    phase = np.stack([pauli.omega_phase_factors(m, n) for m in range(1 << n)])
    wht_in = np.random.default_rng(5).standard_normal((4, 64))
    _save("blocks_n3.npz", locs=locs, gather=gather, phase=phase, xtx=pauli.xtx_diagonal_full(n),
          wht_in=wht_in, wht_out=pauli.walsh_hadamard_transform(wht_in),
          digit_rows=pauli.setting_digit_rows(0, 3**n, n))


def c1():
    ghz = simulate.StateDescriptor("ghz", 4)
    rec = simulate.exact_record(ghz)
    _save("c1_ghz4_exact.npz", **_run_reference(rec.counts, 4, rec.shots))
    rec = simulate.sample_counts(ghz, shots=1000, seed=SEED)
    _save("c1_ghz4_sampled.npz", **_run_reference(rec.counts, 4, 1000))


def small():
    cases = [
        ("small_random1.npz", simulate.StateDescriptor("random", 1, state_seed=3), 100, 11),
        ("small_random2.npz", simulate.StateDescriptor("random", 2, state_seed=4), 500, 12),
        ("small_random3.npz", simulate.StateDescriptor("random", 3, state_seed=5), 4096, 13),
        ("small_productz5.npz", simulate.StateDescriptor("productz", 5, bits=0b10110), None, None),
        ("small_maxmixed6.npz", simulate.StateDescriptor("maxmixed", 6), None, None),
        ("small_ghz2_sampled.npz", simulate.StateDescriptor("ghz", 2), 1000, 7),
    ]
    for name, state, shots, seed in cases:
        if shots is None:
            rec = simulate.exact_record(state)
        else:
            rec = simulate.sample_counts(state, shots=shots, seed=seed)
        _save(name, **_run_reference(rec.counts, state.n, rec.shots))


def c2():
    n = 8
    rho = O.dense_state("w", n)
    counts = _reference_sample_from_rho(rho, n, 1000, SEED)
    ours = O.sample_counts_from_theta(O.dense_to_theta(rho), n, 1000, SEED)
    assert np.array_equal(ours, counts), "oracle generator diverges from reference primitives at n=8"
    out = _run_reference(counts, n, 1000, with_step3=False)
    out["counts"] = counts.astype(np.uint16)
    _save("c2_w8.npz", **out)


def c3():
    n = 10
    rho = simulate._random_density(n, 8604)
    counts = _reference_sample_from_rho(rho, n, 1000, SEED)
    ours = O.sample_counts_from_theta(O.dense_to_theta(O.dense_state("random", n, seed=8604)), n, 1000, SEED)
    assert np.array_equal(ours, counts), "oracle generator diverges from reference primitives at n=10"
    rec = MeasurementRecord(n=n, shots=1000, counts=counts)
    theta = pipeline.step_one_least_squares(rec, workers=8)
    mu = pipeline.step_two_assemble(theta, workers=1)
    stride_t, stride_m = 97, 13
    _save("c3_random10.npz", n=n, shots=1000, seed=SEED, state_seed=8604,
          counts_sha256=np.array(hashlib.sha256(counts.astype(np.int64).tobytes()).hexdigest()),
          theta_stride=stride_t, theta_sample=theta[::stride_t], theta_norm=np.linalg.norm(theta),
          mu_stride=stride_m, mu_sample=mu.ravel()[::stride_m], mu_norm=np.linalg.norm(mu),
          mu_diag=np.diag(mu).copy())


def validate_messages():
    msgs = {}
    rng = np.random.default_rng(20240811)
    counts = rng.multinomial(50, np.full(4, 0.25), size=9).astype(np.int64)
    counts[3, 0] += 1
    try:
        MeasurementRecord(n=2, shots=50, counts=counts).validate()
    except ValueError as exc:
        msgs["bad_row_sum"] = str(exc)
    bad = counts.copy()
    bad[3, 0] -= 1
    bad[5, 1] = -1
    try:
        MeasurementRecord(n=2, shots=50, counts=bad).validate()
    except ValueError as exc:
        msgs["negative"] = str(exc)
    try:
        MeasurementRecord(n=2, shots=50, counts=counts[:8]).validate()
    except ValueError as exc:
        msgs["shape"] = str(exc)
    try:
        MeasurementRecord(n=2, shots=50, counts=counts.astype(float)).validate()
    except ValueError as exc:
        msgs["dtype"] = str(exc)
    ok = counts.copy()
    ok[3, 0] -= 1
    _save("validate.npz", counts_bad_row=counts, counts_ok=ok, messages=np.array(json.dumps(msgs)))


def files():
    from pauli_lre import records, statefile

    d = os.path.join(HERE, "files")
    os.makedirs(d, exist_ok=True)
    st = simulate.parse_state("ghz", 2)
    rec = simulate.sample_counts(st, 50, seed=SEED)
    records.write_record(rec, os.path.join(d, "record_ghz2.txt"))
    st3 = simulate.parse_state("random:8604", 3)
    rec3 = simulate.sample_counts(st3, 200, seed=SEED)
    records.write_record(rec3, os.path.join(d, "record_random3.txt"))
    rho = pipeline.reconstruct(rec3, workers=1).rho
    statefile.write_state(os.path.join(d, "state_random3.plre"), rho)
    msgs = {}
    lines = open(os.path.join(d, "record_ghz2.txt")).read().splitlines()
    tmp = tempfile.mkdtemp()
    for name, L in record_perturbations(lines).items():
        path = os.path.join(tmp, name + ".txt")
        with open(path, "w") as fh:
            fh.write("\n".join(L) + ("\n" if L else ""))
        try:
            records.read_record(path)
            msgs["record:" + name] = None
        except records.RecordFormatError as exc:
            msgs["record:" + name] = str(exc)
    blob = open(os.path.join(d, "state_random3.plre"), "rb").read()
    for name, b in state_perturbations(blob).items():
        path = os.path.join(tmp, "state.plre")
        with open(path, "wb") as fh:
            fh.write(b)
        try:
            statefile.read_state(path)
            msgs["state:" + name] = None
        except ValueError as exc:
            msgs["state:" + name] = str(exc).replace(path, "<path>")
    with open(os.path.join(d, "messages.json"), "w") as fh:
        json.dump(msgs, fh, indent=1, sort_keys=True)
    print("wrote files/ (", ", ".join(sorted(os.listdir(d))), ")")


def metrics_cases():
    from pauli_lre import metrics

    out = {}
    reports = {}
    cases = [("ghz4", simulate.StateDescriptor("ghz", 4), 16 * 60, 31),
             ("maxmixed4", simulate.StateDescriptor("maxmixed", 4), 16 * 40, 32),
             ("productz3", simulate.StateDescriptor("productz", 3, bits=0b101), 8 * 50, 33)]
    for name, st, shots, seed in cases:
        rec = simulate.sample_counts(st, shots=shots, seed=seed)
        res = pipeline.reconstruct(rec, workers=1)
        d = 1 << st.n
        rep = metrics.evaluate_errors(st, res.rho, res.mu, n0=shots / d)
        out[f"{name}_mu"] = res.mu
        out[f"{name}_rho"] = res.rho
        reports[name] = json.loads(rep.to_json())
        reports[name]["shots"] = shots
    preds = {}
    for label, st in [("ghz3", simulate.StateDescriptor("ghz", 3)), ("productz2", simulate.StateDescriptor(
            "productz", 2, bits=2)), ("maxmixed4", simulate.StateDescriptor("maxmixed", 4)),
            ("random3", simulate.StateDescriptor("random", 3, state_seed=9)),
            ("random4", simulate.StateDescriptor("random", 4, state_seed=10))]:
        rho = simulate.dense_matrix(st)
        out[f"pred_{label}_rho"] = rho
        preds[label] = metrics.predicted_mse_dense(rho, 37.0)
    fids = {}
    for k, (a, b) in enumerate([(5, 6), (7, 8)]):
        ra = simulate.dense_matrix(simulate.StateDescriptor("random", 3, state_seed=a))
        rb = simulate.dense_matrix(simulate.StateDescriptor("random", 3, state_seed=b))
        out[f"fid{k}_a"], out[f"fid{k}_b"] = ra, rb
        fids[f"fid{k}"] = metrics.fidelity(ra, rb, method="general")
    lam = np.array([0.5, 0.3, 0.2, 0.0, -0.01, 0.01, 0.0, 0.0])
    fids["maxmixed_spectrum"] = metrics.fidelity_with_maxmixed(lam, 8)
    out["maxmixed_spectrum"] = lam
    _save("metrics.npz", reports=np.array(json.dumps(reports)), preds=np.array(json.dumps(preds)),
          fids=np.array(json.dumps(fids)), **out)


def exact_sources():
    """reconstruct() on ExactFrequencies sources (pipeline.py:42-59,224-249): the reference's
    own timing flow (bench.median_step_times) — random states n = 2..5 (non-dyadic, fp64
    frequencies), ghz and maxmixed at n = 3 (dyadic), and a plain duck-typed source."""
    cases = {}
    for kind, n, seed in [("random", 2, 11), ("random", 4, 0), ("random", 5, 7), ("ghz", 3, 0), ("maxmixed", 3, 0)]:
        st = simulate.StateDescriptor(kind, n, state_seed=seed)
        res = pipeline.reconstruct(pipeline.ExactFrequencies(st), workers=1)
        tag = f"{kind}{n}_{seed}"
        cases.update({f"{tag}_theta": res.theta, f"{tag}_mu": res.mu, f"{tag}_rho": res.rho,
                      f"{tag}_eigenvalues": res.eigenvalues,
                      f"{tag}_probs": simulate.probabilities_block(st, 0, 3**n)})
    # theta_to_probabilities / exact_probabilities on single settings
    st = simulate.StateDescriptor("random", 3, state_seed=5)
    theta = simulate.dense_to_theta(simulate.dense_matrix(st).astype(np.complex128))
    cases["random3_5_dense_theta"] = theta
    cases["random3_5_p_w7"] = simulate.theta_to_probabilities(theta, 7, 3)
    cases["ghz3_p_w5"] = simulate.exact_probabilities(simulate.StateDescriptor("ghz", 3), 5)
    _save("exact_sources.npz", **cases)


if __name__ == "__main__":
    todo = sys.argv[1:] or ["kat", "blocks", "c1", "small", "validate_messages", "c2", "c3", "files", "exact_sources",
                            "metrics_cases"]
    for name in todo:
        globals()[name]()
