"""Benchmark of the B200 LRE hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--n 14]

One "step" = one full LRE reconstruction (steps (i)+(ii): counts -> theta ->
mu) of the C5 workload: n=14 GHZ, 3^14 settings x 2^14 outcomes, 1000 shots
per setting (seed 1602), counts generated on the device as uint16.  Counts
(157 GB) are far larger than L2 (126 MB), so no L2 flush is needed between
steps.  `value` = seconds per reconstruction with counts resident in HBM
(CUDA events, max over ranks); `e2e` = the same reconstruction through the
public streaming API from pinned HOST counts (H2D inside the timed region)
with mu read back to the host.  `--impl reference` times the reference
algorithm's CPU port (oracle/, kind "port") on the host cores, one full
reconstruction measured in K pieces, with the real reference package timed
beside it at n = 4..12.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "14-qubit LRE reconstruction seconds at 1/2/4/8 B200; achieved HBM GB/s"
PAPER_STEPS_12_S = (2.78 + 0.08) * 3600.0  # PAPER.md:167,169 (GTX 780, steps i+ii at n=14)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(n: int, c: int) -> float:
    """B(n) = c*6^n (counts read once) + 32*4^n (theta w+r, mu w)."""
    return c * 6.0**n + 32.0 * 4.0**n


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.lines:  # region shorter than nvidia-smi's start-up: one query at its end
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                self.lines.extend(l.strip() for l in out.stdout.splitlines() if l.strip())
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference timings (measured, never extrapolated from a cost model)
# ---------------------------------------------------------------------------

def workload_name(args) -> str:
    """BASELINE.json config C5 (n = 14; other n are the parity configs C1-C4 shapes)."""
    return (f"C5: n={args.n} {args.state.upper()}, 3^{args.n} settings x 2^{args.n} outcomes, "
            f"{args.shots} shots/setting, seed {args.seed}, one reconstruction (steps i+ii) per step")


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def device_record_rows(state_kind: str, n: int, shots: int, seed: int, lo: int, hi: int, out=None, state_seed=0):
    """Rows [lo, hi) of the C-config record, drawn by the device generator (the same
    record the B200 arm reconstructs) and copied to host memory — input preparation
    only, outside every CPU timed region."""
    import torch

    if not torch.cuda.is_available():
        # CPU-only containers (the bench's own CPU tests): the oracle's GHZ sampler
        # (numpy Philox per setting, simulate.py:216-242) at small n
        from oracle import lre_oracle as O

        if state_kind != "ghz":
            raise RuntimeError(f"no GPU: only GHZ records can be drawn on the host, not {state_kind}")
        rows = O.sample_ghz_counts(n, shots, seed, lo, hi)
        if out is None:
            return rows
        out[: hi - lo].copy_(torch.from_numpy(rows.astype(np.uint16 if shots <= 65535 else np.int32)))
        return out[: hi - lo].numpy()

    import paper_1602_08604_b200 as lre
    from paper_1602_08604_b200.simulate import dense_to_theta, generate_counts_from_theta, generate_device_counts

    if state_kind == "random":
        # C3: the reference's Ginibre state _random_density(n, seed) (simulate.py:105-111),
        # beyond the StateDescriptor cap of n <= 8, sampled from its Pauli coefficients
        d = 1 << n
        rng = np.random.default_rng(state_seed)
        g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        rho = g @ g.conj().T
        rho /= np.trace(rho).real
        dev = generate_counts_from_theta(dense_to_theta(rho, as_tensor=True), n, shots, seed, lo, hi)
    else:
        st = lre.StateDescriptor(state_kind, n, state_seed=state_seed)
        dev = generate_device_counts(st, shots, seed=seed, w_begin=lo, w_end=hi)
    if out is None:
        return dev.cpu().numpy()
    out[: hi - lo].copy_(dev)
    del dev
    return out[: hi - lo].numpy()


# the parity configs of BASELINE.json timed on the CPU: (n, state, shots, state_seed)
PER_N = [(4, "ghz", 1000, 0), (8, "w", 1000, 0), (10, "random", 1000, 8604), (12, "ghz", 1000, 0)]


def _import_reference():
    """The unmodified reference package (pip-installed into baseline/_ref, numba cache in /tmp)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "pauli_lre")):
        return None, "baseline/_ref is not installed (python -m pip install --no-index --no-deps --target baseline/_ref <copy of /root/reference/pkg>)"
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "lre_numba_cache"))
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import pauli_lre.pipeline as P
        import pauli_lre.records as R
        return (P, R), None
    except Exception as exc:  # numba or numpy missing on the box
        return None, f"{type(exc).__name__}: {str(exc)[:120]}"


def reference_per_n(configs=PER_N, repeats: int = 3):
    """The real reference (pauli_lre.pipeline.step_one_least_squares with all host cores +
    step_two_assemble, workers=1, the faster setting for its numpy step ii) on the
    configs' records, with the reference's own methodology (bench.py:18-37): one
    discarded warm-up, median of `repeats`.  Returns a list of rows."""
    mods, why = _import_reference()
    threads = os.cpu_count() or 1
    rows = []
    for n, kind, shots, sseed in configs:
        counts = device_record_rows(kind, n, shots, 1602, 0, 3**n, state_seed=sseed)
        row = {"n": n, "state": kind, "shots": shots, "cores": threads}
        if mods is not None:
            P, R = mods
            rec = R.MeasurementRecord(n=n, shots=shots, counts=counts)
            rec.validate()
            t1s, t2s = [], []
            for rep in range(repeats + 1):
                a = time.perf_counter()
                theta = P.step_one_least_squares(rec, workers=threads)
                b = time.perf_counter()
                P.step_two_assemble(theta, workers=1)
                c = time.perf_counter()
                if rep:
                    t1s.append(b - a)
                    t2s.append(c - b)
            row.update(kind="reference", t_step1_s=statistics.median(t1s), t_step2_s=statistics.median(t2s))
            row["t_s"] = row["t_step1_s"] + row["t_step2_s"]
        else:
            row.update(kind="reference", unavailable=why)
        # the C port beside it (same records, same methodology)
        from oracle import c_oracle as C

        tp = []
        for rep in range(repeats + 1):
            a = time.perf_counter()
            theta = C.step_one(counts, n, shots, threads)
            mu = np.empty((1 << n, 1 << n), dtype=np.complex128)
            C.step_two_scatter(theta, n, 0, 1 << n, mu, threads)
            if rep:
                tp.append(time.perf_counter() - a)
        row["port_t_s"] = statistics.median(tp)
        rows.append(row)
    return rows


def port_tiled(n: int, shots: int, seed: int, state_kind: str, steps: int, warmup: int):
    """One full C5 reconstruction by the C port of the reference (oracle/lre_oracle.c:
    per-setting WHT + scatter into per-worker 4^n partials, ordered merge, Gram
    division; step (ii) per-mask complex WHT + XOR-diagonal scatter), measured in
    `steps` pieces: step k = step (i) over settings shard k (the partials persist
    across shards) and step (ii) over masks shard k; the merge + Gram division is
    part of the last step-(i) piece.  Nothing is extrapolated: the sum of the step
    times is the measured wall time of one complete reconstruction on all host
    cores.  The shard counts come from the device generator (untimed)."""
    import torch

    from oracle import c_oracle as C

    C.build()
    threads = os.cpu_count() or 1
    settings, d = 3**n, 1 << n
    bounds = [settings * k // steps for k in range(steps + 1)]
    mbounds = [d * k // steps for k in range(steps + 1)]
    width = max(b - a for a, b in zip(bounds[:-1], bounds[1:]))
    host = torch.empty((width, d), dtype=torch.uint16 if shots <= 65535 else torch.int32,
                       pin_memory=torch.cuda.is_available())
    # warm-up: the same code on a throw-away accumulator (thread pool, first touch of the shard buffer)
    rows = device_record_rows(state_kind, n, shots, seed, 0, min(settings, 64), out=host)
    for _ in range(max(1, warmup)):
        w = C.Step1Accumulator(n, shots, threads)
        w.add(rows, 0)
        w.close()
    acc = C.Step1Accumulator(n, shots, threads)
    t_i, t_ii = [], []
    for k in range(steps):
        rows = device_record_rows(state_kind, n, shots, seed, bounds[k], bounds[k + 1], out=host)
        a = time.perf_counter()
        acc.add(rows, bounds[k])
        t_i.append(time.perf_counter() - a)
    a = time.perf_counter()
    theta = acc.finish()
    t_merge = time.perf_counter() - a
    acc.close()
    del host
    mu = np.empty((d, d), dtype=np.complex128)
    for k in range(steps):
        a = time.perf_counter()
        C.step_two_scatter(theta, n, mbounds[k], mbounds[k + 1], mu, threads)
        t_ii.append(time.perf_counter() - a)
    per_step = [t_i[k] + t_ii[k] + (t_merge if k == steps - 1 else 0.0) for k in range(steps)]
    return {"per_step_s": per_step, "t_step1_s": sum(t_i) + t_merge, "t_step2_s": sum(t_ii), "t_merge_s": t_merge,
            "value": sum(per_step), "cores": threads, "theta_head": theta[:4].tolist()}


def cpu_baseline(n: int, shots: int, seed: int, state_kind: str, fraction: int = 16):
    """The b200 arm's reported CPU baseline: the C port on a bounded sample of the C5
    workload, plus the real reference at the small configs.  The sample is the first
    1/`fraction` of the settings (step i) and of the masks (step ii); the per-run
    fixed cost (zero-filling the workers' 4^n partials, the ordered merge and the
    Gram division, which a full run pays once) is timed separately, so value =
    fixed + (sample - fixed) x fraction.  The bench's reference arm measures the
    full reconstruction without any scaling."""
    from oracle import c_oracle as C

    C.build()
    threads = os.cpu_count() or 1
    settings, d = 3**n, 1 << n
    s_hi, m_hi = settings // fraction, d // fraction
    # fixed cost: a full-size accumulator fed one setting per worker
    rows = device_record_rows(state_kind, n, shots, seed, 0, threads)
    a = time.perf_counter()
    acc = C.Step1Accumulator(n, shots, threads)
    acc.add(rows, 0)
    acc.finish()
    acc.close()
    t_fixed = time.perf_counter() - a
    rows = device_record_rows(state_kind, n, shots, seed, 0, s_hi)
    a = time.perf_counter()
    acc = C.Step1Accumulator(n, shots, threads)
    acc.add(rows, 0)
    theta = acc.finish()
    acc.close()
    t1 = time.perf_counter() - a
    del rows
    mu = np.empty((d, d), dtype=np.complex128)
    a = time.perf_counter()
    C.step_two_scatter(theta, n, 0, m_hi, mu, threads)
    t2 = time.perf_counter() - a
    del mu, theta
    per_n = reference_per_n(PER_N[:3], repeats=1)
    value = t_fixed + max(0.0, t1 - t_fixed) * fraction + t2 * fraction
    return {"value": value, "unit": "s", "cores": threads, "kind": "port",
            "sample": (f"n={n} {state_kind.upper()} C5 record: C port step (i) on settings [0, {s_hi}) of {settings} "
                       f"({t1:.2f} s, of which {t_fixed:.2f} s is the per-run fixed cost: zeroing the {threads} worker "
                       f"partials, merge, Gram division) and step (ii) on masks [0, {m_hi}) of {d} ({t2:.2f} s); "
                       f"value = fixed + variable x {fraction}. The full, unscaled reconstruction is the "
                       f"--impl reference line."),
            "cpu_model": cpu_model(), "per_n": per_n}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def traffic_from_profiles(n: int):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(str(n))
    except Exception:
        return None


def host_record(counts, chunk_rows, torch):
    """Copy the device record to HOST memory in slabs of whole chunks: pinned
    when the host allows it (a 157 GB single pinned allocation is refused on
    these boxes), otherwise pageable.  Returns ([(lo, hi, tensor)], pinned)."""
    rows = counts.shape[0]
    slab_rows = chunk_rows * 4
    for pin in (True, False):
        slabs = []
        try:
            for lo in range(0, rows, slab_rows):
                hi = min(rows, lo + slab_rows)
                t = torch.empty((hi - lo, counts.shape[1]), dtype=counts.dtype, pin_memory=pin)
                t.copy_(counts[lo:hi])
                slabs.append((lo, hi, t))
            return slabs, pin
        except Exception:
            del slabs
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    raise MemoryError("could not stage the record in host memory")


class MuPipe:
    """Step (ii) into one of two device buffers and its D2H on a side stream:
    step k's mu copy-out overlaps step k+1's H2D (PCIe is full duplex).
    Every step's result still reaches pinned host memory inside the timed
    region (drain() before the closing event)."""

    def __init__(self, plan, mu_host, torch):
        from paper_1602_08604_b200 import _lib

        self.lib, self.plan, self.torch = _lib, plan, torch
        d = 1 << plan.n
        self.dev = [torch.empty((d, d), dtype=torch.complex128, device=plan.device) for _ in range(2)]
        self.host = [mu_host, torch.empty_like(mu_host, pin_memory=True)]
        self.d2h = torch.cuda.Stream(plan.device)
        self.done = [torch.cuda.Event() for _ in range(2)]
        self.k = 0

    def assemble_and_copy(self, comp):
        b = self.k % 2
        comp.wait_event(self.done[b])  # the previous copy-out of this buffer has finished
        d = 1 << self.plan.n
        self.lib.call("lre_assemble", self.plan.theta.data_ptr(), self.plan.layout, self.plan.n, 0, d,
                      self.dev[b].data_ptr(), comp.cuda_stream)
        ready = self.torch.cuda.Event()
        ready.record(comp)
        self.d2h.wait_event(ready)
        with self.torch.cuda.stream(self.d2h):
            self.host[b].copy_(self.dev[b], non_blocking=True)
            self.done[b].record(self.d2h)
        self.k += 1

    def drain(self, comp):
        for e in self.done:
            comp.wait_event(e)


def e2e_host(plan, slabs, n, mu_host, chunk_rows, steps, warmup, torch, lre_dtype):
    """Public streaming API from HOST counts: H2D chunks (copy stream)
    overlapped with the first pass (lre_step1_stage), then the remaining
    passes (lre_step1_finish), assembly (lre_assemble) and the D2H of mu, all
    inside the timed region."""
    dev = plan.device
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    width = slabs[0][2].shape[1]
    bufs = [torch.empty((chunk_rows, width), dtype=slabs[0][2].dtype, device=dev) for _ in range(2)]
    ev_copy = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    pipe = MuPipe(plan, mu_host, torch)

    def one():
        k = 0
        for s_lo, s_hi, slab in slabs:
            for lo in range(s_lo, s_hi, chunk_rows):
                hi = min(s_hi, lo + chunk_rows)
                b = k % 2
                copy.wait_event(ev_used[b])
                with torch.cuda.stream(copy):
                    bufs[b][: hi - lo].copy_(slab[lo - s_lo:hi - s_lo], non_blocking=True)
                    ev_copy[b].record(copy)
                comp.wait_event(ev_copy[b])
                plan.stage(bufs[b][: hi - lo], lre_dtype, lo, hi, comp, validate=True)
                ev_used[b].record(comp)
                k += 1
        plan.finish(comp)
        pipe.assemble_and_copy(comp)

    for _ in range(warmup):
        one()
    pipe.drain(comp)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(steps):
        one()
    pipe.drain(comp)
    e1.record(comp)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    plan.verify()  # the chunks were validated on the device inside the timed region; raise if any row was bad
    del bufs
    return e0.elapsed_time(e1) / 1e3 / steps, wall / steps


def e2e_outcomes(plan, st, shots, seed, n, mu_host, chunk_rows, steps, torch):
    """Same public streaming path, but the host record is an outcome list
    (2 B per shot, OutcomeRecord): each chunk's outcomes go H2D and are
    histogrammed into dense counts on the device (lre_counts_from_outcomes)
    before lre_step1_stage.  Returns (device s/step, wall s/step, h2d bytes,
    pinned) or raises."""
    from paper_1602_08604_b200.simulate import generate_device_outcomes

    dev = plan.device
    rows = 3**n
    host = []
    pinned = True
    for lo in range(0, rows, chunk_rows):
        hi = min(rows, lo + chunk_rows)
        o = generate_device_outcomes(st, shots, seed=seed, w_begin=lo, w_end=hi, device=dev)
        try:
            h = torch.empty(tuple(o.shape), dtype=torch.uint16, pin_memory=pinned)
        except Exception:
            pinned = False
            h = torch.empty(tuple(o.shape), dtype=torch.uint16)
        h.copy_(o)
        host.append((lo, hi, h))
        del o
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    bufs = [torch.empty((chunk_rows, shots), dtype=torch.uint16, device=dev) for _ in range(2)]
    ev_copy = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    pipe = MuPipe(plan, mu_host, torch)

    def one():
        for k, (lo, hi, h) in enumerate(host):
            b = k % 2
            copy.wait_event(ev_used[b])
            with torch.cuda.stream(copy):
                bufs[b][: hi - lo].copy_(h, non_blocking=True)
                ev_copy[b].record(copy)
            comp.wait_event(ev_copy[b])
            plan.stage_outcomes(bufs[b][: hi - lo], lo, hi, comp, validate=True)
            ev_used[b].record(comp)
        plan.finish(comp)
        pipe.assemble_and_copy(comp)

    one()
    pipe.drain(comp)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(steps):
        one()
    pipe.drain(comp)
    e1.record(comp)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    plan.verify()
    h2d = sum(h.numel() * 2 for _, _, h in host)
    del bufs, host
    plan._dense = None
    return e0.elapsed_time(e1) / 1e3 / steps, wall / steps, h2d, pinned


def run_b200(args):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.gpus > 1 or args.force_dist:
        return run_dist(args, rank, world, local)

    import paper_1602_08604_b200 as lre
    from paper_1602_08604_b200 import _lib
    from paper_1602_08604_b200.simulate import generate_device_counts

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, shots, seed = args.n, args.shots, args.seed
    st = lre.StateDescriptor(args.state, n)
    peak, peak_kind = peaks()

    counts = generate_device_counts(st, shots, seed=seed, device=dev)
    rec = lre.DeviceRecord(n=n, shots=shots, counts=counts, seed=seed, state=st.label())
    rec.validate()
    c = counts.element_size()
    ctype = str(counts.dtype).replace("torch.", "")
    lre_dtype = rec.lre_dtype

    base = None
    if not args.no_cpu_baseline:
        try:
            base = cpu_baseline(n, shots, seed, args.state)
        except Exception as exc:
            base = {"value": None, "error": f"{type(exc).__name__}: {str(exc)[:160]}"}

    plan = lre.LREPlan(n, shots, dev)
    s = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 3)):
        plan.run(counts, lre_dtype, s)
    torch.cuda.synchronize()

    # --- timed region: K full reconstructions, counts resident in HBM ---
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        evs[0].record(s)
        for i in range(args.steps):
            plan.run(counts, lre_dtype, s)
            evs[i + 1].record(s)
        torch.cuda.synchronize()
        time.sleep(0.25)
    launches = _lib.launch_count() - launches0
    per = [evs[i].elapsed_time(evs[i + 1]) / 1e3 for i in range(args.steps)]
    t_step = statistics.median(per)

    # --- per-kernel timing of the dominant kernel (fold pass 1) and the rest ---
    k = max(3, min(args.steps, 10))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s)
    for _ in range(k):
        plan.stage(counts, lre_dtype, 0, 3**n, s)
    e[1].record(s)
    for _ in range(k):
        plan.finish(s)
    e[2].record(s)
    for _ in range(k):
        plan.step2(s)
    e[3].record(s)
    torch.cuda.synchronize()
    t_pass1 = e[0].elapsed_time(e[1]) / 1e3 / k
    t_rest1 = e[1].elapsed_time(e[2]) / 1e3 / k
    t_asm = e[2].elapsed_time(e[3]) / 1e3 / k
    # the repeated finish() above re-reads ping-ponged intermediates: restore a
    # valid theta / mu (used by step iii when the e2e runs are skipped)
    plan.run(counts, lre_dtype, s)
    pass1_bytes = c * 6.0**n  # algorithmic: every count read once (the Y1 write is not counted)
    q1 = min(n, 7)
    tma = counts.dtype == torch.uint16 and shots <= 1213 and n >= 6 and os.environ.get("LRE_P1") == "tma"
    variant = os.environ.get("LRE_P1", "ldg")
    p1_name = (f"tile_tma_kernel<{q1}> (pass 1, TMA ring)" if tma else
               f"tile_ring_kernel<{q1}> (pass 1, cp.async ring)" if variant == "ring" and counts.dtype == torch.uint16
               else f"tile_pass_kernel<{q1}> (pass 1, LDG)") if n >= 6 else "vfold_kernel (pass 1)"
    achieved = pass1_bytes / t_pass1 / 1e9
    traffic = traffic_from_profiles(n)
    whole = algorithmic_bytes(n, c) / t_step / 1e9

    # --- e2e through the public streaming API with host buffers ---
    e2e = None
    if not args.no_e2e:
        host_bytes = counts.numel() * c
        avail = _mem_available()
        if avail is None or avail > host_bytes + (16 << 30):
            try:
                q = int(_lib.load().lre_shard_quantum(n))
                chunk = max(1, (2 << 30) // (counts.shape[1] * c))
                chunk = max(q, chunk // q * q)
                slabs, pinned = host_record(counts, chunk, torch)
                mu_host = torch.empty(tuple(plan.mu.shape), dtype=plan.mu.dtype, pin_memory=True)
                del rec
                counts = None
                torch.cuda.empty_cache()
                ksteps = max(1, min(args.steps, args.e2e_steps))
                t_e2e, wall_e2e = e2e_host(plan, slabs, n, mu_host, chunk, ksteps, 1, torch, lre_dtype)
                e2e = {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": int(host_bytes),
                       "d2h_bytes_per_step": int(mu_host.numel() * mu_host.element_size()),
                       "wall_s_per_step": wall_e2e, "host_memory": "pinned" if pinned else "pageable",
                       "steps": ksteps,
                       "api": "LREPlan.stage(validate=True)/finish + lre_assemble (lre_validate_counts + "
                              "lre_step1_stage, lre_step1_finish, lre_assemble) from host counts",
                       "pipelining": "mu of step k is copied out on a side stream while step k+1's counts go in "
                                     "(double-buffered device mu); every step's H2D and D2H complete inside the "
                                     "timed region"}
                del slabs, mu_host
            except Exception as exc:  # keep the device-side line even if the host side fails
                e2e = {"value": None, "unit": "s", "error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        else:
            e2e = {"value": None, "unit": "s", "skipped": f"host RAM {avail >> 30} GiB < record {host_bytes >> 30} GiB"}
        # secondary: the same record as raw-shot outcome lists (2 B per shot)
        try:
            rec = counts = None
            torch.cuda.empty_cache()
            q = int(_lib.load().lre_shard_quantum(n))
            chunk = max(q, max(1, (2 << 30) // ((1 << n) * c)) // q * q)
            mu_host = torch.empty(tuple(plan.mu.shape), dtype=plan.mu.dtype, pin_memory=True)
            ksteps = max(1, min(args.steps, args.e2e_steps))
            t_o, wall_o, h2d_o, pin_o = e2e_outcomes(plan, st, shots, seed, n, mu_host, chunk, ksteps, torch)
            e2e_out = {"value": t_o, "unit": "s", "h2d_bytes_per_step": int(h2d_o),
                       "d2h_bytes_per_step": int(mu_host.numel() * mu_host.element_size()),
                       "wall_s_per_step": wall_o, "host_memory": "pinned" if pin_o else "pageable", "steps": ksteps,
                       "api": "OutcomeRecord chunks -> LREPlan.stage_outcomes (lre_counts_from_outcomes + "
                              "lre_step1_stage) -> finish -> step2",
                       "same_record": "identical counts (same Philox stream) as the dense record"}
            del mu_host
        except Exception as exc:
            e2e_out = {"value": None, "unit": "s", "error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        if e2e is not None:
            e2e["outcome_record"] = e2e_out

    # --- step (iii), adjacent to the hot path and timed separately (north star):
    # Hermitian eigensolve (cuSOLVER through torch.linalg.eigh) + simplex projection
    step3 = None
    if not args.no_step3:
        rec = counts = None  # free the record (157 GB at n = 14) for the eigensolver's workspace
        torch.cuda.empty_cache()
        try:
            plan.step2(s)  # mu of the last reconstruction (the e2e runs assemble into their own buffers)
            warm = torch.eye(64, dtype=torch.complex128, device=dev) / 64  # cuSOLVER handle + module load
            lre.step_three_project(warm)
            torch.cuda.synchronize()
            e3 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e3[0].record(s)
            rho, evals = lre.step_three_project(plan.mu)
            e3[1].record(s)
            torch.cuda.synchronize()
            step3 = {"value": e3[0].elapsed_time(e3[1]) / 1e3, "unit": "s", "what": "step_three_project(mu): "
                     "Hermiticity/trace checks + torch.linalg.eigh (cuSOLVER, library code) + simplex projection + "
                     "V diag(lambda) V^H; not part of value", "projected": rho is not plan.mu,
                     }
            del rho, evals
        except Exception as exc:
            step3 = {"value": None, "unit": "s", "error": f"{type(exc).__name__}: {str(exc)[:160]}"}

    line = {
        "metric": METRIC,
        "value": t_step,
        "unit": "s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": t_step * 1e3,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": t_step / PAPER_STEPS_12_S if n == 14 else None,
        "dtype": "i32/i64 exact integer folds, f64 theta/mu",
        "data": "synthetic: device generator, Philox4x32-10 per (seed, setting), multinomial shots",
        "config": {"workload": workload_name(args), "n": n, "state": args.state, "shots": shots,
                   "counts": f"{ctype}, resident in HBM", "count_bytes": c,
                   "l2": "inputs larger than L2 (counts >> 126 MB); no flush",
                   "passes": plan.passes,
                   "vs_baseline_ref": "paper GTX 780 steps (i)+(ii) at n=14, 2.86 h (PAPER.md:167,169)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": p1_name,
                     "algorithmic_bytes_per_launch": pass1_bytes, "avg_launch_s": t_pass1, "peak_kind": peak_kind},
        "whole_path": {"algorithmic_bytes": algorithmic_bytes(n, c), "achieved_GBps": whole, "frac": whole / peak,
                       "t_pass1_s": t_pass1, "t_pass2_s": t_rest1, "t_assemble_s": t_asm},
        "cpu_baseline": base,
        "e2e": e2e,
        "step3": step3,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line))


def run_dist(args, rank: int, world: int, local: int):
    """bench.py --gpus N under torchrun (one process per GPU, NCCL).

    Settings shard over ranks (3^7-aligned ranges, counts generated in place
    by the (seed, setting)-keyed generator); each rank folds its shard into
    int64 numerators (mask-major), one reduce_scatter over NCCL leaves rank g
    the masks [g 2^n/P, (g+1) 2^n/P), which it finalises and assembles into its
    column-block slice of mu (paper_1602_08604_b200/distributed.py).  `value`
    = median over steps of the max over ranks of the per-step device time.
    """
    import torch
    import torch.distributed as dist

    import paper_1602_08604_b200 as lre
    from paper_1602_08604_b200 import _lib, distributed as D
    from paper_1602_08604_b200.simulate import generate_device_counts

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    # keep stdout to the one JSON line: native libraries (the NCCL version banner) write
    # to fd 1 directly, so fd 1 points at stderr until the line is printed
    sys.stdout.flush()
    stdout_fd = os.dup(1)
    os.dup2(2, 1)
    dist.init_process_group("nccl", device_id=dev)
    n, shots, seed = args.n, args.shots, args.seed
    q = int(_lib.load().lre_shard_quantum(n))
    lo, hi = D.shard_ranges(n, world, q)[rank]
    st = lre.StateDescriptor(args.state, n)
    counts = generate_device_counts(st, shots, seed=seed, w_begin=lo, w_end=hi, device=dev)
    rec = lre.DeviceRecord(n=n, shots=shots, counts=counts, w_begin=lo, seed=seed, state=st.label()).validate()
    comp = D.DeviceCompute(n, shots, lo, hi, world, rank, dev)
    runner = D.ShardedLRE(comp)
    s = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 3)):
        runner.step(counts, rec.lre_dtype)
    torch.cuda.synchronize()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().tolist()

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        evs[0].record(s)
        for i in range(args.steps):
            runner.step(counts, rec.lre_dtype)
            evs[i + 1].record(s)
        torch.cuda.synchronize()
        dist.barrier()
    launches = _lib.launch_count() - l0
    per = max_over_ranks([evs[i].elapsed_time(evs[i + 1]) / 1e3 for i in range(args.steps)])
    t_step = statistics.median(per)

    # step (i) of the shard alone (the dominant kernel sequence), max over ranks
    k = max(3, min(args.steps, 10))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(s)
    for _ in range(k):
        comp.partial_numerators(counts, rec.lre_dtype)
    e[1].record(s)
    torch.cuda.synchronize()
    t_s1 = max_over_ranks([e[0].elapsed_time(e[1]) / 1e3 / k])[0]
    c = counts.element_size()
    shard_bytes = float(counts.numel() * c)
    shard_max = float(max(h - l for l, h in D.shard_ranges(n, world, q)) * (1 << n) * c)
    peak, peak_kind = peaks()

    # e2e: host-resident shard -> H2D -> step -> D2H of this rank's mu slice
    e2e = None
    if not args.no_e2e:
        try:
            host = torch.empty(tuple(counts.shape), dtype=counts.dtype, pin_memory=True)
            host.copy_(counts)
            mu_host = torch.empty(tuple(comp.mu.shape), dtype=comp.mu.dtype, pin_memory=True)
            dcounts = counts
            ksteps = max(1, min(args.steps, args.e2e_steps))
            for i in range(ksteps + 1):
                if i == 1:
                    dist.barrier()
                    torch.cuda.synchronize()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                dcounts.copy_(host, non_blocking=True)
                runner.step(dcounts, rec.lre_dtype)
                mu_host.copy_(comp.mu, non_blocking=True)
            e1.record(s)
            torch.cuda.synchronize()
            t_e2e = max_over_ranks([e0.elapsed_time(e1) / 1e3 / ksteps])[0]
            h2d = int(max_over_ranks([float(host.numel() * c)])[0])
            e2e = {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": int(shard_bytes * world),
                   "d2h_bytes_per_step": int(mu_host.numel() * mu_host.element_size() * world),
                   "h2d_bytes_per_rank_max": h2d, "host_memory": "pinned",
                   "api": "ShardedLRE.step (lre_step1 NUM_I64 + NCCL reduce_scatter + lre_finalize + lre_assemble) "
                          "on counts copied from host each step"}
            del host, mu_host
        except Exception as exc:
            e2e = {"value": None, "unit": "s", "error": f"{type(exc).__name__}: {str(exc)[:200]}"}

    sys.stdout.flush()
    os.dup2(stdout_fd, 1)
    os.close(stdout_fd)
    if rank == 0:
        b = algorithmic_bytes(n, c)
        print(json.dumps({
            "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_step * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": t_step / PAPER_STEPS_12_S if n == 14 else None,
            "dtype": "i32/i64 exact integer folds, f64 theta/mu",
            "data": "synthetic: device generator per shard, Philox4x32-10 per (seed, setting), multinomial shots",
            "config": {"workload": workload_name(args), "n": n, "state": args.state, "shots": shots,
                       "counts": f"{str(counts.dtype).replace('torch.', '')}, shard resident in HBM",
                       "l2": "inputs larger than L2; no flush",
                       "parallelism": f"settings sharded /{world} (3^{min(n, 7)}-aligned), int64 numerator "
                                      f"reduce_scatter by X-mask over NCCL, mu column blocks /{world}"},
            "roofline": {"bound": "hbm", "achieved": shard_max / t_s1 / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": shard_max / t_s1 / 1e9 / peak, "traffic": None,
                         "kernel": "step (i) of the largest shard (tile pass + vector passes, int64 mask-major out)",
                         "algorithmic_bytes_per_launch": shard_max, "avg_launch_s": t_s1, "peak_kind": peak_kind},
            "whole_path": {"algorithmic_bytes": b, "achieved_GBps": b / t_step / 1e9,
                           "frac_of_world_peak": b / t_step / 1e9 / (peak * world)},
            "cpu_baseline": None,
            "e2e": e2e,
            "exchange": {"collective": "reduce_scatter_tensor (NCCL), int64 numerators",
                         "chunks": comp.K, "nccl_bytes_per_rank": runner.nccl_bytes,
                         "overlap": "chunk k finalised + assembled (lre_finalize, lre_assemble_slab) while chunk k+1 "
                                    "transfers on a side stream" if comp.K > 1 else "none (one chunk)",
                         "measured_on_hardware": world > 1},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }), flush=True)
    dist.destroy_process_group()


def _mem_available():
    try:
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except Exception:
        return None
    return None


# ---------------------------------------------------------------------------
# reference arm (CPU port of the reference algorithm)
# ---------------------------------------------------------------------------

def run_reference(args):
    """`bench.py --impl reference`: the reference's CPU LRE on this box's host cores, same
    metric / unit / config as the B200 arm.  The K timed steps are K consecutive pieces
    of ONE full C5 reconstruction by the C port of the reference (port_tiled; the
    reference is Python + numba and compiles to nothing here, so per the tier rules
    the port is the arm), value = their sum = seconds per reconstruction, measured.
    The real reference package (pauli_lre from baseline/_ref, numba) is timed beside
    it on the parity configs n = 4, 8, 10, 12 (cpu_baseline.per_n).  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    if torch.cuda.is_available():
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    n, shots, seed = args.n, args.shots, args.seed
    t_start = time.perf_counter()
    tiled = port_tiled(n, shots, seed, args.state, max(1, args.steps), args.warmup)
    per_n = reference_per_n() if not args.no_per_n and torch.cuda.is_available() else []
    v = tiled["value"]
    k = len(tiled["per_step_s"])
    line = {
        "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": k, "warmup": args.warmup,
        "ms_per_step": v / k * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: the B200 arm's C5 record (device generator, Philox4x32-10 per "
                                "(seed, setting)), copied to host memory shard by shard outside the timed region",
        "config": {"workload": workload_name(args), "n": n, "state": args.state, "shots": shots,
                   "counts": "uint16 host shards (pinned), one per step"},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "s", "cores": tiled["cores"], "kind": "port",
                         "sample": (f"the whole workload: step k of {k} = step (i) over settings shard k (worker "
                                    f"partials persist across shards) + step (ii) over masks shard k; merge + Gram "
                                    f"division in the last step; t_step1 {tiled['t_step1_s']:.2f} s, t_step2 "
                                    f"{tiled['t_step2_s']:.2f} s; C port of pipeline.py:62-161, all host threads"),
                         "cpu_model": cpu_model(), "per_step_s": tiled["per_step_s"], "per_n": per_n},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_start,
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    # --qubits: torchrun's own parser mistakes a bare "--n" for its --nnodes/--nproc-per-node
    ap.add_argument("--qubits", "--n", dest="n", type=int, default=14)
    ap.add_argument("--state", default="ghz", choices=("ghz", "w", "maxmixed"))
    ap.add_argument("--shots", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=1602)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-step3", action="store_true", help="skip the separately timed step (iii) eigen-projection")
    ap.add_argument("--force-dist", action="store_true", help="run the torch.distributed path even at world size 1")
    ap.add_argument("--no-per-n", action="store_true", help="reference arm: skip the per-n table of the real reference")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
