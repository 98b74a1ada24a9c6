"""Benchmark of the B200 state-vector engine on BASELINE.json's configs.

Default workload (N=1): config 2 -- 28-qubit random brickwork, depth 20
(830 gates: 560 Haar-random U3 + 270 CNOT), complex128, from |0...0>.
One step = evolve(prepare("0"*28), circuit) on resident HBM state.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
                    [--extra ucc12,expect30,ucc32,fused30]

Prints ONE JSON line (rank 0).  value = amplitude-updates/s (sum over the 830
gates of 2^n, per second, whole job); e2e = the same metric through the public
backend API with host buffers (gate arrays in, full amplitude vector out to
pinned host memory) inside the timed region.  roofline = the dominant kernel
(qsv_pass, the NVRTC-specialised tile pass): FP64-bound, achieved FP64 TFLOP/s
of the instructions it executes (ncu counts) over the step time, vs the
MEASURED DFMA peak (tools/peaks_probe.cu), with the HBM view beside it.
cpu_baseline = the reference (oracle/_ref: vqekit + Cython kernels) on all
host cores, a gate sample with the circuit's U3:CNOT mix.  --extra adds
configs 1 / 3 / 4, the 30 q fused-gate roofline and the 33 q weak-scaling base.

For N > 1 (torchrun, one rank per GPU) the line measures the SHARDED engine
(distributed.py) on the config-5 family: n = 33 + log2(N) qubits, 2^33
amplitudes (128 GiB) per GPU (weak scaling; config 5 itself at N = 8).
Relayouts swap chunks in place over peer memory (CUDA IPC mapping of the
partner's shard + swap kernel, each rank one half of a pair); NCCL carries the
plumbing (barriers, handle and partial gathers).  value = total
amplitude-updates/s of the whole job.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_QUBITS = 28
LAYERS = 20
SEED = 0
# dram__bytes_read.sum + dram__bytes_write.sum of one config-2 pass (ncu --set full, r01)
TRAFFIC_PER_LAUNCH = 4.295412e9 + 4.238421e9


def load_fp64_peak() -> tuple[float, str]:
    """Measured DFMA/s of this B200 (tools/peaks_probe.cu -> profiles/r02_peaks_probe.json);
    fallback: 148 SMs x 64 DFMA/clk x 1.965 GHz."""
    try:
        with open(os.path.join(REPO, "profiles", "r02_peaks_probe.json")) as fh:
            return float(json.load(fh)["dfma_per_s"]), "measured (tools/peaks_probe.cu)"
    except Exception:
        return 148 * 64 * 1.965e9, "nominal 148 x 64 DFMA/clk x 1.965 GHz"


def load_fp64_counts() -> dict | None:
    """FP64-pipe instructions (thread level) the specialised passes of one
    config-2 step execute, from ncu (smsp__sass_thread_inst_executed_op_
    {dfma,dmul,dadd}_pred_on.sum over the step's launches): a property of the
    compiled plan, so it is measured once per build and timed live here."""
    try:
        with open(os.path.join(REPO, "profiles", "r02_fp64_counts.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


def fp64_roofline(t_step: float, passes: int, nominal_dfma: int, hbm: dict) -> dict:
    """The config-2 step is FP64-bound: achieved FP64 TFLOP/s (DFMA = 2 flop,
    DMUL / DADD = 1) of the instructions actually executed, against the
    measured DFMA peak; the HBM view rides along."""
    peak_dfma, src = load_fp64_peak()
    counts = load_fp64_counts()
    out = {"bound": "fp64", "unit": "TFLOP/s", "peak": 2 * peak_dfma / 1e12, "peak_source": src,
           "kernel": "qsv_pass (NVRTC-specialised tile pass)", "traffic": hbm["traffic"],
           "nominal_dfma_per_step": nominal_dfma,
           "nominal_note": "8 DFMA per amplitude per dense 2x2 complex gate (SURVEY 8(d)); the "
                           "kernels issue fewer (normalised U3 forms: 6 per amplitude, 4 for "
                           "phase-deferred shears)",
           "hbm": hbm}
    norm_now = os.environ.get("QSV_U3_NORM", "1") != "0"
    cz_now = os.environ.get("QSV_CZ_DEFER", "1") != "0"
    if (counts and counts.get("passes") == passes and bool(counts.get("u3_norm")) == norm_now
            and bool(counts.get("cz_defer")) == cz_now):
        flops = 2 * counts["dfma"] + counts["dmul"] + counts["dadd"]
        inst = counts["dfma"] + counts["dmul"] + counts["dadd"]
        out.update({"achieved": flops / t_step / 1e12, "frac": flops / t_step / 1e12 / out["peak"],
                    "fp64_pipe_frac": inst / t_step / peak_dfma,
                    "fp64_inst_per_step": counts, "counts_source": counts.get("source")})
    else:
        out.update({"achieved": None, "frac": None,
                    "counts_source": "missing or stale profiles/r02_fp64_counts.json"})
    return out


def load_peaks() -> tuple[float, str]:
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# reference / CPU baseline
# ---------------------------------------------------------------------------


def _reference_modules():
    ref = os.path.join(REPO, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "vqekit")):
        sys.path.insert(0, ref)
        try:
            import vqekit.circuit as RC
            import vqekit.kernels as RK
            import vqekit.statevector as RSV
            if RK.IMPLEMENTATION == "cython":
                return "reference", RC, RSV
        except Exception:
            pass
    return "port", None, None


def host_info(workers: int | None = None) -> dict:
    """Cores, CPU model, RAM (and W) recorded beside every CPU number
    (BASELINE.md 3)."""
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    ram = None
    try:
        import psutil

        ram = round(psutil.virtual_memory().total / 2**30, 1)
    except Exception:
        pass
    d = {"os_cpu_count": os.cpu_count(), "cpu_model": model, "ram_gib": ram}
    if workers is not None:
        d["workers"] = workers
    return d


def _avail_ram() -> int:
    try:
        import psutil

        return int(psutil.virtual_memory().available)
    except Exception:
        return 16 << 30


def ref_sample_gates(circuit, step: int, worker: int):
    """Gates of one reference-arm step: 2 U3 + 1 CNOT (the circuit's 560:270
    mix), taken at positions that rotate with the step and the worker so the
    sample walks the whole circuit."""
    u3 = [g for g in circuit.gates if g.kind == "U3"]
    cx = [g for g in circuit.gates if g.kind == "CNOT"]
    k = 37 * worker + 3 * step
    return [u3[(2 * k) % len(u3)], u3[(2 * k + 1) % len(u3)], cx[k % len(cx)]]


def _ref_gate_worker(wid, n, steps, barrier, out_q):
    """One reference worker: its own 2^n state; each step applies the sample
    gates with the reference's own per-gate routine (statevector._apply_gate,
    statevector.py:57-62 -- the body of evolve's loop, Cython kernels)."""
    import numpy as np

    from paper_2208_10978_b200 import workloads as W

    _, RC, RSV = _reference_modules()
    circ = W.brickwork(n, LAYERS, SEED)
    amps = np.zeros(1 << n, dtype=np.complex128)
    amps[0] = 1.0
    times = []
    for k in range(steps):
        gates = ref_sample_gates(circ, k, wid)
        barrier.wait()
        t0 = time.perf_counter()
        for g in gates:
            RSV._apply_gate(amps, g.kind, tuple(g.qubits), tuple(p.value for p in g.params))
        t1 = time.perf_counter()
        barrier.wait()
        times.append((t0, t1))
    out_q.put((wid, times))


def reference_gate_throughput(n: int, steps: int, warmup: int, workers: int | None = None) -> dict:
    """The reference's own CPU gate loop on the config-2 circuit family, with
    all the host cores it can use: the reference evolve is single-threaded
    (no prange in _cykernels.pyx), so W independent worker processes each
    run the sample on their own 2^n state, concurrently (barrier per step).
    Step time = latest finish - earliest start over the workers."""
    import multiprocessing as mp

    kind, _, _ = _reference_modules()
    if kind != "reference":
        raise RuntimeError("oracle/_ref (the reference build) is missing")
    if workers is None:
        by_ram = max(1, (_avail_ram() - (8 << 30)) // (16 << n))  # 1 state + headroom each
        workers = int(max(1, min(os.cpu_count() or 1, by_ram)))
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(workers)
    q = ctx.Queue()
    total = warmup + steps
    procs = [ctx.Process(target=_ref_gate_worker, args=(w, n, total, barrier, q)) for w in range(workers)]
    for p in procs:
        p.start()
    res = dict(q.get() for _ in procs)
    for p in procs:
        p.join()
    per_step = []
    for k in range(warmup, total):
        t0 = min(res[w][k][0] for w in res)
        t1 = max(res[w][k][1] for w in res)
        per_step.append(t1 - t0)
    t = sum(per_step) / len(per_step)
    value = workers * 3 * (1 << n) / t
    return {"value": value, "unit": "amplitude-updates/s", "cores": workers, "kind": "reference",
            "seconds_per_step": t,
            "sample": (f"{workers} worker processes x (2 U3 + 1 CNOT of the {n}q depth-{LAYERS} "
                       f"brickwork, rotating through all 830 gates) per step via "
                       f"vqekit.statevector._apply_gate (oracle/_ref, Cython kernels; evolve's "
                       f"single 16*2^n-byte state copy per circuit excluded)"),
            "host": host_info(workers)}


def reference_ucc12(evals: int = 3) -> dict:
    """Config 1 in full on the reference: evolve + expectation through its own
    StateVectorBackend (engine.py:59-75; 1 core -- evolve is single-threaded
    and the backend's expectation is the serial statevector.expectation)."""
    _, RC, RSV = _reference_modules()
    import vqekit.engine as RE
    import vqekit.pauli as RP

    from paper_2208_10978_b200 import workloads as W

    cfg = W.config1(seed=0)
    n = cfg["n_qubits"]
    rgates = tuple(RC.Gate(g.kind, g.qubits, tuple(RC.Constant(p.value) for p in g.params))
                   for g in cfg["circuit"].gates)
    circ = RC.Circuit(n, rgates, 0)
    terms = []
    for t in cfg["hamiltonian"].terms:
        terms.append(RP.PauliTerm(complex(t.coefficient),
                                  RP.PauliString(tuple(t.string.factors))))
    h = RP.PauliSum(tuple(terms))
    be = RE.StateVectorBackend()
    s0 = be.prepare(cfg["reference"])
    e = be.expectation(be.evolve(s0, circ), h)  # warm
    t0 = time.perf_counter()
    for _ in range(evals):
        e = be.expectation(be.evolve(s0, circ), h)
    dt = (time.perf_counter() - t0) / evals
    return {"value": 1.0 / dt, "unit": "energy evals/s", "cores": 1, "kind": "reference",
            "energy": e, "s_per_eval": dt,
            "sample": f"config 1 in full ({len(rgates)} gates + 500 strings), {evals} evaluations "
                      "through vqekit.engine.StateVectorBackend (1 thread)",
            "host": host_info(1)}


def reference_expect30(workers: int | None = None) -> dict:
    """Config 3 (30 q, 10,000 strings) on the reference, extrapolated from a
    stratified sample: one string per worker (first half Z-only, the rest
    with flips, from the config-3 Hamiltonian) measured through the
    reference's own expectation_parallel (fork pool, OPENBLAS_NUM_THREADS=1,
    engine.py:177-199) on the config-3 state; time per string per worker x
    10,000 / W = the extrapolated full expectation."""
    import numpy as np

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    _, RC, RSV = _reference_modules()
    import vqekit.engine as RE
    import vqekit.pauli as RP

    from paper_2208_10978_b200 import workloads as W

    n = 30
    if workers is None:
        by_ram = (_avail_ram() - (24 << 30)) // (16 << n)  # state + one scratch per worker
        workers = int(max(1, min(os.cpu_count() or 1, by_ram)))
    h = W.config3_hamiltonian(seed=0)
    zs = [t for t in h.terms if all(a == "Z" for _, a in t.string.factors)]
    fl = [t for t in h.terms if not all(a == "Z" for _, a in t.string.factors)]
    pick = zs[: workers // 2] + fl[: workers - workers // 2]
    terms = tuple(RP.PauliTerm(complex(t.coefficient), RP.PauliString(tuple(t.string.factors)))
                  for t in pick)
    hs = RP.PauliSum(terms)
    amps = W.config3_state(seed=0)
    st = RSV.StateVector(n, amps)
    plan = RE.plan_partition(hs, workers)
    old = RE._PARALLEL_MIN_TERMS
    RE._PARALLEL_MIN_TERMS = 1  # a W-string sample must still take the fork-pool path
    try:
        t0 = time.perf_counter()
        RE.expectation_parallel(st, hs, plan)
        dt = time.perf_counter() - t0
    finally:
        RE._PARALLEL_MIN_TERMS = old
    per_string = dt  # each worker measured one string in dt (wall, incl. fork)
    full = per_string * len(h.terms) / workers
    return {"value": 1.0 / full, "unit": "expectations/s", "cores": workers, "kind": "reference",
            "s_per_eval_extrapolated": full, "sample_seconds": dt, "extrapolated": True,
            "sample": f"{len(pick)} strings ({workers // 2} Z-only + {workers - workers // 2} "
                      "with flips) of the config-3 H, one per worker, via "
                      "vqekit.engine.expectation_parallel (fork pool, OPENBLAS_NUM_THREADS=1) "
                      "on the config-3 state; x 10,000 / W",
            "host": host_info(workers)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    r = reference_gate_throughput(N_QUBITS, args.steps, args.warmup)
    value = r["value"]
    line = {
        "impl": "reference", "metric": "amplitude-updates/s", "value": value,
        "unit": "amplitude-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["seconds_per_step"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": "config2: 28q random brickwork depth 20 (830 gates), seed 0",
                   "sample": "2 U3 + 1 CNOT per worker per step"},
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "host")},
        "e2e": {"value": value, "unit": "amplitude-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# engine
# ---------------------------------------------------------------------------


def extra_ucc12(steps=20):
    import torch

    from paper_2208_10978_b200 import engine
    from paper_2208_10978_b200 import statevector as sv
    from paper_2208_10978_b200 import workloads as W

    cfg = W.config1(seed=0)
    be = engine.StateVectorBackend()
    s0 = be.prepare(cfg["reference"])
    # warm-up to steady state: plan, prepared program, specialised passes
    # (compiled once a structure has run QSV_JIT_HOT_USES times)
    for _ in range(6):
        be.expectation(be.evolve(s0, cfg["circuit"]), cfg["hamiltonian"])
    t0 = time.perf_counter()
    for _ in range(steps):
        e = be.expectation(be.evolve(s0, cfg["circuit"]), cfg["hamiltonian"])
    dt = (time.perf_counter() - t0) / steps
    passes = sv.last_plan_stats()["n_passes"]
    # a VQE iteration as a caller runs it: bind the parametric ansatz at new
    # angles (vectorised bind, no Gate objects), evolve, expectation
    from paper_2208_10978_b200.circuit import bind

    param = W.parametric_rotations_circuit(cfg["n_qubits"], cfg["strings"])
    thetas = cfg["thetas"]
    for _ in range(6):  # warm-up: the prepared program gets its specialised passes
        e_b = be.expectation(be.evolve(s0, bind(param, thetas)), cfg["hamiltonian"])
    assert abs(e_b - e) <= 1e-12 * max(1.0, abs(e))
    t0 = time.perf_counter()
    t_bind = 0.0
    for k in range(steps):
        tb = time.perf_counter()
        bound = bind(param, thetas + 1e-3 * k)
        t_bind += time.perf_counter() - tb
        be.expectation(be.evolve(s0, bound), cfg["hamiltonian"])
    dl = (time.perf_counter() - t0) / steps
    # reverse-mode gradient of the energy over all 1,872 parameters
    sv.reverse_gradient(param, thetas, cfg["hamiltonian"], s0)
    t0 = time.perf_counter()
    for _ in range(3):
        sv.reverse_gradient(param, thetas, cfg["hamiltonian"], s0)
    dg = (time.perf_counter() - t0) / 3
    return {"workload": "config1: 12q UCCSD-shaped (1,872 rotations = 37,824 gates) + 500-term H",
            "metric": "energy evals/s", "value": 1.0 / dt, "ms_per_eval": dt * 1e3, "energy": e,
            "passes": passes, "vqe_loop_evals_per_s": 1.0 / dl,
            "vqe_loop_bind_ms": t_bind / steps * 1e3, "gradient_ms": dg * 1e3,
            "gradient_params": int(param.n_params)}


def extra_expect30(steps=3):
    import torch

    from paper_2208_10978_b200 import statevector as sv
    from paper_2208_10978_b200 import workloads as W

    n = 30
    h = W.config3_hamiltonian(seed=0)
    s = sv.StateVector._empty(n)
    view = torch.as_tensor(s, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    view.copy_(torch.randn(view.shape, dtype=torch.float64, device="cuda", generator=g))
    view /= torch.linalg.vector_norm(view)
    torch.cuda.synchronize()
    sv.expectation_terms(s, h)  # plan + warm
    t0 = time.perf_counter()
    for _ in range(steps):
        re, im, _ = sv.expectation_terms(s, h)
    dt = (time.perf_counter() - t0) / steps
    st = sv.last_plan_stats()
    prods = len(h) * (1 << n)
    peak, peak_kind = load_peaks()
    peak_dfma, fp_src = load_fp64_peak()
    gbs = st["n_passes"] * 16 * (1 << n) / dt / 1e9
    roof = {"bound": "issue", "hbm": {"achieved": gbs, "peak": peak, "unit": "GB/s",
                                      "frac": gbs / peak, "peak_source": peak_kind,
                                      "algorithmic_bytes": st["n_passes"] * 16 * (1 << n)},
            "note": "each sweep reads the state once (16 B x 2^30); the work is the "
                    "per-(string, pair) products, signs and transforms"}
    try:
        with open(os.path.join(REPO, "profiles", "r02_expect30_counts.json")) as fh:
            cnt = json.load(fh)
        if cnt.get("sweeps") == st["n_passes"]:
            sm_clk = 1.965e9
            issue_peak = 148 * 4 * sm_clk  # warp instructions / s (one per SMSP per clock)
            fp = cnt["dfma"] + cnt["dmul"] + cnt["dadd"]
            roof.update({"achieved": cnt["warp_inst"] / dt, "peak": issue_peak,
                         "unit": "warp-instructions/s", "frac": cnt["warp_inst"] / dt / issue_peak,
                         "fp64_pipe_frac": fp / dt / peak_dfma, "counts": cnt,
                         "peak_note": "148 SMs x 4 schedulers x 1 warp-instruction/clk x 1.965 GHz"})
    except Exception:
        pass
    return {"workload": "config3: 30q expectation, 10,000 strings (30% Z-only), random state "
                        "(torch-generated on device)",
            "metric": "expectations/s", "value": 1.0 / dt, "ms_per_eval": dt * 1e3,
            "sweeps": st["n_passes"], "term_amplitude_products_per_s": prods / dt,
            "hbm_gbs_sweeps": gbs, "roofline": roof}


def extra_fused30(steps=3):
    """North-star fused gate application at 30 qubits: a config-4-shaped UCC
    circuit (all singles + 2,000 doubles, 15 electrons) on 30 qubits, evolve
    only, resident state.  Reports HBM GB/s over the launched passes
    (32 B x 2^30 per pass) against MEASURED_PEAKS.json."""
    import torch

    from paper_2208_10978_b200 import engine
    from paper_2208_10978_b200 import statevector as sv
    from paper_2208_10978_b200 import workloads as W

    cfg = W.config4(seed=0, n_qubits=30, n_electrons=15, n_doubles=2000, n_terms=10)
    be = engine.StateVectorBackend()
    s0 = be.prepare(cfg["reference"])

    def timed():
        psi = be.evolve(s0, cfg["circuit"])  # plan + specialise
        psi.synchronize()
        del psi
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            psi = be.evolve(s0, cfg["circuit"])
            psi.synchronize()
            ts.append(time.perf_counter() - t0)
            st = sv.last_plan_stats()
            del psi
        return min(ts), st

    # the roofline is a 30-qubit one: the full state, parity reduction off
    old = os.environ.get("QSV_PARITY")
    os.environ["QSV_PARITY"] = "0"
    try:
        dt, st = timed()
    finally:
        if old is None:
            del os.environ["QSV_PARITY"]
        else:
            os.environ["QSV_PARITY"] = old
    dt_half, st_half = timed()  # default: the HF state's parity class as a 29-qubit half
    passes = st["n_passes"]
    peak, _ = load_peaks()
    gbs = (passes * 32.0 - 16.0) * (1 << 30) / dt / 1e9  # first pass synthesises the HF state
    return {"workload": "30q UCC-shaped circuit (config 4 construction at n=30, 15 e): "
                        f"{st['n_rotations']} Pauli rotations, evolve only",
            "metric": "amplitude-updates/s", "value": st["n_rotations"] * (1 << 30) / dt,
            "s_per_evolve": dt, "passes": passes, "hbm_gbs": gbs, "hbm_frac": gbs / peak,
            "parity_reduced": {"s_per_evolve": dt_half, "passes": st_half["n_passes"],
                               "note": "default path: even-flip (number-conserving) rotations keep the HF "
                                       "state's index-parity class, evolved exactly as a 29-qubit half "
                                       "(symmetry.py); the roofline above is the full 30-qubit state"}}


def extra_brick33(steps=2):
    """Single-GPU base of the weak-scaling family the N > 1 lines run: the
    config-5 brickwork construction (depth 10) on 33 qubits = 2^33 amplitudes
    (128 GiB), one B200, from |0...0> (R_1 of E_N = R_N / (N R_1))."""
    from paper_2208_10978_b200 import statevector as sv
    from paper_2208_10978_b200 import workloads as W

    n = 33
    circ = W.brickwork(n, 10, SEED)
    sv.release_pool()
    psi = sv.evolve(sv.init_state("0" * n), circ)  # plan + specialise
    psi.synchronize()
    del psi
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        psi = sv.evolve(sv.init_state("0" * n), circ)
        psi.synchronize()
        ts.append(time.perf_counter() - t0)
        passes = sv.last_plan_stats()["n_passes"]
        del psi
    dt = min(ts)
    return {"workload": f"config5 construction on 33q (depth 10, {len(circ.gates)} gates), 1 GPU, "
                        "128 GiB state", "metric": "amplitude-updates/s",
            "value": len(circ.gates) * float(1 << n) / dt, "s_per_evolve": dt, "passes": passes}


def extra_ucc32(steps=1):
    from paper_2208_10978_b200 import engine
    from paper_2208_10978_b200 import statevector as sv
    from paper_2208_10978_b200 import workloads as W

    cfg = W.config4(seed=0)
    be = engine.StateVectorBackend()
    s0 = be.prepare(cfg["reference"])
    psi = be.evolve(s0, cfg["circuit"])
    e = be.expectation(psi, cfg["hamiltonian"])
    del psi
    t0 = time.perf_counter()
    for _ in range(steps):
        psi = be.evolve(s0, cfg["circuit"])
        st_ev = sv.last_plan_stats()
        e = be.expectation(psi, cfg["hamiltonian"])
        del psi
    dt = (time.perf_counter() - t0) / steps
    psi = be.evolve(s0, cfg["circuit"])
    psi.synchronize()
    t1 = time.perf_counter()
    psi2 = be.evolve(s0, cfg["circuit"])
    psi2.synchronize()
    t_ev = time.perf_counter() - t1
    del psi, psi2
    n_eff = sv.last_reduction()["n_eff"] or 32
    peak, _ = load_peaks()
    gbs = (st_ev["n_passes"] * 32.0 - 16.0) * (1 << n_eff) / t_ev / 1e9  # first pass: write only
    return {"workload": "config4: 32q UCC (16,512 rotations) + 5,000-term H",
            "metric": "energy evals/s", "value": 1.0 / dt, "s_per_eval": dt, "energy": e,
            "decomposed_gates": len(cfg["circuit"].gates),
            "evolve_passes": st_ev["n_passes"], "s_per_evolve": t_ev, "evolve_hbm_gbs": gbs,
            "evolve_hbm_frac": gbs / peak, "evolved_qubits": n_eff,
            "symmetry": ("index-parity reduction: the UCC rotations have even flips, so the HF state's "
                         "parity class (half of the 2^32 amplitudes) is evolved exactly as a "
                         f"{n_eff}-qubit state and the energy is taken on it (symmetry.py; QSV_PARITY=0 "
                         "runs the full 32 q)") if n_eff < 32 else None}


def run_engine(args, rank, world, local):
    import numpy as np
    import torch

    from paper_2208_10978_b200 import engine
    from paper_2208_10978_b200 import statevector as sv
    from paper_2208_10978_b200 import workloads as W
    from paper_2208_10978_b200 import _lib
    from paper_2208_10978_b200.circuit import flatten_bound

    torch.cuda.set_device(local)
    dev = local
    circ = W.brickwork(N_QUBITS, LAYERS, SEED)
    G = len(circ.gates)
    dim = 1 << N_QUBITS
    be = engine.StateVectorBackend(device=dev)

    # library stream -> torch events
    probe = sv.init_state("0" * N_QUBITS, dev)
    probe._ensure()
    import ctypes
    sp = ctypes.c_void_p()
    _lib.check(_lib.lib().qsv_get_stream(probe.handle, ctypes.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", dev))
    del probe

    def step():
        return sv.evolve(be.prepare("0" * N_QUBITS), circ)

    for _ in range(args.warmup):
        psi = step()
        del psi
    stats = sv.last_plan_stats()
    passes = stats["n_passes"]
    torch.cuda.synchronize(dev)

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    _, jit_before = _lib.jit_info()
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize(dev)
        start.record(stream)
        for _ in range(args.steps):
            psi = step()
            del psi
        end.record(stream)
        torch.cuda.synchronize(dev)
    _, jit_after = _lib.jit_info()
    t_step = start.elapsed_time(end) / 1e3 / args.steps
    # |0..0> is synthesised by the first pass (qsv_evolve_basis): the step is
    # exactly its passes
    t_pass = t_step / passes

    t_max = t_step
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_step], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())

    value = world * G * dim / t_max
    n_u1 = sum(1 for g in circ.gates if len(g.qubits) == 1)

    # e2e: public API with host buffers (gate arrays in, full state out to
    # pinned host memory) every step.  Steps are pipelined the way a caller
    # streaming circuits would run them: step k's state download (copy
    # stream, PCIe-bound) overlaps step k+1's evolve; the timed region ends
    # when the last download has landed.
    host_out = [torch.empty(dim, dtype=torch.complex128, pin_memory=True).numpy() for _ in range(2)]
    kinds, qubits, values = flatten_bound(circ)
    h2d = kinds.nbytes + qubits.nbytes + values.nbytes
    e2e_steps = max(2, args.steps)
    psi = be.evolve(be.prepare("0" * N_QUBITS), circ)
    psi.download_into(host_out[0])
    del psi
    t0 = time.perf_counter()
    prev = None
    for k in range(e2e_steps):
        sv._FLAT_CACHE.clear()  # re-read the gate list from the host objects every step
        psi = be.evolve(be.prepare("0" * N_QUBITS), circ)
        psi.download_async(host_out[k % 2])
        if prev is not None:
            prev.wait_download()
        prev = psi
    prev.wait_download()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    del prev, psi
    e2e_val = world * G * dim / t_e2e
    if rank == 0:
        assert abs(np.linalg.norm(host_out[0]) - 1.0) < 1e-9
        assert np.array_equal(host_out[0], host_out[1])

    peak, peak_kind = load_peaks()
    # 32 B x 2^n per pass (16 read + 16 write), except the first pass, which
    # synthesises |0..0> and only writes: mean over the step's launches
    alg_bytes = (32.0 * passes - 16.0) / passes * dim
    achieved = alg_bytes / t_pass / 1e9
    line = {
        "metric": "amplitude-updates/s", "value": value, "unit": "amplitude-updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {"workload": "config2: 28q random brickwork depth 20 (830 gates: 560 U3 + 270 CNOT), "
                               "seed 0, from |0...0>", "n_qubits": N_QUBITS, "gates": G,
                   "hbm_passes_per_step": passes, "l2": "state 4 GiB >> 126 MB L2 (no flush needed)",
                   "parallelism": f"replica x{world}"},
        "e2e": {"value": e2e_val, "unit": "amplitude-updates/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": 16 * dim, "ms_per_step": t_e2e * 1e3, "steps": e2e_steps,
                "note": "StateVector.download_async: step k's 4 GiB D2H overlaps step k+1's "
                        "evolve; timed until the last download completes"},
        "roofline": fp64_roofline(t_step, passes, n_u1 * dim * 8,
                                  {"achieved": achieved, "peak": peak, "unit": "GB/s",
                                   "frac": achieved / peak, "peak_source": peak_kind,
                                   "algorithmic_bytes_per_launch": alg_bytes,
                                   "ms_per_launch": t_pass * 1e3,
                                   "traffic": TRAFFIC_PER_LAUNCH,
                                   "traffic_source": "ncu dram__bytes_read+write of one pass "
                                                     "(profiles/r01_jit_pass_ncu.txt)"}),
        # specialised pass launches counted by the library over the timed
        # region (the evolve from |0..0> needs no separate set_basis kernel)
        "gpu_launches": int(jit_after - jit_before),
        "clocks": clocks.summary(),
    }

    extras = [e for e in (args.extra or "").split(",") if e and e != "none"]
    if rank == 0 and extras:
        line["extra"] = {}
        for e in extras:
            fn = {"ucc12": extra_ucc12, "expect30": extra_expect30, "ucc32": extra_ucc32,
                  "fused30": extra_fused30, "brick33": extra_brick33}[e]
            try:
                line["extra"][e] = fn()
            except Exception as exc:  # an extra must never cost the headline line
                line["extra"][e] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference's own gate loop on all host cores, 2 steps (~20 s)
        try:
            r = reference_gate_throughput(N_QUBITS, steps=2, warmup=0)
            line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                      "host", "seconds_per_step")}
        except Exception as exc:
            line["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        ex = line.get("extra", {})
        cpu_legs = {"ucc12": reference_ucc12, "expect30": reference_expect30}
        for name, fn in cpu_legs.items():
            if name in ex and "error" not in ex[name]:
                try:
                    ex[name]["cpu_reference"] = fn()
                    ex[name]["vs_cpu_reference"] = ex[name]["value"] / ex[name]["cpu_reference"]["value"]
                except Exception as exc:
                    ex[name]["cpu_reference"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        if "ucc32" in ex and "error" not in ex["ucc32"] and "value" in line.get("cpu_baseline", {}):
            # config 4 cannot run on the CPU (64 GiB state + copy, ~5e5 gates):
            # per-core gate rate at 28 q x the decomposed gate count at 32 q,
            # plus 5,000 strings at the per-string cost of the config-3 sample x 4
            cb = line["cpu_baseline"]
            gates32 = ex["ucc32"].get("decomposed_gates", 0)
            t_ev = gates32 * float(1 << 32) / cb["value"]
            e30 = ex.get("expect30", {}).get("cpu_reference", {})
            t_h = (e30["s_per_eval_extrapolated"] * 4 * 5_000 / 10_000
                   if "s_per_eval_extrapolated" in e30 else 0.0)
            ex["ucc32"]["cpu_reference"] = {
                "kind": "reference", "extrapolated": True, "cores": cb["cores"],
                "s_per_eval_extrapolated": t_ev + t_h, "value": 1.0 / (t_ev + t_h),
                "unit": "energy evals/s",
                "sample": "evolve: decomposed gates x 2^32 / the reference's all-core gate rate "
                          "(cpu_baseline); H: 5,000 strings x 4 (32 q vs 30 q) at the config-3 "
                          "sample's per-string rate on its W workers"}
            ex["ucc32"]["vs_cpu_reference"] = ex["ucc32"]["value"] * (t_ev + t_h)
    if rank == 0:
        print(json.dumps(line), flush=True)


def _swap_launches() -> int:
    import ctypes

    from paper_2208_10978_b200 import _lib

    v = ctypes.c_int64()
    _lib.check(_lib.lib().qsv_swap_info(ctypes.byref(v)))
    return v.value


def nvlink_alltoall_probe(local: int, nbytes: int = 1 << 30, iters: int = 5) -> dict:
    """Measured all-to-all bandwidth between the ranks (torch.distributed
    all_to_all_single over NCCL): bytes each GPU sends to the others per
    second -- the denominator of the relayout's NVLink fraction."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    n = (nbytes // 8 // world) * world
    src = torch.empty(n, dtype=torch.float64, device=f"cuda:{local}").fill_(1.0)
    dst = torch.empty_like(src)
    for _ in range(2):
        dist.all_to_all_single(dst, src)
    torch.cuda.synchronize(local)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    a.record()
    for _ in range(iters):
        dist.all_to_all_single(dst, src)
    b.record()
    torch.cuda.synchronize(local)
    t = torch.tensor([a.elapsed_time(b) / 1e3 / iters], device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sent = 8 * n * (world - 1) / world
    return {"GB_per_s_per_gpu": sent / float(t.item()) / 1e9, "bytes_per_gpu": sent,
            "how": f"all_to_all_single of {8 * n / 2**30:.2f} GiB per rank, max over ranks, "
                   f"{iters} iterations"}


def run_engine_dist(args, rank, world, local):
    """Sharded brickwork, weak scaling at config 5's shard size: 2^33
    amplitudes (128 GiB) per GPU, n = 33 + log2(N) qubits, depth 10 (N = 8
    is config 5 itself: 36 q)."""
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2208_10978_b200 import _lib
    from paper_2208_10978_b200 import distributed as D
    from paper_2208_10978_b200 import workloads as W

    if args.dist_backend != "nccl":  # single-GPU plumbing test: ranks share the visible GPUs
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    g = world.bit_length() - 1
    n = int(os.environ.get("QSV_BENCH_LOCAL_QUBITS", "33")) + g
    layers = int(os.environ.get("QSV_BENCH_LAYERS", "10"))
    circ = W.brickwork(n, layers, SEED)
    G = len(circ.gates)
    comm = D.ProcessGroupComm()
    be = D.DistributedBackend(comm, D.CudaEngine(local))

    def step():
        return be.evolve(be.prepare("0" * n), circ)

    nvl = nvlink_alltoall_probe(local) if args.dist_backend == "nccl" else None
    for _ in range(args.warmup):
        psi = step()
        del psi
    torch.cuda.synchronize(local)
    dist.barrier()
    torch.cuda.synchronize(local)
    _, launches0 = _lib.jit_info()
    swaps0 = _swap_launches()
    with ClockSampler(local) as clocks:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        relayout_s = 0.0
        relayouts = 0
        sent = 0
        for _ in range(args.steps):
            psi = step()
            for sh in psi.shards.values():
                sh.synchronize()
            relayout_s += psi.stats["relayout_seconds"]
            relayouts += psi.stats["relayouts"]
            sent += psi.stats["relayout_bytes_sent"]
            del psi
        end.record()
        torch.cuda.synchronize(local)
    _, launches1 = _lib.jit_info()
    swaps1 = _swap_launches()
    t_step = start.elapsed_time(end) / 1e3 / args.steps
    dev_t = "cuda" if args.dist_backend == "nccl" else "cpu"
    tt = torch.tensor([t_step, relayout_s / args.steps], device=dev_t)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max, t_swap = float(tt[0].item()), float(tt[1].item())
    value = G * (1 << n) / t_max
    n_local = n - g
    passes = (launches1 - launches0) / args.steps

    # e2e: the public API with host inputs every step -- the gate list is
    # flattened from the host Circuit objects, the state is evolved, and the
    # step's result read back to the host is an observable, <Z_0 Z_{n-1}> +
    # <X_0> (a 2^n-amplitude state is 16 TiB... at config 5 the state itself
    # is 1 TiB, so no caller downloads it); max over ranks
    from paper_2208_10978_b200.pauli import PauliString, PauliSum, PauliTerm

    obs = PauliSum((PauliTerm(1.0, PauliString(((0, "Z"), (n - 1, "Z")))),
                    PauliTerm(0.5, PauliString(((0, "X"),)))))
    e2e_steps = max(2, min(args.steps, 4))
    from paper_2208_10978_b200 import circuit as C

    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        C._FLAT_STRUCTS.clear()  # re-read the gate list from the host objects every step
        psi = step()
        val = be.expectation(psi, obs)
        del psi
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([t_e2e], device=dev_t)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())

    # UCC energy evals/s at P GPUs (BASELINE metric; config 4 sharded):
    # every rank takes part; one warm-up evaluation (plans, specialisation)
    extras = [e for e in (args.extra or "").split(",") if e and e != "none"]
    ucc = None
    if "ucc32" in extras:
        nq = int(os.environ.get("QSV_BENCH_UCC_QUBITS", "32"))
        cfg = W.config4(seed=0, n_qubits=nq, n_electrons=nq // 2)
        s0 = be.prepare(cfg["reference"])
        e = be.expectation(be.evolve(s0, cfg["circuit"]), cfg["hamiltonian"])
        dist.barrier()
        torch.cuda.synchronize(local)
        t0 = time.perf_counter()
        psi = be.evolve(s0, cfg["circuit"])
        e = be.expectation(psi, cfg["hamiltonian"])  # returns a float: synchronised
        rel, sent_u = psi.stats["relayouts"], psi.stats["relayout_bytes_sent"]
        del psi
        tu = torch.tensor([time.perf_counter() - t0], device=dev_t)
        dist.all_reduce(tu, op=dist.ReduceOp.MAX)
        ucc = {"workload": f"config4 construction at {nq}q (UCC rotations + 5,000-term H), "
                           f"state sharded x{world}",
               "metric": "energy evals/s", "value": 1.0 / float(tu.item()),
               "s_per_eval": float(tu.item()), "energy": e, "relayouts": rel,
               "relayout_bytes_sent_per_gpu": sent_u}

    peak, peak_kind = load_peaks()
    if rank == 0:
        t_local = max(t_max - t_swap, 1e-12)
        hbm = passes * 32.0 * (1 << n_local) / t_local / 1e9 if passes else None
        swap_gbs = (sent / args.steps) / max(t_swap, 1e-12) / 1e9
        line = {
            "metric": "amplitude-updates/s", "value": value, "unit": "amplitude-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "config": {"workload": f"config5 family: {n}q random brickwork depth {layers} "
                                   f"({G} gates), seed {SEED}, sharded over {world} GPUs "
                                   f"(2^{n_local} amplitudes = {16 * (1 << n_local) / 2**30:.0f} GiB "
                                   f"per GPU, {g} global qubits)" + (" = config 5" if n == 36 else ""),
                       "n_qubits": n, "gates": G, "parallelism": f"state sharded x{world} (global qubits)",
                       "l2": f"shard {16 * (1 << n_local) / 2**30:.2f} GiB >> 126 MB L2 (no flush needed)"},
            "e2e": {"value": G * (1 << n) / t_e2e, "unit": "amplitude-updates/s",
                    "h2d_bytes_per_step": int(G * 40), "d2h_bytes_per_step": 16 * world,
                    "ms_per_step": t_e2e * 1e3, "steps": e2e_steps, "observable": val,
                    "note": "host Circuit flattened + evolve + <Z0 Z_{n-1}> + 0.5<X0> to the host "
                            "every step (per-rank partials gathered); max over ranks"},
            "swap": {"relayouts_per_step": relayouts / args.steps,
                     "bytes_sent_per_gpu_per_step": sent / args.steps,
                     "seconds_per_step": t_swap, "GB_per_s": swap_gbs,
                     "nvlink_peak": nvl,
                     "nvlink_frac": (swap_gbs / nvl["GB_per_s_per_gpu"]) if nvl else None},
            "roofline": {"bound": "hbm", "achieved": hbm, "peak": peak, "unit": "GB/s",
                         "frac": (hbm / peak) if hbm else None, "traffic": None,
                         "kernel": "qsv_pass (tile passes between relayouts)",
                         "passes_per_step": passes, "peak_source": peak_kind,
                         "note": "32 B x 2^n_local per pass over the step time minus relayout time"},
            "gpu_launches": int(launches1 - launches0) + int(swaps1 - swaps0),
            "gpu_launches_note": "specialised tile passes + relayout swap kernels over peer memory (qsv_swap_peer)",
            "clocks": clocks.summary(),
        }
        if ucc is not None:
            line["extra"] = {"ucc32_sharded": ucc}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--extra", default="ucc12,fused30,expect30,ucc32,brick33",
                    help="secondary workloads (configs 1, 3, 4 and the 30q fused-gate roofline); 'none' to skip")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # bind the rank's GPU before NCCL creates its communicator;
        # --dist-backend gloo: plumbing test of the sharded path on one GPU
        # (device shards staged through host memory); never a bench number
        if args.dist_backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    if world > 1:
        run_engine_dist(args, rank, world, local)
    else:
        run_engine(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
