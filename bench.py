#!/usr/bin/env python
"""Benchmark of the B200 stabilizer-tableau hot path (BASELINE.json metric: gates/sec and
wall-s for the 180k-qubit depth-1000 Clifford+measure circuit; HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

One step = one full run_single_shot of the configured circuit (every gate window, the
transposes and every measurement collapse) on device-resident inputs. `value` is the circuit's
gates/s, timed with CUDA events (max over ranks); `e2e` is the same metric through the public
API with host buffers (schedule + upload + simulate + record and tableau download).
--config c4: one step = one sample(circuit, 100000 shots) (frames.hpp:163-204) on the resident
engine — the reference shot plus the Pauli frames riding the same device windows.
N > 1 (torchrun): one process per GPU drives one generator-word shard of the SAME tableau
(strong scaling): gate windows run shard-local, measurement windows exchange pivot blocks and
partial products over NCCL inside libqsr (csrc/shard.cpp, csrc/exchange.cu).
--local-shards S (N = 1): the sharded engine with all S shards on the one GPU (the
multi-GPU protocol's overhead, measured on one device).
--impl reference: the reference's own CPU path (oracle/_ref = proj/include/quasar compiled
unmodified) on the host cores; this process never loads libqsr.so.
"""
from __future__ import annotations

import argparse
import ctypes as C
import importlib.util
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": dict(n=1000, depth=100, seed=42, p=1.0, run_seed=7),
    "c2": dict(n=20000, depth=1000, seed=42, p=0.0, run_seed=7),
    "c3": dict(n=50000, depth=100, seed=1000, p=1.0, run_seed=7, segments=10),
    "c4": dict(n=10000, depth=500, seed=42, p=1.0, run_seed=7, shots=100000),
    "c5": dict(n=180000, depth=1000, seed=42, p=0.01, run_seed=7),
}
DESCR = {
    "c1": "random Clifford, 1,000 qubits, depth 100, measure all (generate_random seed 42, run seed 7)",
    "c2": "random Clifford, 20,000 qubits, depth 1,000 (generate_random seed 42, run seed 7)",
    "c3": "mid-circuit-measurement-heavy: 50,000 qubits, 10 segments generate_random(50000,100,1000+r,1.0) "
          "(100 layers then measure every qubit), run seed 7",
    "c4": "many-shot sampling: 10,000 qubits, depth 500, measure all (generate_random(10000,500,42,1.0)), "
          "sample(100000 shots, seed 7)",
    "c5": "paper headline: random Clifford+measure, 180,000 qubits, depth 1,000, "
          "Bernoulli(0.01) final measurements (generate_random(180000,1000,42,0.01), run seed 7)",
}
METRIC = "gates/sec and wall-s for 180k-qubit depth-1000 Clifford+measure; HBM GB/s"
# Kind-exact (reads, writes) in u64 words per generator-word, reference gates.hpp:35-115.
RW = np.array([(1, 0), (2, 0), (1, 0), (2, 2), (2, 1), (2, 1), (4, 2), (4, 3), (4, 2), (4, 4), (4, 4), (0, 0)])
# Frames (frames.hpp:76-94): X / Y / Z only flip signs, which frames do not track.
RW_FRAMES = RW.copy()
RW_FRAMES[0:3] = 0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_dist():
    """paper_2603_14641_b200/dist.py by path: importing the package would load libqsr.so,
    and the reference arm must not map it."""
    spec = importlib.util.spec_from_file_location("qsr_dist", ROOT / "paper_2603_14641_b200" / "dist.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = Path(f"/tmp/qsr_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            # A timed region shorter than nvidia-smi's start-up + one period (c2: ~70 ms) has no
            # sample yet: keep the sampler until its first row lands (at most ~3 s).
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 3.0 and self.proc.poll() is None:
                try:
                    if any(len(l.split(",")) >= 6 for l in self.path.read_text().splitlines()):
                        break
                except OSError:
                    pass
                time.sleep(0.02)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path.exists():
            return None
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:]))
            except ValueError:
                continue
        if not rows:
            return None
        sm = sorted(r[0] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": rows[0][1], "reasons": reasons, "samples": len(rows)}


def gate_bytes(kinds_count, k: int, gate_windows: int, frames: bool = False) -> float:
    rw = RW_FRAMES if frames else RW
    words = float((kinds_count * rw.sum(axis=1)).sum())
    return 8.0 * 2 * k * words + (0.0 if frames else 16.0 * 2 * k * gate_windows)


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---- CPU legs (reference compiled unmodified, oracle/_ref; the C port if absent) ----------
def cpu_oracle():
    from oracle.oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    o = Oracle(kind)
    cores = os.cpu_count() or 1
    o.set_threads(cores)
    return o, kind, cores


def cpu_reference_windows(o, cfg, warm: int, timed: int):
    """Reference apply_window (gates.hpp:147-197) on the first warm+timed layers of the configured
    circuit; returns (gates/s over the timed windows, per-window seconds, mean gates/window)."""
    L = warm + timed
    sec = np.zeros(L, dtype=np.float64)
    gts = np.zeros(L, dtype=np.uint64)
    fn = o.lib.orc_bench_windows
    fn.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p]
    st = fn(cfg["n"], L, cfg["seed"], C.c_void_p(sec.ctypes.data), C.c_void_p(gts.ctypes.data))
    if st != 0:
        raise RuntimeError(o.lib.orc_last_error().decode())
    t = sec[warm:]
    g = gts[warm:].astype(np.float64)
    return float(g.sum() / t.sum()), t, float(g.mean())


def run_reference_arm(args, cfg):
    """`--impl reference`: the reference CPU path on the host cores, rank 0 only (the other
    ranks exit without work). A step is one gate window (layer) of the configured circuit
    through the reference apply_window: the full run is hours on the CPU."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    t0 = time.time()
    o, kind, cores = cpu_oracle()
    rate, t, gpw = cpu_reference_windows(o, cfg, args.warmup, args.steps)
    ms = float(np.mean(t) * 1e3)
    sample = (f"CPU gate-window sample: layers {args.warmup + 1}..{args.warmup + args.steps} of the "
              f"{args.config} circuit ({cfg['n']} qubits, {gpw:.0f} gates per layer) through the reference "
              f"apply_window on a zero-state tableau, {cores} threads, after {args.warmup} untimed layers; "
              f"gates/s over the timed layers. The measurement phase is not part of this arm's step (the "
              f"repo arm's cpu_baseline adds a measurement sample and a whole-run projection)")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "gates/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": {"workload": DESCR[args.config], "step": "CPU gate-window sample (one layer of the circuit)"},
            "cpu_baseline": {"value": rate, "unit": "gates/s", "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": rate, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.time() - t0}
    print(json.dumps(line), flush=True)


def cpu_baseline_with_measurement(q, o, kind, cores, circ, cfg, sched_arrays, record, args, G):
    """The reference CPU path on a bounded sample of the SAME workload, projected to a whole run:
    gate windows (reference apply_window on the circuit's first layers), the CM<->RM transpose
    pair and the first collapses of the first measurement window (reference measure_window,
    measure.hpp:381-442) on the actual scrambled state the circuit reaches there (computed on
    the GPU, downloaded once)."""
    rate, t, gpw = cpu_reference_windows(o, cfg, 1, args.cpu_windows)
    t_win = float(np.mean(t))
    g, off, fl = sched_arrays
    W_u = int((fl == 0).sum())
    n_mwin = int((fl != 0).sum())
    n_prob = int((record["deterministic"] == 0).sum()) if len(record) else 0
    out = {"gate_window_rate": rate, "gate_window_s": t_win, "gate_windows": W_u}
    proj = W_u * t_win
    sample = (f"reference apply_window on layers 2..{1 + args.cpu_windows} of the {args.config} circuit "
              f"({t_win:.2f} s per layer)")
    timed_s = float(np.sum(t))
    if n_mwin and args.cpu_collapses > 0:
        n = cfg["n"]
        w_first = int(np.argmax(fl != 0))
        t_gpu = q.Tableau.zero_state(n)
        for w in range(w_first):
            q.apply_window(t_gpu, g[off[w]:off[w + 1]])
        x, z, s = t_gpu.planes()
        del t_gpu
        # measure_window = 2 transposes + the collapses: time it on m1 and m2 > m1 of the
        # window's first measurements (each on the same snapshot), the difference is m2 - m1
        # collapses; the intercept is the transpose pair.
        m2 = min(args.cpu_collapses, int(off[w_first + 1] - off[w_first]))
        m1 = max(1, m2 // 4)
        t_mw, m_prob = [], []
        for m in (m1, m2):
            xs, zs, ss = (x.copy(), z.copy(), s.copy()) if m == m1 else (x, z, s)
            t0 = time.perf_counter()
            ent, _ = o.measure_window(n, 0, xs, zs, ss, g[off[w_first]:off[w_first] + m], cfg["run_seed"], 0)
            t_mw.append(time.perf_counter() - t0)
            m_prob.append(int((ent["deterministic"] == 0).sum()))
            del xs, zs, ss
        t_col = max(t_mw[1] - t_mw[0], 0.0) / max(m_prob[1] - m_prob[0], 1)
        t_T = max(t_mw[0] - m_prob[0] * t_col, 0.0) / 2
        proj += n_prob * t_col + n_mwin * 2 * t_T
        timed_s += sum(t_mw)
        out.update({"transpose_s": t_T, "collapse_s": t_col, "measure_window_s": t_mw,
                    "collapses_sampled": m_prob, "probabilistic_collapses": n_prob, "measure_windows": n_mwin})
        sample += (f"; reference measure_window on the first {m1} and {m2} measurements of the first "
                   f"measurement window ({t_mw[0]:.1f} s, {t_mw[1]:.1f} s) on the circuit's actual state there "
                   f"(GPU-computed snapshot): {t_col:.2f} s per collapse, {t_T:.2f} s per transpose")
    out["projected_run_s"] = proj
    value = G / proj
    sample += (f"; whole-run projection {proj:.0f} s = {W_u} windows x layer time"
               + (" + collapses x collapse time + 2 transposes per measurement window" if n_mwin else "")
               + f"; {timed_s:.1f} s of CPU work timed on {cores} host threads")
    return {"value": value, "unit": "gates/s", "cores": cores, "kind": kind, "sample": sample, "detail": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-windows", type=int, default=2, help="timed CPU-baseline gate windows (rank 0)")
    ap.add_argument("--cpu-collapses", type=int, default=None,
                    help="CPU-baseline collapses on the GPU snapshot (default: 4 at c5, 32 below)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="skip the measurement-pass profile run")
    ap.add_argument("--local-shards", type=int, default=1,
                    help="N = 1 only: run the sharded engine with this many shards on the one GPU")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.cpu_collapses is None:
        args.cpu_collapses = 8 if cfg["n"] >= 100000 else 32
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    if args.config == "c4":
        return bench_sampling(args, cfg)

    qd = load_dist()
    world, rank, local, dist = qd.init_from_env("nccl")
    from paper_2603_14641_b200 import _lib
    from paper_2603_14641_b200 import quasar as q
    device = local
    t0 = time.time()
    if cfg.get("segments"):  # concatenated measure-all segments
        circ = q.Circuit(cfg["n"], np.concatenate(
            [q.generate_random(cfg["n"], cfg["depth"], cfg["seed"] + r, cfg["p"]).gate_array
             for r in range(cfg["segments"])]))
    else:
        circ = q.generate_random(cfg["n"], cfg["depth"], cfg["seed"], cfg["p"])
    G = len(circ)
    nm = circ.measure_count()
    log(f"[rank {rank}] generated {G} gates ({nm} measurements) in {time.time() - t0:.1f}s")
    t0 = time.time()
    sched = q.schedule_windows(circ)
    sched_arrays = sched.arrays()
    _, offs, flags = sched_arrays
    gate_windows = int((flags == 0).sum())
    meas_windows = int((flags != 0).sum())
    log(f"[rank {rank}] scheduled {len(flags)} windows in {time.time() - t0:.2f}s")
    n = cfg["n"]
    k = (n + 63) // 64
    n_pad = 64 * k
    run_seed = cfg["run_seed"]
    nccl_id = qd.share_nccl_id(dist, rank) if world > 1 else None
    shards = world if world > 1 else args.local_shards

    def make_engine():
        if world > 1:
            return q.ShardedEngine(circ, world, device=device, exchange="nccl", rank=rank, nccl_id=nccl_id)
        if shards > 1:
            return q.ShardedEngine(circ, shards, device=device, exchange="local")
        return q.Engine(circ, device=device)  # circuit upload: scheduled + gate-fused (fuse.hpp)

    t0 = time.time()
    eng = make_engine()
    log(f"[rank {rank}] engine ({'sharded x%d' % shards if shards > 1 else 'single'}) up in {time.time() - t0:.1f}s")
    kg_local = q.shard_range(n, world, rank)[1] if world > 1 else k

    for i in range(args.warmup):
        ms = eng.run(run_seed)
        log(f"[rank {rank}] warmup {i}: {ms:.1f} ms  {eng.stats()}")

    launches0 = q.launch_count()
    barrier(dist)
    step_ms, gate_ms, gate_launch, gate_dev_bytes, tr_ms, meas_ms = [], 0.0, 0, 0.0, 0.0, 0.0
    with Clocks(device) as clk:
        for i in range(args.steps):
            ms = eng.run(run_seed)
            st = eng.stats()
            step_ms.append(ms)
            gate_ms += st["gate_ms"]
            gate_launch += st["gate_launches"]
            gate_dev_bytes += st.get("gate_bytes", 0.0)
            tr_ms += st["transpose_ms"]
            meas_ms += st["measure_ms"]
            log(f"[rank {rank}] step {i}: {ms:.1f} ms  {st}")
    barrier(dist)
    launches = q.launch_count() - launches0
    total_ms = qd.max_over_ranks(dist, float(np.sum(step_ms)))
    ms_per_step = total_ms / args.steps
    value = G * args.steps / (total_ms * 1e-3)
    record = eng.record() if world == 1 and shards == 1 else None

    # Roofline of the gate-window kernel: algorithmic bytes per launch over the average launch
    # duration measured above with CUDA events on the engine's stream. The bytes are those of the
    # device gates actually launched (kind-exact words), i.e. after the exact gate
    # fusion (SWAP relabelling, single-qubit runs folded into the next two-qubit gate);
    # `unfused_*` restates the reference-semantics bytes of the same windows.
    peak, peak_src = peaks()
    kinds = np.bincount(circ.gate_array["kind"], minlength=12)
    launches_per_step = gate_launch / args.steps
    gb_ref_step = gate_bytes(kinds, k if (world == 1 and shards > 1) else kg_local, gate_windows)
    gb_step = gate_dev_bytes / args.steps if gate_dev_bytes > 0 else gb_ref_step
    per_launch_bytes = gb_step / max(launches_per_step, 1)
    per_launch_s = (gate_ms / max(gate_launch, 1)) * 1e-3
    traffic_entries = []
    tp = ROOT / "profiles" / "gate_window_traffic.json"
    if tp.exists():
        try:
            traffic_entries = json.loads(tp.read_text()).get("entries", [])
        except Exception:
            traffic_entries = []

    def traffic_of(kernel):
        fused = os.environ.get("QSR_FUSE", "1") != "0" and world == 1 and shards == 1
        for d in traffic_entries:
            if (d.get("config") == args.config and d.get("kernel", "").startswith(kernel) and shards == 1
                    and bool(d.get("fused", fused)) == fused):
                return d.get("dram_bytes_per_launch")
        return None

    gate_roof = None
    if gate_launch:
        achieved = per_launch_bytes / per_launch_s / 1e9
        gate_roof = {"bound": "hbm", "kernel": "k_gate_window", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic_of("k_gate_window"),
                     "bytes_per_launch": per_launch_bytes, "launch_ms": per_launch_s * 1e3,
                     "ms_per_step": gate_ms / args.steps, "unfused_bytes_per_step": gb_ref_step,
                     "effective_unfused_gbs": gb_ref_step / (gate_ms / args.steps * 1e-3) / 1e9,
                     "peak_source": peak_src}
    # Transposes (k_transpose, 4 plane launches per measurement window): 2 planes x (read +
    # write) x 8 B x n_pad x 2kg per direction.
    tr_roof = None
    if meas_windows and tr_ms > 0:
        tr_bytes = meas_windows * 2 * (2 * 2 * 8.0 * n_pad * 2 * kg_local)
        a = tr_bytes / (tr_ms / args.steps * 1e-3) / 1e9
        tr_roof = {"bound": "hbm", "kernel": "k_transpose", "achieved": a, "peak": peak, "unit": "GB/s",
                   "frac": a / peak, "bytes_per_step": tr_bytes, "ms_per_step": tr_ms / args.steps,
                   "traffic": traffic_of("k_transpose")}
    # Measurement pass (k_batch_absorb): one more run, outside the timed region, with CUDA events
    # around every absorb launch and a device count of the rows each batch rewrites; algorithmic
    # bytes per rewritten row = x and z read + written over its k words (32 k B) + one phase byte
    # per 64-word slice.
    absorb_roof = None
    if meas_windows and world == 1 and shards == 1 and not args.no_profile:
        prof = eng.profile(run_seed)
        if prof["absorb_launches"]:
            ab = prof["absorb_rows"] * (32.0 * prof["row_words"] + prof["absorb_slices"])
            a = ab / (prof["absorb_ms"] * 1e-3) / 1e9
            absorb_roof = {"bound": "hbm", "kernel": "k_batch_absorb", "achieved": a, "peak": peak, "unit": "GB/s",
                           "frac": a / peak, "bytes_per_launch": ab / prof["absorb_launches"],
                           "launch_ms": prof["absorb_ms"] / prof["absorb_launches"],
                           "launches_per_step": prof["absorb_launches"], "ms_per_step": prof["absorb_ms"],
                           "rows_per_launch": prof["absorb_rows"] / prof["absorb_launches"],
                           "traffic": traffic_of("k_batch_absorb"),
                           "how": "one profile run after the timed steps (events around each absorb launch)"}
    # The line's roofline = the kernel class that dominates the step.
    cands = [(r["ms_per_step"], r) for r in (gate_roof, tr_roof, absorb_roof) if r]
    roofline = max(cands, key=lambda c: c[0])[1] if cands else None
    st = eng.stats()
    del eng

    # e2e through the public API with host buffers, every step: N = 1 -> qsr_run_single_shot
    # (schedule, validation, packed gate upload, simulation, record download) + final tableau
    # download into pinned memory; N > 1 -> qsr_sharded_run_circuit on every rank (the same
    # streamed driver on the rank's shard, sharded measurement), record download and this rank's
    # tableau columns.
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    # Host buffers: the full tableau at N = 1; each rank's own columns (1/N of it) at N > 1.
    plane = n_pad * 2 * k if world == 1 else n_pad * 2 * kg_local
    px, pz = C.c_void_p(), C.c_void_p()
    _lib.check(_lib.lib.qsr_host_alloc(plane * 8, C.byref(px)))
    _lib.check(_lib.lib.qsr_host_alloc(plane * 8, C.byref(pz)))
    ps = np.empty(2 * k, dtype=np.uint64)
    rec = np.zeros(max(nm, 1), dtype=_lib.ENTRY_DTYPE)
    e2e_s = []
    barrier(dist)
    for i in range(e2e_steps):
        t1 = time.perf_counter()
        if world > 1 or shards > 1:
            if world > 1:  # the streamed sharded driver: plan / fuse / upload behind the device
                e = q.ShardedEngine(circ, world, device=device, exchange="nccl", rank=rank, nccl_id=nccl_id,
                                    streamed_seed=run_seed)
            else:
                e = make_engine()
                e.run(run_seed)
            _lib.check(_lib.lib.qsr_sharded_record(e._h, _lib.ptr(rec)))
            if world > 1:  # this rank's columns, compact
                _lib.check(_lib.lib.qsr_sharded_tableau_local(e._h, C.cast(px, _lib.pu64), C.cast(pz, _lib.pu64),
                                                              _lib.ptr(ps, C.c_uint64)))
            else:  # local shards of one process: the full reference layout
                _lib.check(_lib.lib.qsr_sharded_tableau(e._h, C.cast(px, _lib.pu64), C.cast(pz, _lib.pu64),
                                                        _lib.ptr(ps, C.c_uint64)))
            del e
        else:
            rep = _lib.Report_t()
            h = C.c_void_p()
            _lib.check(_lib.lib.qsr_run_single_shot(circ._h, None, run_seed, device, C.byref(h), _lib.ptr(rec),
                                                    C.byref(rep)))
            _lib.check(_lib.lib.qsr_tableau_download(h, C.cast(px, _lib.pu64), C.cast(pz, _lib.pu64),
                                                     _lib.ptr(ps, C.c_uint64)))
            _lib.lib.qsr_tableau_destroy(h)
        e2e_s.append(time.perf_counter() - t1)
        log(f"[rank {rank}] e2e {i}: {e2e_s[-1]:.2f} s")
    barrier(dist)
    _lib.lib.qsr_host_free(px)
    _lib.lib.qsr_host_free(pz)
    e2e_total = qd.max_over_ranks(dist, float(np.sum(e2e_s))) if e2e_steps else float("nan")
    e2e_value = G * e2e_steps / e2e_total if e2e_steps else None
    h2d = world * (8 * G + 4 * nm)
    d2h = world * 8 * nm + 2 * 8 * (n_pad * 2 * k) + 8 * 2 * k  # all ranks together: the tableau once

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            o, kind, cores = cpu_oracle()
            cpu = cpu_baseline_with_measurement(q, o, kind, cores, circ, cfg, sched_arrays,
                                                record if record is not None else np.zeros(0, _lib.ENTRY_DTYPE),
                                                args, G)
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "unit": "gates/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": DESCR[args.config], "qubits": n, "depth": cfg["depth"] * cfg.get("segments", 1),
                   "gates": G, "measurements": nm, "windows": int(len(flags)), "gate_windows": gate_windows,
                   "measure_windows": meas_windows,
                   "parallelism": (f"generator-row shards x{world} (NCCL)" if world > 1 else
                                   f"generator-row shards x{shards} on one GPU (local exchange)"
                                   if shards > 1 else "single GPU"),
                   "l2": f"inputs larger than L2 (tableau {2 * n_pad * 2 * k * 8 / 1e9:.2f} GB vs 126 MB L2); "
                         "no flush needed"},
        "wall_s_per_step": ms_per_step / 1e3,
        "phase_ms_per_step": {"gate_windows": gate_ms / args.steps, "transpose": tr_ms / args.steps,
                              "measure": meas_ms / args.steps},
        "roofline": roofline,
        "kernels": {"gate_window": gate_roof, "transpose": tr_roof, "measure_absorb": absorb_roof},
        "e2e": {"value": e2e_value, "unit": "gates/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "s_per_step": e2e_total / max(e2e_steps, 1)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sampling(q, o, kind, cores, circ, cfg, sched_arrays, record, args, G, shots):
    """Reference sample() (frames.hpp:163-204) on bounded samples of the c4 workload, projected to
    a whole call: schedule_windows, the reference shot (gate windows + transposes + collapses on
    the circuit's actual state, as cpu_baseline_with_measurement), the frames' windows on 100k
    shots (apply_window_frames) and the final measure_sample."""
    base = cpu_baseline_with_measurement(q, o, kind, cores, circ, cfg, sched_arrays, record, args, G)
    d = base["detail"]
    n = cfg["n"]
    g, off, fl = sched_arrays
    t0 = time.perf_counter()
    o.schedule(n, circ.gate_array)
    t_sched = time.perf_counter() - t0
    xf, zf = o.init_frames(n, shots, cfg["run_seed"])
    wins = [w for w in range(len(fl)) if not fl[w]][:1 + args.cpu_windows]
    o.apply_window_frames(n, shots, xf, zf, g[off[wins[0]]:off[wins[0] + 1]])  # untimed
    t0 = time.perf_counter()
    for w in wins[1:]:
        o.apply_window_frames(n, shots, xf, zf, g[off[w]:off[w + 1]])
    t_fwin = (time.perf_counter() - t0) / max(len(wins) - 1, 1)
    kf = (shots + 63) // 64
    mw = [w for w in range(len(fl)) if fl[w]]
    t_ms = 0.0
    if mw:
        meas = g[off[mw[0]]:off[mw[0] + 1]]
        measured = np.zeros(n, dtype=np.uint32)
        words = np.zeros(n * kf, dtype=np.uint64)
        t0 = time.perf_counter()
        o.measure_sample(n, shots, xf, zf, meas, cfg["run_seed"], 1, measured, 0, words)
        t_ms = (time.perf_counter() - t0) * len(mw)
    proj = d["projected_run_s"] + t_sched + d["gate_windows"] * t_fwin + t_ms
    d.update({"schedule_s": t_sched, "frames_window_s": t_fwin, "measure_sample_s": t_ms, "projected_run_s": proj})
    base["value"] = G / proj
    base["sample"] += (f"; plus reference schedule_windows ({t_sched:.1f} s), apply_window_frames on {shots} "
                       f"shots ({t_fwin:.2f} s per layer, {len(wins) - 1} layers timed) and measure_sample "
                       f"({t_ms:.2f} s): whole sample() call projected at {proj:.0f} s")
    return base


def bench_sampling(args, cfg):
    """c4: one step = sample(circuit, shots, seed) on the resident engine (reference shot + frames
    riding its windows, record fold), CUDA-event timed. N > 1: each rank samples its shot-word
    slice (frames.hpp:63 keys are global; no communication), weak in shots per GPU = strong in
    the total (the SAME 100k shots are split)."""
    qd = load_dist()
    world, rank, local, dist = qd.init_from_env("nccl")
    from paper_2603_14641_b200 import _lib
    from paper_2603_14641_b200 import quasar as q
    device = local
    n, shots, seed = cfg["n"], cfg["shots"], cfg["run_seed"]
    t0 = time.time()
    circ = q.generate_random(n, cfg["depth"], cfg["seed"], cfg["p"])
    G = len(circ)
    nm = circ.measure_count()
    sched_arrays = q.schedule_windows(circ).arrays()
    _, offs, flags = sched_arrays
    gate_windows = int((flags == 0).sum())
    log(f"[rank {rank}] generated + scheduled {G} gates in {time.time() - t0:.1f}s")
    eng = q.Engine(circ, device=device)
    for i in range(args.warmup):
        _, ms = eng.sample(shots, seed, record=False, world=world, rank=rank)
        log(f"[rank {rank}] warmup {i}: {ms:.1f} ms")
    launches0 = q.launch_count()
    barrier(dist)
    step_ms, gate_ms, gb, fb, fms = [], 0.0, 0.0, 0.0, 0.0
    with Clocks(device) as clk:
        for i in range(args.steps):
            _, ms = eng.sample(shots, seed, record=False, world=world, rank=rank)
            st = eng.stats()
            b, f_ms = eng.frames_stats()
            step_ms.append(ms)
            gate_ms += st["gate_ms"]
            gb += st["gate_bytes"]
            fb += b
            fms += f_ms
            log(f"[rank {rank}] step {i}: {ms:.1f} ms  frames windows {f_ms:.1f} ms  {st}")
    barrier(dist)
    launches = q.launch_count() - launches0
    total_ms = qd.max_over_ranks(dist, float(np.sum(step_ms)))
    ms_per_step = total_ms / args.steps
    value = G * args.steps / (total_ms * 1e-3)
    peak, peak_src = peaks()
    # The frames' gate windows (k_gate_window without signs, on the frames' own stream, beside the
    # reference shot) dominate: their algorithmic bytes (frames rule words x shot-words) over
    # their event-timed runs. The reference shot's tableau windows are reported beside them.
    fa = fb / (fms * 1e-3) / 1e9 if fms else None
    roof = {"bound": "hbm", "kernel": "k_gate_window (frames instance, no signs)", "achieved": fa, "peak": peak,
            "unit": "GB/s", "frac": fa / peak if fa else None, "traffic": None,
            "bytes_per_step": fb / args.steps, "ms_per_step": fms / args.steps, "peak_source": peak_src}
    ta = gb / (gate_ms * 1e-3) / 1e9 if gate_ms else None
    tab = {"bound": "hbm", "kernel": "k_gate_window (reference-shot tableau)", "achieved": ta, "peak": peak,
           "unit": "GB/s", "frac": ta / peak if ta else None, "bytes_per_step": gb / args.steps,
           "ms_per_step": gate_ms / args.steps,
           "note": "10k-qubit tableau (2 x 25 MB) is L2-resident: frac above 1 is L2 bandwidth"}
    record = eng.record()
    del eng
    # e2e: the public sample() call (qsr_sample / qsr_sample_shard: schedule + upload streamed,
    # reference shot + frames, fold) and the ShotRecord download to the host.
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    e2e_s = []
    rec_bytes = 0
    # The record words land in pinned host memory (as the c5 leg's tableau does), allocated once
    # outside the timed region.
    kf_all = (shots + 63) // 64
    pinned = q.PinnedBuffer(8 * max(nm, 1) * (kf_all // world + 1))

    def e2e_call():
        if world > 1:
            return q.sample_shard(circ, shots, seed, world, rank, device=device, out=pinned.array)[1]
        return q.sample(circ, shots, seed, device=device, out=pinned.array)

    if e2e_steps:
        e2e_call()  # one untimed call (first-use allocations), like the device leg's warm-up
    barrier(dist)
    for i in range(e2e_steps):
        t1 = time.perf_counter()
        r = e2e_call()
        e2e_s.append(time.perf_counter() - t1)
        rec_bytes = int(r.words.nbytes + 4 * len(r.measured))
        log(f"[rank {rank}] e2e {i}: {e2e_s[-1]:.3f} s")
    barrier(dist)
    e2e_total = qd.max_over_ranks(dist, float(np.sum(e2e_s)))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            o, kind, cores = cpu_oracle()
            cpu = cpu_baseline_sampling(q, o, kind, cores, circ, cfg, sched_arrays, record, args, G, shots)
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "unit": "gates/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": DESCR["c4"], "qubits": n, "depth": cfg["depth"], "gates": G, "measurements": nm,
                   "shots": shots, "gate_windows": gate_windows,
                   "parallelism": f"shot-word slices x{world}" if world > 1 else "single GPU",
                   "step": "one sample() call on the resident engine (gates/s of the circuit per call)",
                   "l2": "frames planes 2 x 125 MB + record 125 MB > 126 MB L2; no flush needed"},
        "shots_per_s": shots * args.steps / (total_ms * 1e-3),
        "wall_s_per_step": ms_per_step / 1e3,
        "roofline": roof,
        "kernels": {"frames_window": roof, "tableau_window": tab},
        "e2e": {"value": G * e2e_steps / e2e_total if e2e_steps else None, "unit": "gates/s",
                "h2d_bytes_per_step": world * 12 * G, "d2h_bytes_per_step": world * rec_bytes,
                "s_per_step": e2e_total / max(e2e_steps, 1)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
