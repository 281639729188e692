#!/usr/bin/env python
"""Benchmark of the B200 stabilizer-tableau hot path (BASELINE.json metric: gates/sec and
wall-s for the 180k-qubit depth-1000 Clifford+measure circuit; HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

One step = one full run_single_shot of the configured circuit (every gate window, the
transposes and every measurement collapse) on device-resident inputs. `value` is the circuit's
gates/s, timed with CUDA events (max over ranks); `e2e` is the same metric through the public
API with host buffers (schedule + upload + simulate + record and tableau download).
N > 1 (torchrun): one process per GPU drives one generator-word shard of the SAME tableau
(strong scaling): gate windows run shard-local, measurement windows exchange pivot blocks and
partial products over NCCL inside libqsr (csrc/shard.cpp, csrc/exchange.cu).
--local-shards S (N = 1): the sharded engine with all S shards on the one GPU (the
multi-GPU protocol's overhead, measured on one device).
"""
from __future__ import annotations

import argparse
import ctypes as C
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
    "c5": dict(n=180000, depth=1000, seed=42, p=0.01, run_seed=7),
}
DESCR = {
    "c1": "random Clifford, 1,000 qubits, depth 100, measure all (generate_random seed 42, run seed 7)",
    "c2": "random Clifford, 20,000 qubits, depth 1,000 (generate_random seed 42, run seed 7)",
    "c3": "mid-circuit-measurement-heavy: 50,000 qubits, 10 segments generate_random(50000,100,1000+r,1.0) "
          "(100 layers then measure every qubit), run seed 7",
    "c5": "paper headline: random Clifford+measure, 180,000 qubits, depth 1,000, "
          "Bernoulli(0.01) final measurements (generate_random(180000,1000,42,0.01), run seed 7)",
}
METRIC = "gates/sec and wall-s for 180k-qubit depth-1000 Clifford+measure; HBM GB/s"
# Kind-exact (reads, writes) in u64 words per generator-word, reference gates.hpp:35-115.
RW = np.array([(1, 0), (2, 0), (1, 0), (2, 2), (2, 1), (2, 1), (4, 2), (4, 3), (4, 2), (4, 4), (4, 4), (0, 0)])


def log(*a):
    print(*a, file=sys.stderr, flush=True)


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


def gate_bytes(circuit, k: int, gate_windows: int) -> float:
    kinds = np.bincount(circuit.gate_array["kind"], minlength=12)
    words = float((kinds * RW.sum(axis=1)).sum())
    return 8.0 * 2 * k * words + 16.0 * 2 * k * gate_windows


def barrier(dist):
    if dist is not None:
        dist.barrier()


def cpu_reference_windows(cfg, warm: int, timed: int):
    """Reference CPU path (oracle/_ref, all host cores) on the first warm+timed layers of the
    configured circuit; returns (gates/s over the timed windows, per-window seconds, kind, cores)."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    o = Oracle(kind)
    cores = os.cpu_count() or 1
    o.set_threads(cores)
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
    return float(g.sum() / t.sum()), t, kind, cores


def run_reference_arm(args, cfg, world, rank, dist):
    if rank != 0:
        return
    t0 = time.time()
    rate, t, kind, cores = cpu_reference_windows(cfg, args.warmup, args.steps)
    ms = float(np.mean(t) * 1e3)
    sample = (f"first {args.warmup}+{args.steps} gate windows (layers) of the {args.config} circuit on a "
              f"{cfg['n']}-qubit zero-state tableau; reference apply_window, {cores} threads; "
              f"{args.warmup} untimed, {args.steps} timed; gates/s over the timed windows")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "gates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": DESCR[args.config], "step": "one gate window (bounded CPU sample)"},
            "cpu_baseline": {"value": rate, "unit": "gates/s", "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": rate, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.time() - t0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-windows", type=int, default=2, help="timed CPU-baseline windows (rank 0)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--local-shards", type=int, default=1,
                    help="N = 1 only: run the sharded engine with this many shards on the one GPU")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    from paper_2603_14641_b200 import dist as qd
    world, rank, local, dist = qd.init_from_env("nccl")
    if args.impl == "reference":
        run_reference_arm(args, cfg, world, rank, dist)
        return

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
    _, offs, flags = sched.arrays()
    gate_windows = int((flags == 0).sum())
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
    step_ms, gate_ms, gate_launch, gate_dev_bytes = [], 0.0, 0, 0.0
    with Clocks(device) as clk:
        for i in range(args.steps):
            ms = eng.run(run_seed)
            st = eng.stats()
            step_ms.append(ms)
            gate_ms += st["gate_ms"]
            gate_launch += st["gate_launches"]
            gate_dev_bytes += st.get("gate_bytes", 0.0)
            log(f"[rank {rank}] step {i}: {ms:.1f} ms  {st}")
    barrier(dist)
    launches = q.launch_count() - launches0
    total_ms = qd.max_over_ranks(dist, float(np.sum(step_ms)))
    ms_per_step = total_ms / args.steps
    value = G * args.steps / (total_ms * 1e-3)

    # Roofline of the dominant kernel (gate windows): algorithmic bytes per launch over the
    # average launch duration measured above with CUDA events on the engine's stream. The bytes
    # are those of the device gates actually launched (kind-exact words), i.e. after
    # the exact gate fusion (SWAP relabelling, single-qubit runs folded into the next two-qubit
    # gate); `unfused_*` restates the reference-semantics bytes of the same windows and the
    # resulting effective bandwidth.
    launches_per_step = gate_launch / args.steps
    gb_ref_step = gate_bytes(circ, k if (world == 1 and shards > 1) else kg_local, gate_windows)
    gb_step = gate_dev_bytes / args.steps if gate_dev_bytes > 0 else gb_ref_step
    per_launch_bytes = gb_step / launches_per_step
    per_launch_s = (gate_ms / gate_launch) * 1e-3
    achieved = per_launch_bytes / per_launch_s / 1e9
    effective = gb_ref_step / (gate_ms / args.steps * 1e-3) / 1e9
    peak, peak_src = peaks()
    kernel = "k_gate_segment" if os.environ.get("QSR_GATE_ENGINE") == "segment" else "k_gate_window"
    traffic = None
    tp = ROOT / "profiles" / "gate_window_traffic.json"
    if tp.exists():
        try:
            for d in json.loads(tp.read_text()).get("entries", []):
                fused = os.environ.get("QSR_FUSE", "1") != "0" and world == 1 and shards == 1
                if (d.get("config") == args.config and d.get("kernel", "").startswith(kernel) and shards == 1
                        and bool(d.get("fused", False)) == fused):
                    traffic = d.get("dram_bytes_per_launch")
        except Exception:
            pass
    st = eng.stats()
    del eng

    # e2e through the public API with host buffers, every step: N = 1 -> qsr_run_single_shot
    # (schedule, validation, packed gate upload, simulation, record download) + final tableau
    # download into pinned memory; N > 1 -> ShardedEngine create (schedule + upload per rank),
    # run, record download and this rank's tableau columns.
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
            rate, t, kind, cores = cpu_reference_windows(cfg, 1, args.cpu_windows)
            cpu = {"value": rate, "unit": "gates/s", "cores": cores, "kind": kind,
                   "sample": f"reference apply_window on the first 1+{args.cpu_windows} layers of the "
                             f"{args.config} circuit ({cfg['n']} qubits), first window untimed; "
                             f"{float(np.sum(t)):.1f} s timed on {cores} host threads"}
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "unit": "gates/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": DESCR[args.config], "qubits": n, "depth": cfg["depth"], "gates": G,
                   "measurements": nm, "windows": int(len(flags)), "gate_windows": gate_windows,
                   "parallelism": (f"generator-row shards x{world} (NCCL)" if world > 1 else
                                   f"generator-row shards x{shards} on one GPU (local exchange)"
                                   if shards > 1 else "single GPU"),
                   "l2": f"inputs larger than L2 (tableau {2 * n_pad * 2 * k * 8 / 1e9:.2f} GB vs 126 MB L2); "
                         "no flush needed"},
        "wall_s_per_step": ms_per_step / 1e3,
        "phase_ms_per_step": {"gate_windows": gate_ms / args.steps, "transpose": st["transpose_ms"],
                              "measure": st["measure_ms"]},
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "bytes_per_launch": per_launch_bytes, "launch_ms": per_launch_s * 1e3,
                     "unfused_bytes_per_step": gb_ref_step, "effective_unfused_gbs": effective,
                     "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": "gates/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "s_per_step": e2e_total / max(e2e_steps, 1)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
