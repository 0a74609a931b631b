#!/usr/bin/env python
"""Benchmark of the batched full-order PIC step (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One "step" = one fused gather-kick-drift-deposit pass over all Np x p particles
with the per-instance Poisson solve in the same kernel (picrom_pic_step), on
device-resident state; instance groups are pipelined on separate streams.  The
default workload is BASELINE.json configs[1] (C2: two-stream, p = 32 instances
x 250,000 particles, Nx = 128, cubic splines).  L2 is flushed once before the
timed block; the K steps then run back to back (the production schedule), so
each step pays the write-back of the previous one.  The line also carries the
C1/C5 full-order and C3/C4 reduced-model sections (`other_configs`, N = 1), the
oracle port's CPU rate at the config's degree (`cpu_baseline`) and the
unmodified P1 reference from baseline/_ref (`reference_p1`).
Multi-GPU (torchrun): every rank runs its own independent C2 batch (instance
sharding, no collective on the data path; weak scaling); time = max over ranks.

`--impl reference` times the reference algorithm's CPU implementation (the
numpy oracle port in oracle/ at the config's degree, all host cores via column
threads like VlasovSystem(workers=...)) on the same config; rank 0 only.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-pushes/s (Np x p x steps) fp64 on 1 B200; % of HBM roofline"
UNIT = "pushes/s"
BYTES_PER_PUSH = 32          # x, v read + write, fp64
DATA = "synthetic (seeded loading per SURVEY.md §8(d); BASELINE names no dataset)"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the soak and the timed region:
    NVML polled every 10 ms from a thread (the timed block of K = 20 steps is
    ~1.4 ms, far below nvidia-smi's 200 ms loop); falls back to the
    `nvidia-smi -lms 200` loop of the profiling recipe when pynvml is missing."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index):
        self.rows = []           # (sm MHz, max MHz, reasons bitmask or list)
        self.proc = None
        self.gpu = gpu_index
        self._stop = threading.Event()
        self._thread = None
        self.source = None

    def _device_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v for v in vis.split(",") if v.strip() != ""]
            if self.gpu < len(ids) and ids[self.gpu].strip().isdigit():
                return int(ids[self.gpu])
        return self.gpu

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self._device_index())
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), int(rs)))
                    except pynvml.NVMLError:
                        pass
                    self._stop.wait(0.01)
            self.source = "nvml 10 ms"
            self._thread = threading.Thread(target=poll, daemon=True)
            self._thread.start()
            return
        except Exception:
            self.source = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.source = "nvidia-smi 200 ms"
        threading.Thread(target=self._read, daemon=True).start()

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7 and parts[0].replace(".", "").isdigit() and parts[1].replace(".", "").isdigit():
                mask = sum(self.BITS[names[i]] for i in range(4) if parts[3 + i] == "Active")
                self.rows.append((float(parts[0]), float(parts[1]), mask))

    def stop(self):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=1.0)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            time.sleep(0.05)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows]
        mask = 0
        for r in self.rows:
            mask |= r[2]
        reasons = sorted(n for n, bit in self.BITS.items() if mask & bit)
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": max(mx),
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


def host_info():
    """CPU model, cores, BLAS threading and library versions of the host timing
    the CPU rows."""
    import platform

    import scipy
    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")}
                for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception:  # pragma: no cover
        pass
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0)), "blas": blas,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "numpy": np.__version__, "scipy": scipy.__version__,
            "python": platform.python_version()}


def bench_config(w, world):
    """The `config` dict both arms print (identical keys and values)."""
    n, p = w.num_particles, w.p
    return w.describe() | {
        "parallelism": f"instance-sharded replicas, {world} rank(s), no data-path collective",
        "l2": "flushed (256 MiB write + 256 MiB read) before the timed block; the K steps run back "
              "to back and each moves 32 B/push (C2: 256 MB > 126 MB L2), so inputs exceed L2",
        "state_bytes": 2 * n * p * 8}


def cpu_oracle_rate(w, seconds=10.0, max_steps=20, warm=1):
    """Reference algorithm on the host cores: the oracle port (degree-p
    B-splines, oracle/pic_loop.py) with column threads like
    VlasovSystem(workers=cores), reference-order Verlet steps."""
    from oracle import fe_bspline as fe
    from oracle import pic_loop
    from paper_2201_05555_b200 import workloads as wl
    cores = len(os.sched_getaffinity(0))
    x, v = wl.generate(w)
    n, p = x.shape
    L = float(w.lengths[0])
    sysm = pic_loop.System(fe.Mesh(L, w.num_cells, w.degree), fe.Charge(n, L), workers=cores)
    st = pic_loop.Stepper(sysm)
    t = 0.0
    for _ in range(warm):
        x, v, t = st.step(x, v, t, w.dt)
    steps, t0 = 0, time.perf_counter()
    while steps < max_steps:
        x, v, t = st.step(x, v, t, w.dt)
        steps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    el = time.perf_counter() - t0
    return {"value": n * p * steps / el, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{w.name} full size ({p} x {n}), {steps} reference-order Verlet steps "
                      f"(fullorder.py:122-134) in {el:.1f} s, numpy oracle port at degree "
                      f"{w.degree} (oracle/pic_loop.py), {cores} column threads"}


def reference_p1_rate(w, seconds=10.0, max_steps=20, warm=1):
    """The REAL reference package (picrom from baseline/_ref, pip-installed from
    /root/reference/pkg) on the same particles: VlasovSystem(workers=cores) +
    VerletStepper.step (fullorder.py:57-134).  The reference is P1-only
    (fem.py:1-13), so this row is degree 1 -- labelled, not the config's degree."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "picrom").exists():
        return {"unavailable": "baseline/_ref/picrom not installed"}
    sys.path.insert(0, str(ref))
    try:
        from picrom import fem as rfem
        from picrom import fullorder as rfo
    finally:
        sys.path.remove(str(ref))
    from paper_2201_05555_b200 import workloads as wl
    cores = len(os.sched_getaffinity(0))
    x, v = wl.generate(w)
    n, p = x.shape
    L = float(w.lengths[0])
    sysm = rfo.VlasovSystem(rfem.build_mesh(L, w.num_cells),
                            rfem.ChargeConfig(num_particles=n, length=L), workers=cores)
    st = rfo.VerletStepper(sysm)
    ens = rfo.ParticleEnsemble(x, v, 0.0)
    for _ in range(warm):
        ens = st.step(ens, w.dt)
    steps, t0 = 0, time.perf_counter()
    while steps < max_steps:
        ens = st.step(ens, w.dt)
        steps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    el = time.perf_counter() - t0
    return {"value": n * p * steps / el, "unit": UNIT, "cores": cores, "kind": "reference",
            "degree": 1,
            "sample": f"{w.name} particles ({p} x {n}), {steps} VerletStepper.step calls of the "
                      f"unmodified reference (baseline/_ref/picrom, P1 finite elements -- the "
                      f"reference has no degree {w.degree}) with VlasovSystem(workers={cores}), "
                      f"{el:.1f} s"}


def run_reference(args, w, rank, world):
    """--impl reference: the reference algorithm's CPU implementation on the
    host cores, rank 0 only (the oracle port at the config's degree; the real
    P1 reference beside it)."""
    if rank != 0:
        return
    from oracle import fe_bspline as fe
    from oracle import pic_loop
    from paper_2201_05555_b200 import workloads as wl
    cores = len(os.sched_getaffinity(0))
    x, v = wl.generate(w)
    n, p = x.shape
    L = float(w.lengths[0])
    sysm = pic_loop.System(fe.Mesh(L, w.num_cells, w.degree), fe.Charge(n, L), workers=cores)
    st = pic_loop.Stepper(sysm)
    t = 0.0
    for _ in range(args.warmup):
        x, v, t = st.step(x, v, t, w.dt)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x, v, t = st.step(x, v, t, w.dt)
    el = time.perf_counter() - t0
    val = n * p * args.steps / el
    sample = (f"{w.name} full size ({p} x {n} particles), {args.steps} reference-order Verlet "
              f"steps (fullorder.py:122-134) of the numpy oracle port, degree {w.degree}, "
              f"{cores} column threads")
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "impl": "reference", "config": bench_config(w, world),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_p1": reference_p1_rate(w) if not args.no_cpu_baseline else None,
            "host": host_info()}
    print(json.dumps(line), flush=True)


def fom_measure(args, w, world, local_rank, e2e_steps=None, steps=None, warmup=None,
                clocks_soak=True):
    """Device-timed batched PIC steps + the end-to-end public call for workload w."""
    import torch
    from paper_2201_05555_b200 import fem, fullorder
    from paper_2201_05555_b200 import workloads as wl
    steps = steps or args.steps
    warmup = warmup or args.warmup
    xh, vh = wl.generate(w, layout="pn")                 # (p, N) host
    p, n = xh.shape
    L = float(w.lengths[0])
    sysm = fullorder.VlasovSystem(fem.build_mesh(L, w.num_cells, w.degree), fem.ChargeConfig(n, L))
    xd = torch.from_numpy(xh).cuda()
    vd = torch.from_numpy(vh).cuda()
    run = fullorder.PicRun(sysm, xd, vd, w.dt, warmup + steps + 1)
    run.init_field()
    run.advance(1)                      # the half-kick first step
    e = run.e

    # L2 flush before the timed block (outside the events): a 256 MiB write,
    # then a 256 MiB read so the lines left in L2 are clean.  Inside the block
    # the steps run back to back -- the production schedule of run_full_order:
    # each step's 32 B/push exceed the 126 MB L2 at C2/C5, and the write-back of
    # one step's dirty lines is paid inside the next
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    flush_rd = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    flush_sink = torch.empty((), dtype=torch.float64, device="cuda")

    def l2_flush():
        flush.zero_()
        torch.sum(flush_rd, dim=0, out=flush_sink)

    l2_flush()
    e.launch_block(warmup)
    torch.cuda.synchronize()
    # the K timed steps are one CUDA-graph replay -- the production schedule of
    # run_full_order (graph blocks of steps) -- so the timed region holds the K
    # steps' kernels and no Python launch latency (from Python the first kernel
    # reaches the GPU ~40 us after the start event: +2-3 us per step at K = 20)
    timed_block = None
    try:
        timed_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(timed_graph):
            e.launch_block(steps)
        timed_graph.replay()            # untimed: part of the warm-up
        timed_block = timed_graph.replay
    except RuntimeError:                # capture refused (e.g. another stream busy): plain launches
        torch.cuda.synchronize()
        timed_block = lambda: e.launch_block(steps)
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    if clocks_soak:
        # short soak (untimed) at this exact load; the clock sampler (NVML, 10 ms)
        # keeps polling through it and through the timed K steps that follow
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < args.soak_seconds:
            e.launch_block(16)
            torch.cuda.synchronize()
    l2_flush()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    ev0.record()
    timed_block()                       # exactly K steps, every instance group
    ev1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        tdist.barrier()
    step_ms = ev0.elapsed_time(ev1)
    run.check()
    t_local = torch.tensor([step_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        tdist.all_reduce(t_local, op=tdist.ReduceOp.MAX)
    step_ms = float(t_local[0])
    groups = e.groups

    # end-to-end: the public call with host (pinned) buffers, full configured run
    e2e_steps = e2e_steps or w.num_steps
    xn = torch.from_numpy(np.ascontiguousarray(xh.T)).pin_memory()
    vn = torch.from_numpy(np.ascontiguousarray(vh.T)).pin_memory()
    del run, xd, vd, e
    torch.cuda.empty_cache()
    rec_opts = fullorder.RecordOptions(energy_stride=1, record_snapshots=False)
    # warm-up call of the same shape (engine + CUDA graph capture happen once
    # per system/shape; the timed call is the steady-state user call)
    fullorder.run_full_order(sysm, fullorder.ParticleEnsemble(xn, vn, 0.0), w.dt, e2e_steps * w.dt,
                             record=rec_opts)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rec = fullorder.run_full_order(sysm, fullorder.ParticleEnsemble(xn, vn, 0.0), w.dt,
                                   e2e_steps * w.dt, record=rec_opts)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    assert rec.final_state.x.device.type == "cpu"
    e_local = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        tdist.all_reduce(e_local, op=tdist.ReduceOp.MAX)
        e2e_s = float(e_local[0])
    h2d = 2 * n * p * 8
    d2h = 2 * n * p * 8 + rec.electric_history.nbytes * 2 + rec.potential_history.nbytes * 2
    peak, peak_src = peaks()
    push_avg_s = step_ms / 1e3 / steps
    achieved = BYTES_PER_PUSH * n * p / push_avg_s / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(w.name, {}).get("traffic_bytes_per_launch")
    return {
        "value": n * p * steps * world / (step_ms / 1e3), "ms_per_step": step_ms / steps,
        "steps": steps, "warmup": warmup,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "step_kernel (fused gather-kick-drift-deposit + last-CTA Poisson "
                               f"solve), {groups} instance group(s) pipelined on separate "
                               "streams; achieved = algorithmic bytes per step / device time per "
                               "step of K back-to-back steps",
                     "algorithmic_bytes_per_launch": BYTES_PER_PUSH * n * p,
                     "avg_launch_ms": step_ms / steps, "peak_source": peak_src},
        "kernel_share_of_step": 1.0,
        "instance_groups": groups,
        "e2e": {"value": n * p * e2e_steps * world / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": h2d / e2e_steps, "d2h_bytes_per_step": d2h / e2e_steps,
                "call": f"fullorder.run_full_order({e2e_steps} steps) from pinned host (N,p) "
                        "arrays, host record + final state back", "seconds": e2e_s},
        "gpu_launches": steps * groups,
        "clocks": clk,
    }


def run_ours(args, w, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2201_05555_b200 import _build, _lib
    from paper_2201_05555_b200 import workloads as wl
    _build.build()
    _lib.load()
    # weak scaling: each rank owns an independent batch (distinct seed)
    wr = wl.config(w.name, seed=w.seed + rank) if world > 1 else w
    m = fom_measure(args, wr, world, local_rank, e2e_steps=args.e2e_steps or None)
    if rank != 0:
        tdist.destroy_process_group()
        return
    cpu = ref_p1 = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_rate(w)
        ref_p1 = reference_p1_rate(w)
    line = {
        "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": world, "steps": m["steps"],
        "warmup": m["warmup"], "ms_per_step": m["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": bench_config(w, world),
        "roofline": m["roofline"], "kernel_share_of_step": 1.0, "e2e": m["e2e"],
        "gpu_launches": m["gpu_launches"], "clocks": m["clocks"], "cpu_baseline": cpu,
        "reference_p1": ref_p1, "host": host_info(), "instance_groups": m["instance_groups"],
    }
    if world == 1 and not args.no_rom:
        # the other BASELINE configs on the same GPU, reported beside the
        # headline (each with its own roofline, e2e and CPU row)
        torch.cuda.empty_cache()
        others = {}
        for name in ("C1", "C5"):
            if name == w.name:
                continue
            wo = wl.config(name)
            mo = fom_measure(args, wo, 1, local_rank, steps=(50 if name == "C1" else 5),
                             clocks_soak=False)
            mo["config"] = bench_config(wo, 1)
            if not args.no_cpu_baseline and name == "C1":
                mo["cpu_baseline"] = cpu_oracle_rate(wo, seconds=5.0, max_steps=200)
            others[name] = mo
            torch.cuda.empty_cache()
        sys.path.insert(0, str(ROOT / "tools"))
        import bench_rom
        for name in ("C3", "C4"):
            others[name] = bench_rom.measure(name, steps=5, warmup=2,
                                             cpu=not args.no_cpu_baseline)
            torch.cuda.empty_cache()
        line["other_configs"] = others
        line["reduced_step"] = others["C3"]
    print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--soak-seconds", type=float, default=0.25,
                    help="untimed steps right before the timed block (clocks sampled under this load); "
                         "0.25 s = the length of a whole C5 run, 8 x a C2 run: the burst regime the "
                         "BASELINE configs themselves run in and MEASURED_PEAKS' copy bandwidth is quoted in")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rom", action="store_true",
                    help="skip the other-config sections (C1/C5 FOM, C3/C4 reduced)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    from paper_2201_05555_b200 import workloads as wl
    w = wl.config(args.config)
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        run_reference(args, w, rank, world)
    else:
        run_ours(args, w, rank, world, local_rank)


if __name__ == "__main__":
    main()
