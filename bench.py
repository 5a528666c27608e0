#!/usr/bin/env python
"""Benchmark: FP64 ADI cell-updates/s (incl. Picard iterations) and % of the
HBM roofline (BASELINE.json metric) on configs[3] -- the large grid
Nr=8192 x Nz=16384, fixed dt 1e-5 -- one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W]
  python bench.py --impl reference   # the reference's own CPU AdiStepper

The kernels are bit-identical to the reference AdiStepper. A "step" is one
accepted ADI time step (AdiStepper::step, solver.cpp:356-373) of the whole
grid. Cell-updates count every half-step attempt's active cells x Picard
iterations. Multi-GPU (torchrun, N > 1): the z-slab / r-slab
partitioned stepper (run_partitioned) over the N GPUs -- total work fixed,
strong scaling; time is the max over ranks.

The CPU numbers (the reference arm and this arm's cpu_baseline) are the
reference's own AdiStepper on the FULL configs[3] grid with bench.cpp:12-25
semantics: one untimed warm-up step, then two timed step() calls on a
LinePool of all host cores; plus a 1-worker row on a z-slice.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}  # B200_PROFILING.md fallback


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return PEAKS_FALLBACK["hbm_gbs"], "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML every
    20 ms when pynvml can open the device, else nvidia-smi every 200 ms."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._nvml = self._open_nvml(index)
        self._t = threading.Thread(target=self._run, daemon=True)

    @staticmethod
    def _open_nvml(index):
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            try:
                uuid = "GPU-" + str(torch.cuda.get_device_properties(index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid.encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown,
                    pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwPowerCap]
            return pynvml, h, float(mx), bits
        except Exception:
            return None

    def _sample_nvml(self):
        nv, h, mx, bits = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.samples.append([str(sm), str(mx), hex(r)] +
                            ["Active" if r & b else "Not Active" for b in bits])

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.02 if self._nvml else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "via": "nvml" if self._nvml else "nvidia-smi"}


_REAL_STDOUT = None


def claim_stdout():
    """Keep stdout for the one JSON line: everything else written to fd 1 by
    this process or its libraries (NCCL prints its version banner there)
    goes to stderr."""
    global _REAL_STDOUT
    if _REAL_STDOUT is None:
        sys.stdout.flush()
        _REAL_STDOUT = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    data = (json.dumps(line) + "\n").encode()
    if _REAL_STDOUT is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        sys.stdout.flush()
        os.write(_REAL_STDOUT, data)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_sample_case(case, nz_sample: int):
    """A z-truncated slice of the workload (same radial lines, materials, tau)."""
    from paper_1912_03744_b200 import configs
    return configs.scaled(case, case.gridspec.radial_divisions, nz_sample,
                          name=case.name + f"-z{nz_sample}")


def run_reference_cpu(case, steps: int, warmup: int, nz_sample, workers: int):
    """The reference's own AdiStepper (oracle/_ref, compiled from its sources)
    on a LinePool of `workers` threads: `warmup` untimed + `steps` timed step()
    calls (bench.cpp:12-25 semantics) on the full grid (nz_sample None) or a
    z-truncated sample."""
    from oracle.oracle import RefStepper, ref_available, PortStepper
    from paper_1912_03744_b200.solver import make_field
    sample = case if nz_sample is None else cpu_sample_case(case, nz_sample)
    g = sample.grid()
    if ref_available():
        stepper, kind = RefStepper(sample, workers=workers), "reference"
    else:
        stepper, kind, workers = PortStepper(sample), "port", 1
    f = make_field(g, sample.solver.T0)
    t = 0.0
    if warmup:
        t, _, _ = stepper.run(f, t, warmup)
    t0 = time.perf_counter()
    t_end, stats, _ = stepper.run(f, t, steps)
    dt = time.perf_counter() - t0
    what = (f"the full {g.nr()}x{g.nz()} {case.name} grid" if nz_sample is None else
            f"{g.nr()}x{g.nz()} z-slice of {case.name} (same radial lines, materials, tau)")
    return {"value": stats["cell_updates"] / dt, "unit": "cell-updates/s", "cores": workers,
            "kind": kind, "seconds": dt,
            "sample": f"{what}, {warmup} warm-up + {steps} timed step() calls "
                      f"(bench.cpp:12-25), {stats['cell_updates']:.3e} cell-updates"}


def cpu_rows(case, nz_sample=None):
    """The CPU baseline of both arms: all host cores on the full grid, and a
    1-worker row on a 1024-row z-slice (bounded run time). nz_sample: a
    z-slice instead of the full grid (the CPU test suite's quick check)."""
    full = run_reference_cpu(case, 2, 1, nz_sample, os.cpu_count() or 1)
    one = run_reference_cpu(case, 1, 0, min(1024, nz_sample or 1024), 1)
    keys = ("value", "unit", "cores", "kind", "sample")
    out = {k: full[k] for k in keys}
    out["one_worker"] = {k: one[k] for k in keys}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-nz", type=int, default=None,
                    help="CPU legs on a z-slice of this many rows (tests); default the full grid")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-supp", action="store_true",
                    help="skip the supplementary configs[1] batched-Thomas measurement")
    ap.add_argument("--partitioned", action="store_true",
                    help="run the partitioned (multi-GPU) stepper even at world size 1 "
                         "(under torchrun: a 1-rank NCCL communicator; validation of that path)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    claim_stdout()

    from paper_1912_03744_b200 import configs
    case = configs.CONFIGS[args.config]()
    grid_desc = {"workload": f"{case.name}: Nr={case.grid().nr()} x Nz={case.grid().nz()} FP64, "
                             f"fixed dt {case.timing.t_src / case.solver.tau_source_divisor:g} s, "
                             "4-layer cryogenic cell, power-law tables (SURVEY 8.0)"}
    metric = "FP64 ADI cell-updates/s (incl. Picard iters)"

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_rows(case, args.cpu_nz)
        line = {"impl": "reference", "metric": metric, "value": r["value"],
                "unit": "cell-updates/s", "n_gpus": args.gpus, "steps": 2,
                "warmup": 1, "higher_is_better": True, "dtype": "f64",
                "data": "synthetic",
                "config": dict(grid_desc, parallelism=f"cpu LinePool x{r['cores']}",
                               note="bench.cpp semantics: 1 untimed warm-up + 2 timed steps "
                                    "of the full grid, whatever --steps/--warmup say"),
                "cpu_baseline": r,
                "e2e": {"value": r["value"], "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        emit(line)
        return

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    pg = None
    if world > 1 or args.partitioned:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        pg = dist

    g = case.grid()
    nr, nz = g.nr(), g.nz()
    active = g.active_cells()
    if world > 1 or args.partitioned:
        run_partitioned(args, case, rank, world, local, pg, grid_desc, metric)
        pg.destroy_process_group()
        return
    stepper = gpu_stepper_for(case, local)
    field = torch.full((nz, nr), case.solver.T0, dtype=torch.float64, device=f"cuda:{local}").t()
    t = 0.0
    # warm-up steps (untimed)
    t, _, _ = stepper.run(field, t, args.warmup)
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(stepper.stream(), device=f"cuda:{local}")
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = stepper.launch_count()
    stepper.enable_kernel_timing(True)
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        t_end, stats, _ = stepper.run(field, t, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = stepper.launch_count() - launches0
    # how the steps were driven: speculative batches (one host read per batch)
    # on this grid; the resident stepper on grids of <= one line block per SM
    spec = {"speculative": stepper.speculation_stats(), "resident": stepper.resident_stats()}
    kernels_desc = stepper.describe()
    kt = stepper.kernel_timing()
    stepper.enable_kernel_timing(False)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if pg:
        pg.all_reduce(ms_t, op=pg.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    updates = stats["cell_updates"] * world
    value = updates / (ms_max / 1e3)

    # Roofline of the dominant kernel: per-launch algorithmic bytes
    # (active cells x 32 B per cell-update) / mean launch time.
    peak, peak_kind = load_peaks()
    sweeps = {"radial": (kt["radial_ms"], kt["radial_launches"]),
              "axial": (kt["axial_ms"], kt["axial_launches"])}
    dom = max(sweeps, key=lambda k: sweeps[k][0])
    dom_ms, dom_n = sweeps[dom]
    per_launch_bytes = active * 32.0
    achieved = per_launch_bytes / (dom_ms / max(dom_n, 1) / 1e3) / 1e9 if dom_n else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f).get(f"{args.config}:exact:{dom}")
        if tr:
            traffic = tr["dram_bytes_per_launch"] / 1e9
            # Picard iteration 1 of every half-step attempt stages the anchor
            # once (iterate == anchor) and moves fewer bytes: weight the
            # per-launch traffic by the launches of each kind in the timed region
            first = tr.get("dram_bytes_first_iteration")
            n1 = stats["steps"] + stats["halvings"]
            if first and dom_n >= n1 > 0:
                traffic = (n1 * first / 1e9 + (dom_n - n1) * traffic) / dom_n

    # e2e through the reference-facing C-ABI with HOST buffers: pcgpu_step_host
    # copies the field H2D, steps, copies D2H every step.
    e2e = None
    if not args.no_e2e:
        host = np.asfortranarray(field.t().contiguous().cpu().numpy().T)
        host_pinned = torch.from_numpy(np.ascontiguousarray(host.T)).pin_memory()
        hp = host_pinned.numpy().T  # (nr, nz) F-ordered view of pinned memory
        n_e2e = max(1, min(args.steps, 3))
        r = stepper.step(hp, t_end)  # untimed: allocates the host-path staging buffer
        t_end += r.tau_used
        upd = 0.0
        if pg:
            pg.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        te = t_end
        for _ in range(n_e2e):
            r = stepper.step(hp, te)
            te += r.tau_used
            upd += active * (r.radial.iterations + r.axial.iterations)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
        if pg:
            pg.all_reduce(e_ms, op=pg.ReduceOp.MAX)
        e2e = {"value": upd * world / (float(e_ms.item()) / 1e3), "unit": "cell-updates/s",
               "h2d_bytes_per_step": nr * nz * 8, "d2h_bytes_per_step": nr * nz * 8,
               "steps": n_e2e, "api": "pcgpu_step_host (C-ABI, host field)",
               "copy_in_overlap": stepper.pipeline_stats()}

    # Supplementary: a simulation through the package's device-resident runner
    # (runner.evolve), the way a user runs many steps: the host
    # field goes in once, every step hands the probe values back to the host,
    # the final field comes back once; both copies are inside the timed region.
    e2e_runner = None
    if not args.no_e2e and world == 1:
        from paper_1912_03744_b200.runner import ProbeSpec, RunnerConfig, evolve
        k_run = max(3, args.steps)
        rcfg = RunnerConfig(t_end=k_run * r.tau_used,
                            probes=[ProbeSpec(0.5e-3, 5e-3), ProbeSpec(1.2e-3, 10e-3)],
                            snapshot_pre_on=False, snapshot_post_off=False)
        dev_field = torch.empty((nz, nr), dtype=torch.float64, device=f"cuda:{local}")
        stepper.enable_kernel_timing(True)  # counts the Picard iterations that ran
        torch.cuda.synchronize()
        # copies and events on torch's stream (the pinned buffer must not be
        # tied to the stepper's stream, which dies with the stepper); evolve
        # blocks the host, so e1 is recorded after it
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        dev_field.copy_(host_pinned, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        res = evolve(stepper, case.timing, dev_field.t(), rcfg.t_end, rcfg)
        host_pinned.copy_(dev_field, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        kt = stepper.kernel_timing()
        stepper.enable_kernel_timing(False)
        r_ms = e0.elapsed_time(e1)
        e2e_runner = {"value": active * (kt["radial_launches"] + kt["axial_launches"]) /
                      (r_ms / 1e3), "unit": "cell-updates/s", "steps": res.steps,
                      "h2d_bytes_total": nr * nz * 8, "d2h_bytes_total": nr * nz * 8,
                      "d2h_bytes_per_step": 8 * len(rcfg.probes),
                      "api": "runner.evolve (pcgpu_evolve: field resident, probes per step)"}

    # Supplementary: configs[1], 131072 x 1024 batched Thomas solves in both
    # layouts (tools/bench_tridiag.py: CUDA events; their parity is tested in
    # tests/test_gpu_parity.py). A parity case, not the bench workload.
    supp = None
    if rank == 0 and world == 1 and not args.no_supp:
        from tools.bench_tridiag import run as run_tridiag
        del stepper
        torch.cuda.empty_cache()
        tri = run_tridiag()
        supp = {"cfg1_tridiag": {"unit": "ms per batched solve (131072 x 1024)",
                                 "parity": "bit-identical per system (tests/test_gpu_parity.py)",
                                 **{k: {kk: v[kk] for kk in ("ms", "GBps_algorithmic",
                                                           "rows_per_s")}
                                    for k, v in tri.items()}}}
        stepper = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        del stepper, field
        torch.cuda.empty_cache()
        cpu = cpu_rows(case, args.cpu_nz)

    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(grid_desc, kernels=kernels_desc,
                           parity="bit-identical to the reference",
                           parallelism=f"replicas x{world}",
                           l2="inputs > L2 (1 GiB FP64 fields)",
                           picard={"radial_iters": stats["radial_iterations"],
                                   "axial_iters": stats["axial_iterations"],
                                   "halvings": stats["halvings"], "steps": stats["steps"]},
                           controller=spec),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "GB per launch (ncu dram__bytes_read+write; mean over the timed launches)",
                         # the same launch time against the DRAM bytes it really moves
                         # (80 B per cell: the exact Thomas working set)
                         "traffic_frac": (traffic / (dom_ms / max(dom_n, 1) / 1e3) / peak
                                          if traffic and dom_n else None),
                         "kernel": f"{dom} Picard iteration",
                         "bytes_per_launch": per_launch_bytes, "launches": dom_n,
                         "ms_per_launch": dom_ms / max(dom_n, 1), "peak_kind": peak_kind,
                         "other_sweep_ms_per_launch": {k: v[0] / max(v[1], 1) for k, v in
                                                       sweeps.items()}},
            "cpu_baseline": cpu, "e2e": e2e, "e2e_runner": e2e_runner, "clocks": clk.summary(),
            "gpu_launches": launches, "supplementary": supp,
        }
        emit(line)
    if pg:
        pg.destroy_process_group()


def run_partitioned(args, case, rank, world, local, pg, grid_desc, metric):
    """configs[3] partitioned over `world` GPUs: z-slabs for the radial sweep,
    NCCL all-to-all transpose to r-slabs for the axial sweep, NCCL allreduce
    of the Picard norm. Total work is fixed: strong scaling."""
    import torch
    from paper_1912_03744_b200.configs import make_source
    from paper_1912_03744_b200.dist import PartitionedAdi, share_unique_id
    g = case.grid()
    dev = torch.device(f"cuda:{local}")
    uid = share_unique_id(rank, dev)
    part = PartitionedAdi(g, case.materials, make_source(case, g), case.timing, case.solver,
                          device=local, rank=rank, world=world, unique_id=uid)
    if os.environ.get("PCGPU_DIST_TRANSPORT", "peer") != "nccl":
        part.enable_peer_transport()  # fused K3/K4 + peer stores over NVLink
    field = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device=dev).t()
    part.set_field(field)
    t, _, _ = part.run(0.0, args.warmup)
    stream = torch.cuda.ExternalStream(part.stream(), device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    l0 = part.launch_count()
    pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        t_end, stats, _ = part.run(t, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    pg.barrier()
    ms_t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    pg.all_reduce(ms_t, op=pg.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    launches = part.launch_count() - l0
    # transpose time, measured separately (synchronising events per transpose)
    part.enable_timing(True)
    part.run(t_end, 1)
    tm = part.timing()
    tr = torch.tensor([tm["transpose_ms"] / max(tm["transposes"], 1)], dtype=torch.float64,
                      device=dev)
    pg.all_reduce(tr, op=pg.ReduceOp.MAX)
    # every rank counts the whole grid's cell-updates (the norm is global)
    value = stats["cell_updates"] / (ms_max / 1e3)
    # Roofline per GPU over the whole step (the partitioned stepper has no
    # per-kernel timers): SURVEY 8(d)'s algorithmic bytes, 32 B per
    # cell-update plus 16 B per cell and attempt for the explicit passes.
    peak, peak_kind = load_peaks()
    alg = 32.0 * stats["cell_updates"] + 16.0 * stats["attempt_cells"]
    achieved = alg / world / (ms_max / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                "kernel": "whole partitioned step per GPU (algorithmic bytes / step time)"}

    # e2e through the partitioned stepper's host-field entry points: every
    # step each rank copies its state lines (1/world of the field) in from
    # pinned host memory and back out, over its own PCIe link
    e2e = None
    if not args.no_e2e:
        part.enable_timing(False)
        host_t = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64).pin_memory()
        hp = host_t.numpy().T  # (nr, nz) Fortran view of pinned memory
        part.get_field_host(hp)
        n_e2e = max(1, min(args.steps, 3))
        te = t_end
        part.set_field_host(hp)  # untimed first pass (page-in of the pinned buffer)
        te, _, _ = part.run(te, 1)
        part.get_field_host(hp)
        pg.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        upd = 0.0
        for _ in range(n_e2e):
            part.set_field_host(hp)
            te, st1, _ = part.run(te, 1)
            part.get_field_host(hp)
            upd += st1["cell_updates"]
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        pg.all_reduce(e_ms, op=pg.ReduceOp.MAX)
        e2e = {"value": upd / (float(e_ms.item()) / 1e3), "unit": "cell-updates/s",
               "h2d_bytes_per_step": g.nr() * g.nz() * 8, "d2h_bytes_per_step": g.nr() * g.nz() * 8,
               "steps": n_e2e,
               "api": "pcgpu_dist_set_field_host / run / get_field_host (C-ABI, host field; "
                      "each rank moves its 1/N of the field)"}
    if rank == 0:
        z0, z1, r0, r1 = part.slabs()
        line = {
            "metric": metric, "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(grid_desc, parallelism=f"z-slab/r-slab x{world}",
                           transport=part.transport(),
                           l2="inputs > L2", rank0_slabs={"z": [z0, z1], "r": [r0, r1]},
                           picard={"radial_iters": stats["radial_iterations"],
                                   "axial_iters": stats["axial_iterations"],
                                   "halvings": stats["halvings"]}),
            "transpose": {"ms_per_transpose_max_rank": float(tr.item()),
                          "transposes_per_step": 3,
                          "fields_per_step": 4,
                          "bytes_per_rank_per_step":
                              4 * 8 * g.nr() * g.nz() // world * (world - 1) // world},
            "roofline": roofline, "clocks": clk.summary(), "gpu_launches": launches, "e2e": e2e,
        }
        emit(line)


def gpu_stepper_for(case, device):
    from paper_1912_03744_b200.configs import make_source
    from paper_1912_03744_b200.solver import AdiStepper, DevicePlan
    g = case.grid()
    return AdiStepper(g, case.materials, make_source(case, g), case.timing, case.solver,
                      DevicePlan(device=device))


if __name__ == "__main__":
    main()
