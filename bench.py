#!/usr/bin/env python
"""Benchmark: FP64 real-space force evaluations, atom-steps/s (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl mine|reference]

A "step" is one real-space force evaluation of the configured workload with
the neighbour lists rebuilt every 20 steps inside the timed region (K = 20
gives exactly one rebuild + 20 evaluations, the config-4 recipe). Default
workload: BASELINE.json config 4 (333,333 rigid 3-site waters, 999,999
atoms, L = 215.3 A: Halgren vdW on H-reduced sites at 9 A + real-space
multipole Ewald (alpha 0.5446) at 7 A + Ewald/Thole permanent field + PCG
induced dipoles to 1e-5 D), which fits one B200 and is the config the
1/2/4/8-GPU metric is quoted on. Synthetic seeded inputs (no dataset).

`value` is device-resident throughput (inputs already in HBM; CUDA events on
the engine stream around the K steps); `e2e` is the same through the C ABI
with host buffers (page-locked, public `host_array`): every step uploads the
coordinates (H2D) and reads back forces and energies (D2H). The roofline
comes from the same K steps run again with CUDA events around every launch
(kernel durations on their own stream) plus a one-stream pass for the
kernels of the step's low-priority second stream. `--impl reference` times
the reference's own CPU implementation (oracle/_ref + the closed-form port
for kernels it lacks) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REBUILD_EVERY = 20
METRIC = "FP64 real-space force evals/sec (atom-steps/s) & % FP64 peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-md", action="store_true",
                    help="skip the extra timing of device-resident MD steps")
    ap.add_argument("--no-polar-forces", action="store_true",
                    help="skip the extra timing of the step with polarization forces")
    ap.add_argument("--no-recip", action="store_true",
                    help="skip the extra timing of the step with reciprocal-space Ewald")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--dd-nccl", action="store_true",
                    help="run the decomposed NCCL path even at one rank (under torchrun "
                         "--nproc-per-node 1): a self-test of the multi-GPU code path")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if p[5 + k].lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload
class Workload:
    def __init__(self, config: int, device: int, seed: int):
        import paper_1906_01211_b200 as m
        self.m = m
        self.config = config
        c = m.CONFIGS[config]
        self.c = c
        self.sys = m.water_box(c["n_mol"], c["box"], seed, c["model"])
        self.n = self.sys.n_sites
        self.eng = m.Engine(self.n, device=device)
        self.eng.upload_system(self.sys)
        if c["model"] == "charmm":
            self.p = m.CharmmParams(c["cutoff"], c["alpha"], m.ELECTRIC, 0, 1)
            self.lists = [(c["cutoff"] + c["skin"], 0, m.SITES_ATOMIC)]
        else:
            terms = {1: m.TERM_VDW | m.TERM_MPOLE, 2: m.TERM_POLAR}.get(
                config, m.TERM_VDW | m.TERM_MPOLE | m.TERM_POLAR)
            self.p = m.AmoebaParams(c["vdw_cutoff"], 0.07, 0.12, c["elec_cutoff"], c["alpha"],
                                    m.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
            self.lists = [(c["elec_cutoff"] + c["skin"], 0, m.SITES_ATOMIC)]
            if terms & m.TERM_VDW:
                self.lists.append((c["vdw_cutoff"] + c["skin"], 1, m.SITES_VDW))
        self.tables = {}
        self.rebuild()

    def rebuild(self):
        for cut, lid, sites in self.lists:
            self.tables[lid] = self.eng.build_neighbor_table(cut, list_id=lid, sites=sites)

    def step(self):
        if self.c["model"] == "charmm":
            self.eng.charmm_step(self.tables[0], self.p)
        else:
            vdw = self.tables.get(1, self.tables[0])
            self.eng.amoeba_step(vdw, self.tables[0], self.p)

    def run(self, steps: int):
        for k in range(steps):
            if k % REBUILD_EVERY == 0:
                self.rebuild()
            self.step()

    # roofline: (kernel name) -> ("fp64", flops) | ("hbm", bytes) per launch
    def algorithmic_work(self, kernel: str):
        from paper_1906_01211_b200.flops import PAIRS_OF, PER_PAIR_FLOPS, stream_bytes
        if kernel not in PAIRS_OF:
            return None
        role, key, excl = PAIRS_OF[kernel]
        lid = 1 if role == "vdw" else 0
        directed, _ = self.eng.count_within(self.tables[lid], self.c[key], excl)
        if kernel in PER_PAIR_FLOPS:
            return "fp64", PER_PAIR_FLOPS[kernel] * directed / 2.0
        return "hbm", stream_bytes(kernel, self.n, directed)


def fft_size(x: float) -> int:
    """Smallest 2^a 3^b 5^c >= x (cuFFT-friendly grid)."""
    n = max(8, int(np.ceil(x)))
    while True:
        k = n
        for p in (2, 3, 5):
            while k % p == 0:
                k //= p
        if k == 1:
            return n
        n += 1


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# launched on the AMOEBA step's low-priority second stream
AUX_KERNELS = {"halgren", "chain_rule", "mpole"}


def md_timing(wl, steps, barrier, device, respa=False, aspc=False):
    """K steps of the workload on the device (mdg_md_run): ms/step and
    ns/day (flexible water: harmonic O-H bonds and H-O-H angles; AMOEBA runs
    include the polarization forces). Velocity Verlet at dt = 0.5 fs, or
    (respa) BAOAB-RESPA at the paper's 2 fs outer step with
    the bonded terms in 4 inner steps of 0.5 fs and a 1/ps Langevin bath at
    300 K. aspc: the AMOEBA PCG starts from the ASPC-extrapolated dipoles
    (the paper's Beeman/ASPC setup) instead of alpha E."""
    m = wl.m
    eng = wl.eng
    n_mol = wl.n // 3
    mass = np.tile([15.999, 1.008, 1.008], n_mol)
    rng = np.random.default_rng(7)
    vel = rng.normal(size=(wl.n, 3)) * np.sqrt(0.0019872041 * 300.0 * 4.184e-4 / mass)[:, None]
    bonds = np.stack([np.repeat(np.arange(n_mol) * 3, 2),
                      (np.arange(n_mol)[:, None] * 3 + np.array([1, 2])).ravel()], 1)
    angles = np.stack([np.arange(n_mol) * 3 + 1, np.arange(n_mol) * 3, np.arange(n_mol) * 3 + 2], 1)
    eng.upload_bonded(bonds, 529.6, 0.9572, angles, 34.05, np.deg2rad(104.52))
    eng.upload_velocities(vel, mass)
    c = wl.c
    dt = 0.5
    if c["model"] == "charmm":
        p = m.MDParams(0, steps, dt, 20, 0, 1, c["cutoff"] + c["skin"], 0.0, 1)
        kw = {"charmm": wl.p}
    else:
        ap = m.AmoebaParams(*[getattr(wl.p, f) for f, _ in wl.p._fields_])
        if ap.terms & m.TERM_POLAR:
            ap.terms |= m.TERM_POLAR_FORCE
        # the static fixture's random lab-frame dipoles / quadrupoles are too
        # strong for dynamics (H...O collapse within ~25 fs); MD carries them
        # at 1/10 in local water frames (rotating with the molecules, torques
        # on), which conserves energy (tests/test_md_integrator.py)
        n = wl.n
        frame = np.zeros(n, np.int32)
        za = np.zeros(n, np.int32)
        xa = np.zeros(n, np.int32)
        o = np.arange(0, n, 3)
        frame[o], za[o], xa[o] = 2, o + 1, o + 2
        frame[o + 1], za[o + 1], xa[o + 1] = 1, o, o + 2
        frame[o + 2], za[o + 2], xa[o + 2] = 1, o, o + 1
        eng.upload_frames(frame, za, xa, 0.1 * np.asarray(wl.sys.dipole),
                          0.1 * np.asarray(wl.sys.quadrupole))
        p = m.MDParams(1, steps, dt, 20, 0, 1, c["elec_cutoff"] + c["skin"],
                       c["vdw_cutoff"] + c["skin"], 1)
        kw = {"amoeba": ap}
    if aspc and c["model"] != "charmm":
        p.predictor = m.PREDICT_ASPC
    if respa:
        dt = p.dt_fs = 2.0
        p.integrator = m.INTEGRATOR_BAOAB_RESPA
        p.inner_steps = 4
        p.friction_ps = 1.0
        p.temperature_k = 300.0
        p.seed = 7
        p.rebuild_every = 5  # the same 10 fs between list rebuilds
    warm = m.MDParams(*[getattr(p, f) for f, _ in p._fields_])
    warm.nsteps = 2
    eng.md_run(warm, energies=False, **kw)
    if barrier:
        barrier()
    eng.synchronize()
    r0 = eng.md_rebuild_count()
    eng.timer_start()
    eng.md_run(p, energies=False, **kw)
    mms = eng.timer_stop()
    rebuilds = eng.md_rebuild_count() - r0
    last_iters = int(eng.fetch_energies()[2]) if c["model"] != "charmm" else None
    # (NVE conservation of both integrators and models is tested in
    # tests/test_md_integrator.py and tests/test_gpu_parity.py)
    what = ("device BAOAB-RESPA (outer: these forces; inner x4: flexible-water bonds/angles; "
            "Langevin 1/ps, 300 K)" if respa else
            "device velocity Verlet with these forces + flexible-water bonds/angles")
    if p.predictor:
        what += "; ASPC dipole predictor"
    return {"what": what + ("" if c["model"] == "charmm" else
                            " + polarization forces; multipoles x0.1 in local water frames"),
            "dt_fs": dt, "steps": steps, "ms_per_step": mms / steps,
            "pcg_iters_last_step": last_iters,
            # incl. the one at the start of the call; more than steps /
            # rebuild_every + 1 when sites moved fast (motion-triggered)
            "list_rebuilds": rebuilds, "rebuild_every": p.rebuild_every,
            "ns_per_day": steps * dt * 1e-6 / (mms * 1e-3) * 86400.0}


def ncu_traffic(name):
    """DRAM bytes per launch of `name` from the committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)["kernels"].get(name)
    except (OSError, KeyError, ValueError):
        return None


def ncu_executed(name):
    """ncu-measured executed FP64 rate of `name` (profiles/ncu_fp64_executed.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_fp64_executed.json")) as f:
            return json.load(f)["kernels"].get(name)
    except (OSError, KeyError, ValueError):
        return None


def fp64_step_fraction(config, ms_per_step, pcg_iters, steps, peak_tflops, n_gpus):
    """The metric's "% FP64 peak" at the step level: executed FP64 flops of one
    config-4 step (ncu dadd + dmul + 2 dfma over every kernel of the step,
    profiles/r2_ncu_fp64_step.json: fixed part + per PCG iteration x this
    run's iterations + the list rebuild / 20) / the measured step time / the
    FP64 peak of the GPUs used (the single-GPU count: halo work that
    N > 1 domains repeat is not counted)."""
    if config != 4:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_fp64_step.json")) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    rebuilds = -(-steps // REBUILD_EVERY)
    flops = (d["per_eval_fixed_flops"] + d["per_pcg_iteration_flops"] * pcg_iters
             + d["per_rebuild_flops"] * rebuilds / steps)
    achieved = flops / (ms_per_step * 1e-3) / 1e12
    peak = peak_tflops * n_gpus
    return {"executed_flops_per_step": flops, "achieved_tflops": round(achieved, 3),
            "peak_tflops": round(peak, 3), "frac": round(achieved / peak, 4),
            "source": "profiles/r2_ncu_fp64_step.json (ncu --metrics, HEAD of round 2)"}


def roofline_of(wl, name, cnt, tot_ms, step_ms, fp64_peak):
    work = wl.algorithmic_work(name)
    if work is None:
        return None
    avg_ms = tot_ms / cnt
    kind, amount = work
    if kind == "fp64":
        achieved = amount / (avg_ms * 1e-3) / 1e12
        peak, unit, src = fp64_peak, "TFLOP/s", "measured DFMA probe in this run (of measured)"
    else:
        achieved = amount / (avg_ms * 1e-3) / 1e9
        peak, src = hbm_peak()
        unit = "GB/s"
    return {"bound": "fp64" if kind == "fp64" else "hbm", "kernel": name,
            "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": ncu_traffic(name),
            "avg_launch_ms": round(avg_ms, 4), "peak_source": src,
            ("flops_per_launch" if kind == "fp64" else "bytes_per_launch"): amount,
            "share_of_step": round(tot_ms / step_ms, 4),
            "ncu_executed_fp64": ncu_executed(name)}


def run_mine(args, world, rank, local):
    import paper_1906_01211_b200 as m
    device = local
    wl = Workload(args.config, device, args.seed + rank)
    eng = wl.eng
    peak = m.fp64_peak_tflops(device)
    for _ in range(args.warmup):
        wl.step()
    wl.rebuild()

    barrier = None
    if world > 1:
        import torch.distributed as dist
        barrier = dist.barrier
    # ---- device-resident timed region (no per-launch profiling events: at
    # the small configs their host cost would starve the GPU)
    if barrier:
        barrier()
    eng.synchronize()
    launches0 = eng.launch_count()
    with ClockSampler(device) as clk:
        eng.timer_start()
        wl.run(args.steps)
        ms = eng.timer_stop()
    launches = eng.launch_count() - launches0
    # ---- the same K steps again with CUDA events bracketing every launch
    # (on the stream it runs on): per-kernel durations for the roofline
    eng.synchronize()
    eng.profile_reset()
    eng.profile(True)
    eng.timer_start()
    wl.run(args.steps)
    prof_ms = eng.timer_stop()
    eng.profile(False)
    prof = eng.profile_report()
    if barrier:
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    energies, virial, iters, rms = eng.fetch_energies()

    # ---- serial profiling pass (one stream): per-kernel durations without
    # the overlap of the step's second stream (the low-priority Halgren /
    # multipole chain stretches over the gaps of the critical path, so its
    # event durations inside the timed region are not kernel times)
    eng.set_overlap(False)
    eng.synchronize()
    eng.profile_reset()
    eng.profile(True)
    eng.timer_start()
    wl.run(args.steps)
    serial_ms = eng.timer_stop()
    eng.profile(False)
    prof_serial = eng.profile_report()
    eng.set_overlap(True)

    # ---- roofline of the dominant kernel (+ every pair kernel, for the record):
    # main-stream kernels from the profiled pass, aux-stream ones from the
    # serial pass; dominance by serial total time
    ranked = sorted(prof_serial.items(), key=lambda kv: -kv[1][1])
    roof = None
    others = {}
    for name, (cnt_s, tot_s) in ranked:
        src = prof_serial if name in AUX_KERNELS or name not in prof else prof
        cnt, tot_ms = src[name]
        r = roofline_of(wl, name, cnt, tot_ms, serial_ms if src is prof_serial else prof_ms, peak)
        if r is None:
            continue
        r["timing"] = "serial pass" if src is prof_serial else "profiled pass (two streams)"
        if roof is None:
            roof = r
        else:
            others[name] = {k: r[k] for k in ("bound", "achieved", "unit", "frac",
                                              "avg_launch_ms", "share_of_step",
                                              "ncu_executed_fp64", "timing")}

    m_host_array = wl.m.host_array
    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        # the step's host buffers live in page-locked memory (the public
        # host_array): coordinates DMA'd in, forces DMA'd out, no staging copy
        xyz = m_host_array((3, wl.n))
        xyz[0], xyz[1], xyz[2] = wl.sys.x, wl.sys.y, wl.sys.z
        x, y, z = xyz[0], xyz[1], xyz[2]
        fbuf = m_host_array((3, wl.n))
        eng.set_force_output(fbuf)  # forces DMA'd while the PCG still runs
        for _ in range(2):
            eng.upload_positions(x, y, z)
            wl.step()
            eng.fetch_forces(out=fbuf)
        wl.rebuild()
        if barrier:
            barrier()
        eng.synchronize()
        t0 = time.perf_counter()
        eng.timer_start()
        for k in range(args.steps):
            eng.upload_positions(x, y, z)            # H2D 24 B/atom
            if k % REBUILD_EVERY == 0:
                wl.rebuild()
            wl.step()
            f = eng.fetch_forces(out=fbuf)           # D2H 24 B/atom
            e = eng.fetch_energies()                 # D2H energies/virial
        e2e_ms = eng.timer_stop()
        wall_ms = (time.perf_counter() - t0) * 1e3
        e2e_ms = max(e2e_ms, wall_ms)
        if barrier:
            import torch
            import torch.distributed as dist
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{device}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": world * wl.n * args.steps / (e2e_ms * 1e-3), "unit": "atom-steps/s",
               "h2d_bytes_per_step": 24 * wl.n, "d2h_bytes_per_step": 24 * wl.n + 8 * (4 + 9 + 2),
               "ms_per_step": e2e_ms / args.steps}
        del f, e

    # ---- 8(f)#1 extension, reported beside the headline (not in it): the
    # same step plus polarization forces/torques at the converged dipoles
    polar_forces = None
    m_ = wl.m
    if getattr(wl.p, "terms", 0) & m_.TERM_POLAR and not args.no_polar_forces:
        base = wl.p.terms
        wl.p.terms = base | m_.TERM_POLAR_FORCE
        wl.step()
        wl.rebuild()
        if barrier:
            barrier()
        eng.synchronize()
        eng.timer_start()
        wl.run(args.steps)
        pms = eng.timer_stop()
        wl.p.terms = base
        if barrier:
            import torch
            import torch.distributed as dist
            t = torch.tensor([pms], dtype=torch.float64, device=f"cuda:{device}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pms = float(t.item())
        polar_forces = {"what": "same step + polarization forces/torques (TERM_POLAR_FORCE)",
                        "value": world * wl.n * args.steps / (pms * 1e-3),
                        "unit": "atom-steps/s", "ms_per_step": pms / args.steps}

    # ---- 8(f)#3 extension, beside the headline: the same step with full
    # Ewald (reciprocal space for the multipoles and inside the PCG)
    with_recip = None
    if getattr(wl.p, "terms", 0) & m_.TERM_POLAR and not args.no_recip:
        grid = fft_size(wl.c["box"] / 1.0)
        eng.set_ewald_recip((grid, grid, grid), 5)
        try:
            wl.step()
            wl.rebuild()
            if barrier:
                barrier()
            eng.synchronize()
            eng.timer_start()
            wl.run(args.steps)
            rms_ = eng.timer_stop()
            er, _, ir, _ = eng.fetch_energies()
        finally:
            eng.set_ewald_recip((0, 0, 0))
        with_recip = {"what": f"same step + reciprocal-space Ewald (smooth PME {grid}^3, order 5: "
                              "multipole energy/forces/torques, the PCG right-hand side and "
                              "operator)", "value": world * wl.n * args.steps / (rms_ * 1e-3),
                      "unit": "atom-steps/s", "ms_per_step": rms_ / args.steps,
                      "pcg_iters": int(ir), "energies_kcal_mol": [float(v) for v in er[:3]]}

    # ---- 8(f)#4 extension, beside the headline: the same forces driving
    # device-resident MD (flexible water bonds/angles, 300 K start): velocity
    # Verlet at 0.5 fs, then BAOAB-RESPA at 2 fs; last, as it moves the
    # engine's coordinates
    md = md_respa = md_aspc = None
    if not args.no_md:
        eng.set_force_output(None)  # no per-step force DMA inside the MD loop
        md = md_timing(wl, args.steps, barrier, device)
        if wl.c["model"] != "charmm":
            md_aspc = md_timing(wl, args.steps, barrier, device, aspc=True)
        md_respa = md_timing(wl, args.steps, barrier, device, respa=True)

    out = {
        "metric": METRIC,
        "value": world * wl.n * args.steps / (ms * 1e-3),
        "unit": "atom-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",  # one fixed system; --gpus N splits it (DD)
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded 3-site water fixture, BASELINE.json generator rules)",
        "config": {"workload": f"BASELINE config {args.config}: {wl.c['n_mol']} waters "
                               f"({wl.n} atoms), L={wl.c['box']} A, "
                               + ("LJ + Ewald charge 9 A" if wl.c["model"] == "charmm" else
                                  "Halgren 9 A + multipole Ewald 7 A + Thole/Ewald PCG 1e-5 D"),
                   "n_atoms": wl.n, "rebuild_every": REBUILD_EVERY,
                   "parallelism": "1 GPU",
                   "l2": "inputs larger than L2 (lists > 126 MB)"},
        "e2e": e2e,
        "with_polar_forces": polar_forces,
        "with_ewald_recip": with_recip,
        "md": md,
        "md_aspc": md_aspc,
        "md_respa": md_respa,
        "gpu_launches": launches,
        "roofline": roof,
        "roofline_other_kernels": others,
        "clocks": clk.summary(),
        "energies_kcal_mol": [float(v) for v in energies[:3]],
        "pcg_iters": int(iters),
        "pcg_rms_debye": float(rms),
        "fp64_peak_tflops_measured": round(peak, 3),
        "fp64_step": fp64_step_fraction(args.config, ms / args.steps, int(iters), args.steps,
                                        peak, 1),
        # profiled pass (same K steps, events around every launch)
        "kernel_ms": {k: round(v[1] / max(v[0], 1), 4) for k, v in sorted(prof.items())},
        "kernel_share": {k: round(v[1] / prof_ms, 4) for k, v in sorted(prof.items())},
        "profiled_ms_per_step": prof_ms / args.steps,
        # one stream, same K steps: kernel-by-kernel durations and their sum
        "serial_pass": {"ms_per_step": serial_ms / args.steps,
                        "kernel_ms": {k: round(v[1] / max(v[0], 1), 4)
                                      for k, v in sorted(prof_serial.items())},
                        "kernel_share": {k: round(v[1] / serial_ms, 4)
                                         for k, v in sorted(prof_serial.items())}},
    }
    return out, wl


def run_dd(args, world, rank, local, backend, ndom):
    """Spatial domain decomposition of the configured box over `ndom` domains
    (strong scaling: the same system split N ways): one domain per rank over
    NCCL (backend "nccl", under torchrun), or all N domains in this process on
    one GPU (backend "local": N ranks emulated on the one device). The PCG
    exchanges halos and sums its scalars on the device every iteration
    (csrc/group.cu)."""
    import paper_1906_01211_b200 as m
    from paper_1906_01211_b200 import dd
    c = m.CONFIGS[args.config]
    s = m.water_box(c["n_mol"], c["box"], args.seed, c["model"])
    if c["model"] == "charmm":
        list_cut = c["cutoff"] + c["skin"]
        params = m.CharmmParams(c["cutoff"], c["alpha"], m.ELECTRIC, 0, 1)
        lists = [(list_cut, 0, m.SITES_ATOMIC)]
    else:
        list_cut = max(c["vdw_cutoff"], c["elec_cutoff"]) + c["skin"]
        terms = {1: m.TERM_VDW | m.TERM_MPOLE, 2: m.TERM_POLAR}.get(
            args.config, m.TERM_VDW | m.TERM_MPOLE | m.TERM_POLAR)
        params = m.AmoebaParams(c["vdw_cutoff"], 0.07, 0.12, c["elec_cutoff"], c["alpha"],
                                m.ELECTRIC, 0.39, 1e-5, 100, 1, terms)
        lists = [(c["elec_cutoff"] + c["skin"], 0, m.SITES_ATOMIC)]
        if terms & m.TERM_VDW:
            lists.append((c["vdw_cutoff"] + c["skin"], 1, m.SITES_VDW))
    halo = list_cut + 1.5
    size = world if backend == "nccl" else ndom
    g = dd.DomainGroup(s, size, halo, device=local, backend=backend, rank=rank,
                       list_cutoff=list_cut)
    assert g.check_halo(s), "halo exchange self-check failed"
    eng0 = g.domains[0].eng

    def step(tables):
        if c["model"] == "charmm":
            g.charmm_step(tables, params)
        else:
            g.amoeba_step(tables, params)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    tables = g.build_lists(lists)
    for _ in range(args.warmup):
        step(tables)
    barrier()
    eng0.synchronize()
    launches0 = g.launch_count()
    with ClockSampler(local) as clk:
        eng0.timer_start()
        for k in range(args.steps):
            if k % REBUILD_EVERY == 0:
                tables = g.build_lists(lists)
            step(tables)
        ms = eng0.timer_stop()
    launches = g.launch_count() - launches0
    ms = max_over_ranks(ms)
    en, w, iters, rms = g.energies()

    # ---- end to end through the public DD API: every step each domain
    # uploads its local coordinates (H2D; the halo then refreshed from the
    # owners by the group exchange), reads back its owned forces (D2H) and
    # the summed energies
    e2e = None
    if not args.no_e2e:
        x, y, z = np.asarray(s.x), np.asarray(s.y), np.asarray(s.z)
        for _ in range(2):
            g.update_positions(x, y, z)
            step(tables)
            g.owned_forces()
        tables = g.build_lists(lists)
        barrier()
        eng0.synchronize()
        t0 = time.perf_counter()
        eng0.timer_start()
        for k in range(args.steps):
            g.update_positions(x, y, z)
            if k % REBUILD_EVERY == 0:
                tables = g.build_lists(lists)
            step(tables)
            g.owned_forces()
            g.energies()
        e_ms = max(eng0.timer_stop(), (time.perf_counter() - t0) * 1e3)
        e_ms = max_over_ranks(e_ms)
        n_loc = sum(len(d.plan.local) for d in g.domains)
        n_own = sum(d.plan.n_owned for d in g.domains)
        e2e = {"value": g.n_global * args.steps / (e_ms * 1e-3), "unit": "atom-steps/s",
               "h2d_bytes_per_step": 24 * n_loc * (world if backend == "nccl" else 1),
               "d2h_bytes_per_step": 24 * n_own * (world if backend == "nccl" else 1)
               + 8 * (4 + 9) * size,
               "ms_per_step": e_ms / args.steps}
    p0 = g.plans[0]
    n_gpus = world if backend == "nccl" else 1
    out = {
        "metric": METRIC,
        "value": g.n_global * args.steps / (ms * 1e-3),
        "unit": "atom-steps/s",
        "n_gpus": n_gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded 3-site water fixture, BASELINE.json generator rules)",
        "config": {"workload": f"BASELINE config {args.config}: {c['n_mol']} waters "
                               f"({g.n_global} atoms), L={c['box']} A, spatial DD",
                   "n_atoms": g.n_global, "rebuild_every": REBUILD_EVERY,
                   "parallelism": f"spatial DD {'x'.join(map(str, p0.dims))} over {size} domains"
                                  + (f" (NCCL, {world} GPUs)" if backend == "nccl" else
                                     f" on 1 GPU (LOCAL group: {size} ranks emulated in one "
                                     "process; no multi-GPU scaling claim)"),
                   "halo_A": halo, "owned_sites_domain0": p0.n_owned,
                   "halo_sites_domain0": int(len(p0.halo)),
                   "l2": "inputs larger than L2 (lists > 126 MB)"},
        "domains": size,
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": None,
        "clocks": clk.summary(),
        "energies_kcal_mol": [float(v) for v in en[:3]],
        "pcg_iters": int(iters),
        "pcg_rms_debye": float(rms),
        "fp64_step": fp64_step_fraction(args.config, ms / args.steps, int(iters), args.steps,
                                        m.fp64_peak_tflops(local), n_gpus),
    }
    g.close()
    return out


def _cpu_curve():
    try:
        with open(os.path.join(ROOT, "profiles", "r2_cpu_cost_curve.json")) as f:
            d = json.load(f)
        return {"file": "profiles/r2_cpu_cost_curve.json", "cpu_model": d["cpu_model"],
                "us_per_atom_step": {str(r["n_atoms"]): round(r["us_per_atom_step"], 3)
                                     for r in d["rows"]}}
    except (OSError, KeyError, ValueError):
        return None


def _cpu_sample_text(r, threads):
    return (f"{'%d independent replicas' % threads if threads > 1 else 'one replica'} of a "
            f"{r['n_sample_atoms']}-atom box of the same generator/density (reference shards "
            f"model, proj/src/bench.cpp:330-360); per step: reference Vec list build/20 + "
            f"Halgren + {r['matvecs_per_step']} tmatxb (oracle/_ref, {r['isa']}), plus "
            f"multipoles + multipole field from the CPU restatement oracle/mdo_fast.c (not "
            f"reference: {100 * r['port_share']:.0f}% of the step); reference protocol: "
            f"{r['warmup']} warm-up, {r['repeats']} interleaved Scalar/Vec repeats, trimmed mean")


def cpu_baseline(args, pcg_iters):
    from oracle import cpu_reference
    threads = 1
    r = cpu_reference.run(args.config, threads, 3, 1, args.seed, matvecs=pcg_iters + 1)
    return {"value": r["value"], "unit": "atom-steps/s", "cores": threads, "kind": "reference",
            "sample": _cpu_sample_text(r, threads), "s_per_step": r["s_per_step"],
            "cpu_model": r["cpu_model"], "scalar_rel": r.get("scalar"),
            "size_curve": _cpu_curve()}


def run_reference(args, world, rank):
    """The reference's own CPU implementation of the path on all host cores
    (oracle/_ref Vec kernels; multipoles from the CPU restatement), same
    metric and unit as the GPU arm, on a bounded sample of the workload."""
    if rank != 0:
        return None
    from oracle import cpu_reference
    threads = os.cpu_count() or 1
    r = cpu_reference.run(args.config, threads, max(3, args.steps // 4), max(1, args.warmup // 3),
                          args.seed)
    cfg = {"workload": f"BASELINE config {args.config} (CPU sample: {r['n_sample_atoms']} "
                       f"atoms per replica; per-atom cost vs size in size_curve)",
           "threads": threads, "same_config": False}
    return {
        "metric": METRIC,
        "impl": "reference",
        "value": r["value"],
        "unit": "atom-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["s_per_step"] * 1e3,
        "higher_is_better": True,
        "scaling": "weak",  # independent replicas, one per core
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded 3-site water fixture, oracle-side generator)",
        "config": cfg,
        "cpu_baseline": {"value": r["value"], "unit": "atom-steps/s", "cores": threads,
                         "kind": "reference", "sample": _cpu_sample_text(r, threads),
                         "cpu_model": r["cpu_model"], "scalar_rel": r.get("scalar"),
                         "size_curve": _cpu_curve()},
        "e2e": {"value": r["value"], "unit": "atom-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def relaunch_torchrun(args) -> int:
    """`bench.py --gpus N` outside torchrun on a box with >= N GPUs: re-run
    this command as N ranks (one per GPU) under torch.distributed.run."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world == 1 and args.gpus > 1:
        import torch
        if torch.cuda.device_count() >= args.gpus:
            sys.exit(relaunch_torchrun(args))
        # fewer GPUs than requested: the N domains run on this one GPU
        out = run_dd(args, 1, 0, 0, "local", args.gpus)
        print(json.dumps(out), flush=True)
        return
    if world > 1 or (args.dd_nccl and "MASTER_ADDR" in os.environ):
        import torch
        import torch.distributed as dist
        assert args.gpus in (1, world), f"--gpus {args.gpus} under a world of {world} ranks"
        torch.cuda.set_device(local)
        # host-side plumbing (barriers, timing max, the NCCL id broadcast); the
        # data path is the group's own NCCL communicator (csrc/group.cu)
        dist.init_process_group("gloo")
        out = run_dd(args, world, rank, local, "nccl", world)
        if rank == 0:
            print(json.dumps(out), flush=True)
        dist.destroy_process_group()
        return
    out, wl = run_mine(args, world, rank, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(args, max(out["pcg_iters"], 1))
        except Exception as e:  # the CPU leg is a reported baseline, not the product
            out["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
