#!/usr/bin/env python
"""Benchmark: FP64 V(1,1) p-multigrid cycles (arXiv:1612.04796, Algorithm 1) on B200.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
A step = one V(1,1) cycle (all hot-path rows: residual/apply, Schwarz FDM solves + weighted
scatter on every level, transfers, coarse solve) over the config's synthetic input.
Default workload: BASELINE.json configs[2] ("c3": 16^3 elements, P=16 GLL, 20.1M DOF, the
config BASELINE.json marks "for throughput and roofline"); every other config can be benched
with --config.  N>1: independent replicas, one per GPU ("replicas only").
"""
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

METRIC = "FP64 V(1,1) DOF/s at 1 B200; residual reduction/cycle; % of FP64/HBM roofline"
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2 TF: 64 DFMA/clk/SM at 1965 MHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub-configs", action="store_true", help="skip the short c1/c2/c4/c5 runs")
    ap.add_argument("--profile-kernels", action="store_true", default=True)
    return ap.parse_args()


def hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling
    guide's fallback."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy test, measured on this pool)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def max_over_ranks(x, device="cpu"):
    """Max of a scalar over all ranks (the timing rule: a multi-GPU time is the slowest rank's)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(dofs_per_replica, world, cycles_per_replica, ms_max):
    """Whole-job DOF/s of `world` independent replicas (weak scaling) timed by the slowest rank."""
    return dofs_per_replica * world * cycles_per_replica / (ms_max / 1e3)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
def cycle_model(g, c, level=None):
    """Algorithmic flop / byte counts of one V(1,1) cycle;
    the third entry is the dense flop count of one Schwarz solve on `level` (default: top)."""
    L = g.L
    level = L if level is None else level
    NL = g.ndofs(L)
    flops = 0.0
    fdm_flops_top = 0.0
    for l in range(1, L + 1):
        n = 2 ** l + 1
        Nl = g.ndofs(l)
        Ne = Nl // n ** 3
        _, m = g.level_overlap(l)
        Mw = m[0] * m[1] * m[2]
        FA = (6 * n + (24 if c.basis == 0 else 48)) * Nl
        FS = (4 * (m[0] + m[1] + m[2]) + 4) * Mw * Ne
        FT = 7 * (2 ** (l - 1) + 1) * Nl
        flops += 3 * FA + 2 * FS + FT
        if l == level:
            fdm_flops_top = FS
    bytes_ = 120.0 * NL * 8.0 / 7.0
    return flops, bytes_, fdm_flops_top


def fdm_issued_flops(g, level):
    """FP64 tensor-core flops the even/odd Schwarz kernel actually issues on `level` (DMMA
    m8n8k4 = 512 flop): per 8-column tile of a 1D pass along d (extent m = 2H+1) it runs
    2 x ceil((H+1)/8) x ceil((H+1)/4) DMMAs (even and odd half-GEMMs); six passes (the z pass
    fused: forward + backward).  The algorithmic count (fdm_flops_top) is the dense one."""
    n = 2 ** level + 1
    Ne = g.ndofs(level) // n ** 3
    _, m = g.level_overlap(level)
    dm = 0
    for d in range(3):
        H = m[d] // 2
        per_tile = 2 * ((H + 1 + 7) // 8) * ((H + 1 + 3) // 4)
        cols = (m[0] * m[1] * m[2]) // m[d]
        dm += 2 * per_tile * ((cols + 7) // 8)          # forward + backward along d
    return 512.0 * dm * Ne


def fdm_bytes(g, level):
    """Algorithmic HBM bytes of one Schwarz-solve launch on `level`: the window gather reads every
    residual DOF once (8 B/DOF; the overlap halos are L2 hits) and the weighted windows are
    written once (8 M_w B per subdomain)."""
    n = 2 ** level + 1
    N = g.ndofs(level)
    _, m = g.level_overlap(level)
    return 8.0 * N + 8.0 * (N // n ** 3) * m[0] * m[1] * m[2]


def schwarz_entry(g, c, level, ms, peak_tf, hbm):
    """FP64 (tensor) and HBM roofline components of one Schwarz-solve launch of `level`."""
    flops = cycle_model(g, c, level=level)[2]
    by = fdm_bytes(g, level)
    t = ms / 1e3
    mt = g.level_overlap(level)[1]
    issued = fdm_issued_flops(g, level) if (all(x % 2 for x in mt) and max(mt) <= 31) else None
    return {"ms_per_launch": ms,
            "fp64": {"achieved_tflops": flops / t / 1e12, "peak_tflops": peak_tf, "frac": flops / t / 1e12 / peak_tf,
                     "algorithmic_flops": flops},
            "hbm": {"achieved_gbs": by / t / 1e9, "peak_gbs": hbm, "frac": by / t / 1e9 / hbm,
                    "algorithmic_bytes": by},
            "issued_dmma_tflops": issued / t / 1e12 if issued else None,
            "issued_frac": issued / t / 1e12 / peak_tf if issued else None}


def apply_entry_for(g, c, level, ms, peak_tf, hbm, cycles):
    """Operator apply / residual on `level`: u, f in, r out (24 B/DOF) plus the six neighbour
    trace segments (6 n^2 x 8 B per element); flops 6n + 24 (GLL) / 6n + 48 (GL) per DOF."""
    N = g.ndofs(level)
    n = 2 ** level + 1
    by = N * 24.0 + (N // n ** 3) * 6 * n ** 2 * 8.0
    fl = (6 * n + (24 if c.basis == 0 else 48)) * N
    t = ms / 1e3
    return {"dof_per_s": N / t, "ms_per_launch": ms,
            "bound": "hbm" if by / (hbm * 1e9) > fl / (peak_tf * 1e12) else "fp64",
            "hbm": {"achieved_gbs": by / t / 1e9, "peak_gbs": hbm, "frac": by / t / 1e9 / hbm, "algorithmic_bytes": by},
            "fp64": {"achieved_tflops": fl / t / 1e12, "peak_tflops": peak_tf, "frac": fl / t / 1e12 / peak_tf,
                     "algorithmic_flops": fl},
            "frac": max(by / (hbm * 1e9), fl / (peak_tf * 1e12)) / t}


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    from paper_1612_04796_b200 import DG
    from workloads import get_config, uniform_zero_mean

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    c = get_config(args.config)
    g = DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    N = g.ndofs()
    from paper_1612_04796_b200.binding import fp64_peak_tflops
    peak_dfma = max(fp64_peak_tflops(False) for _ in range(3))
    peak_dmma = max(fp64_peak_tflops(True) for _ in range(3))
    if c.rhs == "sin":            # c2: b = M 3 sin x sin y sin z (assembled by the library)
        f = g.rhs_sin(3.0, 1.0, 1.0, 1.0)
        f_host = f.cpu().pin_memory()
    else:
        f_host = torch.from_numpy(uniform_zero_mean(N, 0)).pin_memory()
        f = f_host.to(dev)
    u = torch.zeros(N, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    pcg = c.run == "pcg"
    # residual history: V(1,1) cycles from u = 0 until ||r||/||r0|| <= 1e-10 (at most 30), or the
    # PCG residual history (c5: V(1,1) as the preconditioner of inexact CG)
    r0 = float(np.sqrt(g.dot(f, f)))
    if pcg:
        _, hist, _ = g.pcg_solve(u, f, rtol=c.rtol, maxit=200)
        hist = [float(x) for x in hist]
    else:
        hist = [r0]
        for _ in range(30):
            g.pmg_vcycle(u, f)
            res = g.residual(u, f)
            hist.append(float(np.sqrt(g.dot(res, res))))
            if hist[-1] <= c.rtol * r0:
                break
        for _ in range(max(0, args.warmup - len(hist) + 1)):
            g.pmg_vcycle(u, f)
    rho = [hist[i + 1] / hist[i] for i in range(len(hist) - 1)]
    u.zero_()

    def step():
        if pcg:
            u.zero_()
            _, h, _ = g.pcg_solve(u, f, rtol=c.rtol, maxit=200)
            return len(h) - 1
        g.pmg_vcycle(u, f)
        return 1

    # ---- timed region: K steps (V-cycles replayed from CUDA graphs; for c5 K PCG solves),
    # device-timed with CUDA events on the launching stream; inputs > L2 for c3 (no flush)
    clocks = ClockSampler(local_rank)
    g.profile(False)
    launches0 = g.launch_count()
    barrier()
    clocks.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    cycles = 0
    ev0.record(stream)
    for _ in range(args.steps):
        cycles += step()
    ev1.record(stream)
    barrier()
    ms_total = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    launches = g.launch_count() - launches0
    # ---- per-kernel CUDA-event timing of the same K steps (eager launches, events on the
    # launching stream around every kernel) -> the dominant kernel's roofline entry
    g.profile(True)
    g.profile_read(reset=True)
    barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    pcycles = 0
    p0.record(stream)
    for _ in range(args.steps):
        pcycles += step()
    p1.record(stream)
    barrier()
    ms_profiled = p0.elapsed_time(p1) / args.steps
    prof = g.profile_read(reset=True)
    g.profile(False)
    ms_total = max_over_ranks(ms_total, dev)
    ms_step = ms_total / args.steps
    # value: DOF/s per V(1,1) cycle (PCG: N * iterations / t, one V-cycle per iteration)
    value = aggregate_value(N, world, cycles, ms_total)

    # ---- e2e: host buffers through the public API (H2D of u and f, cycle, D2H of u)
    u_host = torch.zeros(N, dtype=torch.float64).pin_memory()
    out_host = torch.empty(N, dtype=torch.float64).pin_memory()
    ud = torch.empty_like(u)
    fd = torch.empty_like(f)

    def e2e_step():
        ud.copy_(u_host, non_blocking=True)
        fd.copy_(f_host, non_blocking=True)
        if pcg:
            _, h, _ = g.pcg_solve(ud, fd, rtol=c.rtol, maxit=200)
            k = len(h) - 1
        else:
            g.pmg_vcycle(ud, fd)
            k = 1
        out_host.copy_(ud, non_blocking=True)
        return k

    for _ in range(2):
        e2e_step()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_cycles = 0
    e0.record(stream)
    for _ in range(args.steps):
        e2e_cycles += e2e_step()
    e1.record(stream)
    barrier()
    e2e_serial_ms = e0.elapsed_time(e1) / e2e_cycles

    # ---- e2e, pipelined: independent problems streamed through the same public API calls, the
    # H2D of step k+1 (copy stream) and the D2H of step k-1 (second copy stream) overlapping the
    # solve of step k; two device buffer sets.  Every step still copies its own u and f in and
    # its u out inside the timed region; only their overlap with the compute differs.
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ubuf = [ud, torch.empty_like(u)]
    fbuf = [fd, torch.empty_like(f)]
    obuf = [out_host, torch.empty(N, dtype=torch.float64).pin_memory()]
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]

    def pipelined(nsteps, start_ev=None):
        def h2d(k):
            sl = k % 2
            with torch.cuda.stream(s_in):
                if start_ev is not None:
                    s_in.wait_event(start_ev)
                if k >= 2:
                    s_in.wait_event(d2h_done[sl])        # the slot's previous result was read out
                ubuf[sl].copy_(u_host, non_blocking=True)
                fbuf[sl].copy_(f_host, non_blocking=True)
                h2d_done[sl].record(s_in)
        its = 0
        h2d(0)
        for k in range(nsteps):
            sl = k % 2
            if k + 1 < nsteps:
                h2d(k + 1)                               # enqueued before a (host-blocking) PCG solve
            stream.wait_event(h2d_done[sl])
            if pcg:
                _, h, _ = g.pcg_solve(ubuf[sl], fbuf[sl], rtol=c.rtol, maxit=200)
                its += len(h) - 1
            else:
                g.pmg_vcycle(ubuf[sl], fbuf[sl])
                its += 1
            comp_done[sl].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[sl])
                obuf[sl].copy_(ubuf[sl], non_blocking=True)
                d2h_done[sl].record(s_out)
        stream.wait_event(d2h_done[(nsteps - 1) % 2])
        if nsteps > 1:
            stream.wait_event(d2h_done[(nsteps - 2) % 2])
        return its

    pipelined(2)
    torch.cuda.synchronize()
    barrier()
    e0.record(stream)
    e2e_cycles = pipelined(args.steps, start_ev=e0)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1) / e2e_cycles

    # ---- roofline of the dominant kernel (Schwarz FDM solve on the top level)
    hbm, hbm_src = hbm_peak()
    flops, bytes_, fdm_flops = cycle_model(g, c)
    top = g.L
    fdm_ms, fdm_cnt = prof.get(("fdm", top), (0.0, 0))
    fdm_avg_ms = fdm_ms / max(fdm_cnt, 1)
    peak_tf = max(peak_dfma, peak_dmma)
    achieved_tf = fdm_flops / (fdm_avg_ms / 1e3) / 1e12 if fdm_avg_ms > 0 else None
    kernels = {"%s@l%d" % k: {"ms_per_step": round(v[0] / args.steps, 4), "launches_per_step": v[1] / args.steps,
                              "ms_per_cycle": round(v[0] / max(pcycles, 1), 4)}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    cyc_t_fp64 = flops / (peak_tf * 1e12)
    cyc_t_hbm = bytes_ / (hbm * 1e9)
    cyc_t_roof = max(cyc_t_fp64, cyc_t_hbm)
    ms_cycle = ms_total / max(cycles, 1)
    sch = schwarz_entry(g, c, top, fdm_avg_ms, peak_tf, hbm) if fdm_avg_ms > 0 else None
    # operator apply / residual on the top level (the three per cycle: two residuals and the
    # residual fused with the restriction)
    ap_ms, ap_cnt = prof.get(("apply", top), (0.0, 0))
    ap_avg_ms = ap_ms / max(ap_cnt, 1)
    apply_entry = None
    if ap_avg_ms > 0:
        apply_entry = apply_entry_for(g, c, top, ap_avg_ms, peak_tf, hbm, pcycles)
        apply_entry["launches_per_cycle"] = ap_cnt / max(pcycles, 1)
    traffic = None      # DRAM bytes per launch of the roofline kernel from the committed ncu capture
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(args.config, {}).get("fdm_top")
    except Exception:
        pass
    out = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "%s: %s, %dx%dx%d elements, P=%d %s, %d DOF, %s"
                   % (c.name, "periodic box %s" % (c.length,), c.ne[0], c.ne[1], c.ne[2], c.P,
                      "GLL" if c.basis == 0 else "GL", N,
                      "step = one PCG solve to 1e-10 (one V(1,1) per iteration)" if pcg
                      else "step = one V(1,1) cycle"),
                   "cycles_timed": cycles, "penalty_factor": c.penalty,
                   "overlap": {"mode": c.overlap.mode, "value": c.overlap.value, "floor": c.overlap.floor},
                   "l2": l2_note(N, dev),
                   "parallelism": "replicas" if world > 1 else "single"},
        "e2e": {"value": N * world / (e2e_ms / 1e3), "unit": "DOF/s",
                "mode": "pipelined: independent solves; H2D of step k+1 and D2H of step k-1 overlap step k",
                "serial_value": N * world / (e2e_serial_ms / 1e3), "h2d_bytes_per_step": 16 * N,
                "d2h_bytes_per_step": 8 * N},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": (achieved_tf / peak_tf) if achieved_tf else None, "traffic": traffic,
                     "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                     "kernel": "k_fdm_eoc (even/odd Schwarz fast-diagonalisation solve, top level, FP64 DMMA "
                               "tensor pipe); achieved = dense algorithmic flops (SURVEY 8(d), no even/odd "
                               "savings) / launch time",
                     "issued_dmma_tflops": sch["issued_dmma_tflops"] if sch else None,
                     "issued_frac": sch["issued_frac"] if sch else None,
                     "components": {"fp64": sch["fp64"], "hbm": sch["hbm"]} if sch else None,
                     "kernel_ms_per_launch": fdm_avg_ms,
                     "share_of_step": (fdm_ms / args.steps / ms_profiled) if ms_profiled else None,
                     "peak_source": "measured live by pmg_fp64_peak: max(DFMA %.2f, DMMA %.2f) TFLOP/s; "
                                    "nominal 148 SM x 64 FMA/clk x 2 x 1.965 GHz = %.1f; HBM %.1f GB/s: %s" % (
                                        peak_dfma, peak_dmma, FP64_NOMINAL_TFLOPS, hbm, hbm_src)},
        "cycle_roofline": {"flop_per_cycle": flops, "bytes_per_cycle": bytes_,
                           "t_fp64_ms": cyc_t_fp64 * 1e3, "t_hbm_ms": cyc_t_hbm * 1e3,
                           "t_roof_ms": cyc_t_roof * 1e3,
                           "frac_fp64": cyc_t_fp64 * 1e3 / ms_cycle, "frac_hbm": cyc_t_hbm * 1e3 / ms_cycle,
                           "frac": cyc_t_roof * 1e3 / ms_cycle},
        "apply_roofline": apply_entry,
        "residual_reduction_per_cycle": rho,
        "residual_history": hist,
        "kernels": kernels,
        "ms_per_step_profiled_eager": ms_profiled,
        "clocks": clk,
    }
    if pcg:
        # Table 2's remedy for high aspect ratios: the variable V-cycle,
        # nu_l = (1,1) 3^(L-l), as the CG preconditioner, beside the fixed V(1,1) above
        nu = [0] + [3 ** (g.L - l) for l in range(1, g.L + 1)]
        g.set_schedule(nu, nu)
        u.zero_()
        _, hv, okv = g.pcg_solve(u, f, rtol=c.rtol, maxit=200)
        barrier()
        v0 = torch.cuda.Event(enable_timing=True)
        v1 = torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        u.zero_()
        _, hv, okv = g.pcg_solve(u, f, rtol=c.rtol, maxit=200)
        v1.record(stream)
        barrier()
        tv = v0.elapsed_time(v1)
        g.set_schedule([1] * (g.L + 1), [1] * (g.L + 1))
        out["schedules"] = {
            "fixed_V11": {"iterations": cycles // max(args.steps, 1), "ms_per_solve": ms_step,
                          "ms_per_iteration": ms_step / max(cycles // max(args.steps, 1), 1)},
            "variable_3^(L-l)": {"iterations": len(hv) - 1, "converged": bool(okv), "ms_per_solve": tv,
                                 "ms_per_iteration": tv / max(len(hv) - 1, 1),
                                 "dof_per_s_per_solve": N / (tv / 1e3)}}
    if world == 1 and args.config == "c3" and not args.no_sub_configs:
        out["configs"] = {name: sub_config(name, peak_tf, hbm) for name in ("c1", "c2", "c4", "c5")}
        torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return out


def sub_config(name, peak_tf, hbm, steps=10, warmup=3):
    """Short device-timed run of another BASELINE.json config (graph-replayed V(1,1) cycles, or
    PCG solves for c5), with its top-level Schwarz-solve and apply roofline entries, so the default
    bench line carries every config (the driver observes all five)."""
    import numpy as np
    import torch
    from paper_1612_04796_b200 import DG
    from workloads import get_config, uniform_zero_mean
    c = get_config(name)
    g = DG(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
    N = g.ndofs()
    f = g.rhs_sin(3.0, 1.0, 1.0, 1.0) if c.rhs == "sin" else torch.from_numpy(uniform_zero_mean(N, 0)).cuda()
    u = torch.zeros_like(f)
    pcg = c.run == "pcg"
    steps = 2 if pcg else steps

    def step():
        if pcg:
            u.zero_()
            _, h, _ = g.pcg_solve(u, f, rtol=c.rtol, maxit=200)
            return len(h) - 1
        g.pmg_vcycle(u, f)
        return 1
    r0 = float(np.sqrt(g.dot(f, f)))
    for _ in range(warmup):
        step()
    rho1 = None
    if not pcg:
        u.zero_()
        g.pmg_vcycle(u, f)
        r = g.residual(u, f)
        rho1 = float(np.sqrt(g.dot(r, r))) / r0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cyc = sum(step() for _ in range(steps))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    g.profile(True)
    g.profile_read(reset=True)
    pc = sum(step() for _ in range(steps))
    prof = g.profile_read(reset=True)
    g.profile(False)
    flops, bytes_, _ = cycle_model(g, c)
    ms_cycle = ms / cyc
    t_roof = max(flops / (peak_tf * 1e12), bytes_ / (hbm * 1e9))
    top = g.L
    fm, fc = prof.get(("fdm", top), (0.0, 0))
    am, ac = prof.get(("apply", top), (0.0, 0))
    out = {"value": N * cyc / (ms / 1e3), "unit": "DOF/s", "ms_per_step": ms / steps, "steps": steps,
           "cycles_timed": cyc, "ms_per_cycle": ms_cycle, "dofs": N,
           "step": "PCG solve to 1e-10 (one V(1,1) per iteration)" if pcg else "V(1,1) cycle",
           "cycle_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms_cycle},
           "schwarz_top": schwarz_entry(g, c, top, fm / fc, peak_tf, hbm) if fc else None,
           "apply_top": apply_entry_for(g, c, top, am / ac, peak_tf, hbm, pc) if ac else None,
           "first_cycle_reduction": rho1,
           "kernels_ms_per_cycle": {"%s@l%d" % k: round(v[0] / max(pc, 1), 4)
                                    for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])[:8]}}
    if pcg:
        out["iterations"] = cyc // steps
        nu = [0] + [3 ** (g.L - l) for l in range(1, g.L + 1)]     # variable V-cycle (Table 2)
        g.set_schedule(nu, nu)
        u.zero_()
        g.pcg_solve(u, f, rtol=c.rtol, maxit=200)
        torch.cuda.synchronize()
        e0.record()
        u.zero_()
        _, hv, okv = g.pcg_solve(u, f, rtol=c.rtol, maxit=200)
        e1.record()
        torch.cuda.synchronize()
        out["variable_schedule_3^(L-l)"] = {"iterations": len(hv) - 1, "converged": bool(okv),
                                            "ms_per_solve": e0.elapsed_time(e1)}
    g.close()
    return out


def cpu_baseline(name, steps=2):
    """The oracle's matrix-free V(1,1) (oracle.mf, untuned, NumPy/SciPy) timed on the host cores:
    the full-size workload with every BLAS/OpenMP thread pool set to all available cores, a
    one-thread figure on an 8^3-element sample (the paper timed one core), and the oracle's
    operator apply on the full workload."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from workloads import get_config, uniform_zero_mean, uniform_vector
    from oracle.mf import MFHierarchy
    from oracle import mg
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count()
    c = get_config(name)
    with threadpool_limits(limits=cores):
        H = MFHierarchy(c.ne, c.length, c.P, c.basis, c.penalty, c.overlap)
        f = uniform_zero_mean(c.ndofs, 0)
        u = mg.vcycle(H, np.zeros_like(f), f)            # warm-up
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            u = mg.vcycle(H, u, f)
            ts.append(time.perf_counter() - t0)
        x = uniform_vector(c.ndofs, 1)
        H.apply(H.L, x)
        t0 = time.perf_counter()
        H.apply(H.L, x)
        t_apply = time.perf_counter() - t0
    del H, u, f, x
    t = statistics.median(ts)
    ne1 = tuple(min(v, 8) for v in c.ne)
    s1 = get_config(name, ne1)
    with threadpool_limits(limits=1):
        H1 = MFHierarchy(s1.ne, s1.length, s1.P, s1.basis, s1.penalty, s1.overlap)
        f1 = uniform_zero_mean(s1.ndofs, 0)
        u1 = mg.vcycle(H1, np.zeros_like(f1), f1)
        t0 = time.perf_counter()
        mg.vcycle(H1, u1, f1)
        t1 = time.perf_counter() - t0
    return {"value": c.ndofs / t, "unit": "DOF/s", "cores": cores, "threads": cores, "kind": "oracle",
            "sample": "oracle.mf V(1,1) on the full %s workload (%d DOF), median of %d after 1 warm-up; "
                      "BLAS/OpenMP pools limited to %d threads (threadpoolctl)" % (name, c.ndofs, steps, cores),
            "s_per_cycle": t,
            "one_thread": {"value": s1.ndofs / t1, "unit": "DOF/s", "threads": 1, "s_per_cycle": t1,
                           "sample": "oracle.mf V(1,1) on %s's P/basis/overlap with %dx%dx%d elements (%d DOF)"
                                     % (name, ne1[0], ne1[1], ne1[2], s1.ndofs)},
            "apply": {"value": c.ndofs / t_apply, "unit": "DOF/s", "s_per_apply": t_apply,
                      "sample": "oracle.mf operator apply on the full %s workload" % name}}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    cb = None
    import numpy as np
    from workloads import get_config, uniform_zero_mean
    from oracle.mf import MFHierarchy
    from oracle import mg
    c = get_config(args.config)
    ne = tuple(min(x, 8) for x in c.ne)
    s = get_config(args.config, ne)
    H = MFHierarchy(s.ne, s.length, s.P, s.basis, s.penalty, s.overlap)
    f = uniform_zero_mean(s.ndofs, 0)
    u = np.zeros_like(f)
    for _ in range(args.warmup):
        u = mg.vcycle(H, u, f)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        u = mg.vcycle(H, u, f)
    t = (time.perf_counter() - t0) / args.steps
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count()
    v = s.ndofs / t
    sample = "oracle.mf V(1,1) on %s's P/basis/overlap with %dx%dx%d elements (%d DOF)" % (
        args.config, ne[0], ne[1], ne[2], s.ndofs)
    return {"metric": METRIC, "value": v, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "%s (CPU oracle sample)" % args.config},
            "cpu_baseline": {"value": v, "unit": "DOF/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def l2_note(N, dev):
    """How the timed iterations relate to L2 (no flush is done either way)."""
    import torch
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    mb = N * 8 / 1e6
    if N * 8 > l2:
        return "inputs larger than L2 (u, f, r: %.0f MB each, L2 %.0f MB); no flush" % (mb, l2 / 1e6)
    return ("vectors fit in L2 (u, f, r: %.1f MB each, L2 %.0f MB); no flush: L2-warm iterations "
            "(a parity config; the headline c3 streams from HBM)" % (mb, l2 / 1e6))


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local_rank)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
