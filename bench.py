#!/usr/bin/env python
"""Benchmark: particle-steps/s of the cuTAMP hot path (BASELINE.json metric) on 1..8 B200.

One bench *step* = one optimisation round over one batch of synthetic particles, i.e. one pass of
every SURVEY §8(a) row: K1 sampling (a2) -> `adam_steps` fused Eq. 4 Adam steps (a3-a10), with an
Eq. 3 check + NCCL all-reduce of the satisfied counts every `check_every` steps (a11, a12) -> local
best-k -> NCCL all-gather -> deterministic merge (a12).  value = particles x Adam steps of all ranks
/ max-over-ranks device time of the timed steps.

Usage:  python bench.py [--gpus N --steps K --warmup W] [--config 2] [--n PER_RANK] [--impl reference]
        (N > 1: launched by torchrun, one process per GPU, NCCL over NVLink)
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from workloads import make_config, CONFIG_NAMES, CONFIG_SIZES  # noqa: E402

METRIC = "particle-steps/sec (cost+grad+update)"
UNIT = "particle-steps/s"
CONFIG_DESC = {
    1: "pick-place skeleton, 7-DOF sphere arm, 1 table",
    2: "obstruction stacking: move 2 obstructors, stack red on blue (3 pick-place)",
    3: "Tetris-4 packing + min-object-distance goal cost",
    4: "Tetris-6 packing with trajectory-knot collision costs",
    5: "Tetris-4 packing skeleton (particle-count sweep)",
    6: "Stick Button: press red directly, press the out-of-reach blue button with the stick (not a BASELINE config)",
    7: "Stick Button, infeasible skeleton: press blue with the fingertip (not a BASELINE config)",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=3,
                   help="BASELINE config (default 3: Tetris-4 + goal at 32,768 particles, the largest single-GPU config)")
    p.add_argument("--n", type=int, default=None, help="particles per rank (default: the config's BASELINE size)")
    p.add_argument("--adam-steps", type=int, default=100)
    p.add_argument("--check-every", type=int, default=10)
    p.add_argument("--k", type=int, default=16)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-ttfs", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--lanes", type=int, default=0, help="lanes per particle in the particle kernel (0 = auto)")
    p.add_argument("--block-threads", type=int, default=0, help="particle-kernel block size (0 = auto)")
    p.add_argument("--block-sync", type=int, default=-1, help="block-synchronous phases (1/0, -1 = auto)")
    p.add_argument("--self-collision", action="store_true", help="add the SELF term (SURVEY §8(f) f2)")
    p.add_argument("--ik-iters", type=int, default=20,
                   help="conditional IK sampler iterations in InitializeParticles (P:521); 0 = uniform confs")
    p.add_argument("--ik-seeds", type=int, default=8, help="IK restarts per conf (1, 2, 4, 8; DESIGN.md R6)")
    p.add_argument("--repeats", type=int, default=5, help="timed regions of exactly --steps steps; value = median")
    p.add_argument("--no-extra", action="store_true", help="skip the extra workloads (config 2, config 1 at 1M, SELF)")
    p.add_argument("--no-overlap", action="store_true", help="all-reduce of the counts on the launching stream")
    p.add_argument("--dist", action="store_true",
                   help="initialise torch.distributed (NCCL) even with one rank: runs the collective path (overlapped "
                        "C1 all-reduce, C2 all-gather, K5 merge) on one GPU")
    p.add_argument("--nvtx", action="store_true", help="NVTX ranges around the phases of a step (profiling)")
    p.add_argument("--lib", default=None, help="A/B experiments: another in-tree build of libtamp.so (exp/<name>/)")
    p.add_argument("--pipeline", type=int, default=-1,
                   help="1: the next batch's sampling + IK on a second stream under this batch's optimisation "
                        "(two contexts); 0: sequential; -1: auto (single-wave particle launches)")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        try:
            return json.load(open(path)), "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------------------------------------
# algorithmic work per particle-step: FP32-pipe instructions of the
# minimal evaluation of each unit (FFMA = 1), independent of how the kernel maps or culls it.
# ------------------------------------------------------------------------------------------------
W_FK = 344          # 7 x (Rz apply 6 + sincos 2) + 8 x 3x4 compose 36
W_SPH_XFORM = 9     # per robot sphere per conf
W_SPH_BWD = 9       # wrench accumulation per robot sphere
W_LINK_BWD = 8 * 6 + 7 * 15   # suffix sums + dq per conf
W_PAIR_SB = 24      # sphere-OBB inactive test: R^T(w-c) 12, |p|-h 3, max 3, |q|^2 3, max 2, cmp 1
W_PAIR_SS = 8       # sphere-sphere inactive test: diff 3, |d|^2 3, radius 1, cmp 1
W_KIN = 90          # target compose 36, M 27, residuals ~27
W_JL = 35
W_PLACE = 100       # decode, support, containment per placed object
W_GOAL_PAIR = 23
W_SEG = 25
W_ADAM = 12         # per coordinate


def algorithmic_instr(w):
    n_fk, S = w["n_fk"], w["n_robot_spheres"]
    return (n_fk * (W_FK + S * (W_SPH_XFORM + W_SPH_BWD) + W_LINK_BWD + W_JL)
            + W_PAIR_SB * w["pairs_sphere_obb"] + W_PAIR_SS * (w["pairs_sphere_sphere"] + w.get("pairs_self", 0))
            + W_KIN * w["n_kin"] + W_PLACE * w["n_place"] + W_GOAL_PAIR * w["n_goal_pairs"]
            + W_SEG * w["n_traj_seg"] + W_ADAM * w["D"])


def algorithmic_instr_check(w):
    """The Eq. 3 check of one particle: the forward part of a step (no wrench accumulation, link backward or
    Adam update)."""
    n_fk, S = w["n_fk"], w["n_robot_spheres"]
    return algorithmic_instr(w) - n_fk * (S * W_SPH_BWD + W_LINK_BWD) - W_ADAM * w["D"]


# ------------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML polled every 2 ms
    from a background thread (the launching thread is not touched), nvidia-smi as a fallback."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.samples = []          # (sm_mhz, max_mhz, reason bitmask)
        self._stop = threading.Event()
        self.nvml = None
        self.proc = None

    def _handle(self, pynvml):
        try:
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = self._handle(pynvml)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), float(mx), int(rs)))
                    except Exception:
                        pass
                    self._stop.wait(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
            self._start_smi()
        return self

    def _start_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def read():
                bits = [0x8, 0x40, 0x20, 0x4]
                for line in self.proc.stdout:
                    f = [x.strip() for x in line.split(",")]
                    try:
                        m = sum(b for b, v in zip(bits, f[2:6]) if v.lower() == "active")
                        self.samples.append((float(f[0]), float(f[1]), m))
                    except (ValueError, IndexError):
                        continue
            self.t = threading.Thread(target=read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def __exit__(self, *a):
        self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if getattr(self, "t", None) is not None:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return None
        sm = [s[0] for s in self.samples]
        reasons = sorted({nm for s in self.samples for b, nm in self.REASONS.items() if s[2] & b})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ------------------------------------------------------------------------------------------------
def free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def spawn_ranks(n, argv, script=None, env=None):
    """One process per GPU of this node: re-launch `script` (default: this file) with argv under
    torch.distributed.run, n ranks, rendezvous on 127.0.0.1.  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script or os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd, env=env)


def dist_init(args):
    """RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* from the environment (torchrun, or spawn_ranks).  NCCL over
    NVLink for the product path, gloo for the (host-only) reference arm."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world} (launch one process per GPU)")
    if world > 1 or getattr(args, "dist", False):
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        if args.impl == "ours":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        return world, rank, local, dist
    return 1, 0, 0, None


def run_round(ctx, seed, args, dist, world, events=None, host_counts=None, host_rec=None, side=None, sampled=False):
    """One bench step (see module docstring).  Returns the merged global best-k records.

    With `side` (a CUDA stream) and NCCL, the SUM all-reduce of each interval's counts (C1) runs on the side
    stream while the next optimisation launch runs on the launching stream (particles never couple, Eq. 4,
    P:461-467, so nothing in the next launch waits for the counts); two count buffers alternate, and a buffer
    is only rewritten after its all-reduce finished.  The counts are the same bytes either way.
    sampled: the batch was already initialised (pipelined rounds, timed_rounds)."""
    nvtx = getattr(args, "nvtx", False)
    if not sampled:
        if nvtx:
            torch.cuda.nvtx.range_push("sample+IK (K1, K1b)")
        ctx.sample(seed)
        if nvtx:
            torch.cuda.nvtx.range_pop()
    n_int = args.adam_steps // args.check_every
    direct = host_counts is not None and world == 1
    overlap = side is not None and dist is not None and not direct
    bufs = getattr(ctx, "_bench_counts", None)
    if overlap and bufs is None:
        bufs = ctx._bench_counts = [torch.zeros_like(ctx.counts_buf) for _ in range(2)]
    main_s = torch.cuda.current_stream() if overlap else None
    for i in range(n_int):
        # check_every fused Adam steps + the Eq. 3 check of the final state: one C-ABI call, one launch for the
        # link mappings (tamp_optimize_and_check; the serial mapping launches the check separately)
        if events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        if nvtx:
            torch.cuda.nvtx.range_push(f"K2 x{args.check_every} + check")
        if overlap:
            if i >= 2:
                main_s.wait_stream(side)                  # buffer i % 2 free again (its all-reduce is done)
            counts, _ = ctx.optimize_check(args.check_every, counts=bufs[i % 2])
        else:
            counts, _ = ctx.optimize_check(args.check_every, counts=host_counts if direct else None)
        if nvtx:
            torch.cuda.nvtx.range_pop()
        if events is not None:
            e1.record()
            events.append((e0, e1))
        if overlap:
            side.wait_stream(main_s)
            with torch.cuda.stream(side):
                dist.all_reduce(counts)                   # NCCL SUM of satisfied counts (C1), overlapped
                if host_counts is not None:
                    host_counts.copy_(counts, non_blocking=True)   # D2H after the all-reduce, same stream
        elif not direct:                                  # (direct: D2H through the C ABI into the host buffer)
            if dist is not None:
                dist.all_reduce(counts)                   # NCCL SUM of satisfied counts (C1)
            if host_counts is not None:
                host_counts.copy_(counts)                 # D2H
    if overlap:
        main_s.wait_stream(side)
    if nvtx:
        torch.cuda.nvtx.range_push("best-k (K4), all-gather, merge (K5)")
    try:
        return _finish_round(ctx, args, dist, world, host_rec)
    finally:
        if nvtx:
            torch.cuda.nvtx.range_pop()


def _finish_round(ctx, args, dist, world, host_rec):
    if host_rec is not None and world == 1:
        ctx.best_k(args.k, out=host_rec)
        return host_rec
    rec = ctx.best_k(args.k)
    if dist is not None:
        gathered = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(gathered, rec)                    # C2
        rec = torch.cat(gathered)
    merged = ctx.merge_best_k(rec, args.k)                # K5
    if host_rec is not None:
        host_rec.copy_(merged)
    return merged


def max_over_ranks(v, dist):
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(args, spec, budget_s, ctx=None):
    """The float64 oracle (as it stands) on the host cores: bounded sample of the same workload.  The same leg
    re-verifies parity in this run: the first 256 particles of the bench context's current state
    (the end of the timed rounds) are re-evaluated by the oracle -- cost, per-term costs, gradient."""
    from oracle import tamp_oracle as O
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    n = 256
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 1, np.arange(n))
    st = O.new_state(x, g)
    O.optimize(spec, csp, st, 1, 1.0 / n)               # warm-up
    t0 = time.perf_counter()
    steps = 0
    while True:
        O.optimize(spec, csp, st, 1, 1.0 / n)
        steps += 1
        if time.perf_counter() - t0 >= budget_s and steps >= 2:
            break
    dt = time.perf_counter() - t0
    # the same sample on one host core (SURVEY §8(d) asks for all cores and 1 core), a third of the budget
    torch.set_num_threads(1)
    t1 = time.perf_counter()
    steps1 = 0
    while True:
        O.optimize(spec, csp, st, 1, 1.0 / n)
        steps1 += 1
        if time.perf_counter() - t1 >= budget_s / 3 and steps1 >= 1:
            break
    dt1 = time.perf_counter() - t1
    out = {"value": n * steps / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
           "value_1core": n * steps1 / dt1,
           "sample": f"{n} particles x {steps} Adam steps of {CONFIG_NAMES[args.config]} "
                     f"(float64 oracle, torch autograd, {cores} threads), {dt:.1f} s; "
                     f"value_1core: {steps1} steps on 1 thread, {dt1:.1f} s"}
    if ctx is not None:
        torch.set_num_threads(cores)
        out["parity_recheck"] = parity_recheck(O, spec, csp, ctx, min(256, ctx.n))
    return out


def parity_recheck(O, spec, csp, ctx, m):
    """Oracle vs the GPU on the first m particles of the bench context's state (north_star tolerances: cost and
    per-term costs rel 1e-4, gradient rel 1e-3).  Particles whose oracle gradient is not smooth within +-1e-5
    (second-difference kink test) are reported, not failed."""
    st = ctx.get_state()
    J, soft, Jc, grad = (t.cpu().numpy()[:m] for t in ctx.eval())
    x = st["x"].cpu().numpy()[:m].astype(np.float64)
    g = st["grasp"].cpu().numpy()[:m].reshape(m, -1, 3, 4).astype(np.float64)
    Jo, Jco, softo, grado = O.cost_and_grad(spec, csp, x, g)
    cost_ok = (np.abs(J - Jo) <= 1e-4 * np.abs(Jo) + 1e-6) & np.all(np.abs(Jc - Jco) <= 1e-4 * np.abs(Jco) + 1e-6, 1)
    gerr = np.abs(grad - grado).max(axis=1)
    gscale = np.abs(grado).max(axis=1)
    grad_ok = gerr <= 1e-3 * gscale + 1e-6
    kink = np.zeros(m, bool)
    bad = np.where(~grad_ok)[0]
    if len(bad):
        r = np.random.default_rng(0).normal(size=(len(bad), x.shape[1]))
        r /= np.linalg.norm(r, axis=1, keepdims=True)
        _, _, _, gp = O.cost_and_grad(spec, csp, x[bad] + 1e-5 * r, g[bad])
        _, _, _, gm = O.cost_and_grad(spec, csp, x[bad] - 1e-5 * r, g[bad])
        kink[bad] = np.abs(gp - 2 * grado[bad] + gm).max(axis=1) > 1e-4 * gscale[bad]
    return {"particles": m, "cost_match": int(cost_ok.sum()), "grad_match": int(grad_ok.sum()),
            "grad_kinks_excluded": int((~grad_ok & kink).sum()), "grad_mismatch_smooth": int((~grad_ok & ~kink).sum()),
            "state": f"bench context after the timed rounds (t = {st['t']})"}


def bench_reference(args, world, rank, dist):
    """--impl reference: the oracle timed on the host cores on a bounded sample of the same workload."""
    if rank != 0:
        return
    from oracle import tamp_oracle as O
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    spec = make_config(args.config)
    csp = O.build_csp(spec)
    n, adam = 128, 4

    def step(seed):
        xs, gs = O.initialize_particles(spec, csp, seed, np.arange(n))
        st = O.new_state(xs, gs)
        O.optimize(spec, csp, st, adam, 1.0 / n)
        cls, counts, J, soft, Jc = O.check(spec, csp, st)
        O.best_k(cls, J, soft, np.arange(n), min(args.k, n))

    for w in range(args.warmup):
        step(100 + w)
    t0 = time.perf_counter()
    for s in range(args.steps):
        step(200 + s)
    dt = time.perf_counter() - t0
    value = n * adam * args.steps / dt
    sample = f"{n} particles x {adam} Adam steps (+ sample, check, best-k) per step, float64 oracle, {cores} threads"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config{args.config}:{CONFIG_NAMES[args.config]}", "particles_per_step": n,
                       "adam_steps_per_step": adam, "parallelism": f"dp{world} (rank 0 runs the oracle)"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def ttfs(ctx, args, dist, world, seed, budget_steps=1000):
    """Time-to-first-satisfying: wall time from sampling to the first all-reduced check with >= 1
    satisfying particle (checks every `check_every` steps, budget 1000 steps)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.sample(seed)
    steps = 0
    while steps < budget_steps:
        counts, _ = ctx.optimize_check(args.check_every)
        steps += args.check_every
        if dist is not None:
            dist.all_reduce(counts)
        if int(counts[-2].item()) > 0:
            return {"s": time.perf_counter() - t0, "steps": steps, "satisfying": int(counts[-2].item())}
    return {"s": None, "steps": steps, "satisfying": 0, "note": "not reached within budget"}


def make_spec(args, cfg, n, self_collision=None):
    spec = make_config(cfg, n=n)
    spec.ik_iters = args.ik_iters
    spec.ik_seeds = args.ik_seeds
    spec.self_collision = args.self_collision if self_collision is None else self_collision
    return spec


def default_n(args, cfg):
    if args.n and cfg == args.config:
        return args.n
    if cfg == 4:
        return 131072 // 8                           # config 4: 128K particles over 8 GPUs (per-rank share)
    return CONFIG_SIZES[cfg]


def roofline(ctx, args, opt_avg, clocks=None, cfg=None, n=None):
    """Roofline of the dominant kernel (k_particle / k_serial: check_every fused Adam steps + the fused Eq. 3 check
    per launch): algorithmic FP32-pipe instructions per launch / the launch's measured duration (CUDA events on
    the launching stream), against 148 SM x 128 lanes x sm_max_mhz (ALU / issue bound)."""
    pk, src = peaks()
    w = dict(ctx.work)
    instr = algorithmic_instr(w)
    instr_check = algorithmic_instr_check(w)
    achieved = (instr * args.check_every + instr_check) * ctx.n / opt_avg / 1e12     # T instr/s per GPU
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(ctx.device).multi_processor_count
    peak = nsm * 128 * sm_max * 1e6 / 1e12
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        ent = tj.get(f"config{cfg}:{n}")
        if ent and args.check_every == 10:
            traffic = ent["dram_read"] + ent["dram_write"]
    except Exception:
        pass
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tinstr/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu --set full capture of this config / N, "
                                                "profiles/ncu_traffic.json; null if none)",
            "algorithmic_bytes_per_launch": ctx.n * (2 * 3 * ctx.D * 4 + 48 * ctx.n_grasp),
            "kernel": "k_serial<MODE_OPT>" if ctx.lanes_per_particle == 1 else "k_particle<MODE_OPT>",
            "note": f"FP32-pipe instructions (FFMA=1) of the minimal per-unit evaluation, {instr} per particle-step "
                    f"x {args.check_every} steps + {instr_check} for the Eq. 3 check fused into the launch; "
                    f"peak = {nsm} SM x 128 lanes x {sm_max:.0f} MHz ({src} sm_max_mhz)"}
    if clocks:
        roof["frac_at_measured_clock"] = achieved / (nsm * 128 * clocks["sm_mhz"] * 1e6 / 1e12)
    return roof


def timed_rounds(ctx, args, dist, world, flush, steps, seed0, side, opt_events=None, ctx2=None, prefetch=None):
    """Exactly `steps` bench steps between a barrier + synchronize on both sides; returns the max-over-ranks
    device time (s) of the steps (CUDA events on the launching stream, L2 flushed before each step, untimed).

    Pipelined rounds (ctx2 and a `prefetch` stream given): two contexts alternate; during step s the next batch's
    InitializeParticles (K1 + the conditional IK sampler) runs on the prefetch stream into the other
    context while this batch's optimisation runs on the launching stream (batches never couple).  Every step waits
    for its prefetch before its end event, so all of a step's work lies inside its timed window and nothing runs
    under the untimed flush; step 0 samples its own batch inside its window.  Same particles, same results."""
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev = []
    main = torch.cuda.current_stream()
    cs = [ctx, ctx2]
    for s in range(steps):
        flush.zero_()                                 # L2 flush between timed steps (not timed)
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record()
        if ctx2 is None:
            run_round(ctx, seed0 + s, args, dist, world, events=opt_events, side=side)
        else:
            cur, nxt = cs[s % 2], cs[(s + 1) % 2]
            if s == 0:
                cur.sample(seed0)
            if s + 1 < steps:
                prefetch.wait_stream(main)
                nxt.sample(seed0 + s + 1, stream=prefetch)
            run_round(cur, seed0 + s, args, dist, world, events=opt_events, side=side, sampled=True)
            main.wait_stream(prefetch)
        r1.record()
        ev.append((r0, r1))
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    return max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / 1e3, dist)


def extra_workload(args, cfg, n, dist, world, rank, dev, flush, side, self_collision=False, steps=3):
    """A further workload of the same metric (not the headline): value, kernel rate and roofline fraction."""
    spec = make_spec(args, cfg, n, self_collision)
    from paper_2411_11833_b200 import TampContext
    ctx = TampContext(spec, n, global_offset=rank * n, n_global=n * world, device=dev)
    for w in range(2):
        run_round(ctx, 50_000 + w, args, dist, world, side=side)
    ev = []
    t = timed_rounds(ctx, args, dist, world, flush, steps, 60_000, side, ev)
    opt_avg = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in ev) / 1e3, dist)
    roof = roofline(ctx, args, opt_avg, cfg=cfg, n=n)
    return {"workload": f"config{cfg}:{CONFIG_NAMES[cfg]}" + (" + SELF" if self_collision else ""),
            "particles_per_gpu": n, "value": n * world * args.adam_steps * steps / t, "unit": UNIT,
            "ms_per_step": t / steps * 1e3, "kernel_ms_per_launch": opt_avg * 1e3,
            "kernel_particle_steps_per_s": n * world * args.check_every / opt_avg,
            "roofline_frac": roof["frac"], "lanes_per_particle": ctx.lanes_per_particle,
            "block_threads": ctx.block_threads, "steps": steps}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (the driver launches torchrun itself)
        if args.impl == "ours" and torch.cuda.device_count() < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} CUDA device(s)")
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:]))
    world, rank, local, dist = dist_init(args)
    if args.impl == "reference":
        bench_reference(args, world, rank, dist)
        if dist is not None:
            dist.destroy_process_group()
        return
    from paper_2411_11833_b200 import TampContext, kernel_launches, lib_path, load
    import paper_2411_11833_b200.build as bld
    if args.lib:
        load(args.lib)
    else:
        bld.build()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    torch.set_num_threads(1)
    cfg = args.config
    n = default_n(args, cfg)
    spec = make_spec(args, cfg, n)
    n_global = n * world
    ctx = TampContext(spec, n, global_offset=rank * n, n_global=n_global, device=dev, lanes_per_particle=args.lanes,
                      block_threads=args.block_threads, block_sync=args.block_sync)
    side = None if (args.no_overlap or dist is None) else torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)    # > 126 MB L2
    # pipelined rounds pay where the particle launches leave SMs idle (one partial wave: config 2); with full waves
    # the prefetch only competes for them (config 3, measured)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    single_wave = ctx.lanes_per_particle > 1 and n <= nsm * (ctx.block_threads // ctx.lanes_per_particle)
    pipeline = args.pipeline if args.pipeline >= 0 else int(single_wave)
    ctx2 = prefetch = None
    if pipeline:
        ctx2 = TampContext(spec, n, global_offset=rank * n, n_global=n_global, device=dev,
                           lanes_per_particle=args.lanes, block_threads=args.block_threads, block_sync=args.block_sync)
        prefetch = torch.cuda.Stream(dev)
    for w in range(args.warmup):
        run_round(ctx, 10_000 + w, args, dist, world, side=side)
        if ctx2 is not None:
            run_round(ctx2, 11_000 + w, args, dist, world, side=side)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches0 = kernel_launches()
    opt_events, reps = [], []
    with ClockSampler(local) as clk:
        for r in range(args.repeats):
            t_round = timed_rounds(ctx, args, dist, world, flush, args.steps, 20_000 + 1000 * r, side, opt_events,
                                   ctx2=ctx2, prefetch=prefetch)
            reps.append((t_round, n_global * args.adam_steps * args.steps / t_round))
    launches = (kernel_launches() - launches0) // args.repeats
    t_round, value = sorted(reps, key=lambda tv: tv[1])[len(reps) // 2]        # median of the repeats
    opt_avg = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in opt_events) / 1e3, dist)
    clocks = clk.summary()
    roof = roofline(ctx, args, opt_avg, clocks, cfg, n)

    # end-to-end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        host_counts = torch.zeros(ctx.n_hard + 2, dtype=torch.int32).pin_memory()
        host_rec = torch.zeros(args.k, ctx.D + 4, dtype=torch.float32).pin_memory()

        def fresh():
            return TampContext(spec, n, global_offset=rank * n, n_global=n_global, device=dev,
                               lanes_per_particle=args.lanes, block_threads=args.block_threads,
                               block_sync=args.block_sync)                 # host descriptor in, every step
        for w_ in range(2):
            run_round(fresh(), 30_000 + w_, args, dist, world, host_counts=host_counts, host_rec=host_rec, side=side)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_steps = max(3, min(args.steps, 10))
        for s in range(e2e_steps):
            run_round(fresh(), 40_000 + s, args, dist, world, host_counts=host_counts, host_rec=host_rec, side=side)
        torch.cuda.synchronize()
        te = max_over_ranks(time.perf_counter() - t0, dist)
        import ctypes
        from paper_2411_11833_b200.tamp import ProblemDesc
        h2d = ctypes.sizeof(ProblemDesc) + 3 * ctx.D * 4
        d2h = (args.adam_steps // args.check_every) * (ctx.n_hard + 2) * 4 + args.k * (ctx.D + 4) * 4
        e2e = {"value": n_global * args.adam_steps * e2e_steps / te, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    extra = []
    if not args.no_extra:
        for ecfg, en, eself in ((2, 8192, False), (1, 1 << 20, False), (cfg, n, True)):
            if ecfg == cfg and not eself:
                continue
            extra.append(extra_workload(args, ecfg, en, dist, world, rank, dev, flush, side, self_collision=eself))

    tt = None if args.no_ttfs else ttfs(ctx, args, dist, world, seed=1000 * cfg)
    # TTFS of config 4 at its global batch (131,072 particles, BASELINE.json: 8 GPUs x 16,384), split over the ranks
    tt_extra = []
    if not args.no_ttfs and not args.no_extra and cfg != 4:
        n4 = 131072 // world
        ctx4 = TampContext(make_spec(args, 4, n4), n4, global_offset=rank * n4, n_global=n4 * world, device=dev)
        t4 = ttfs(ctx4, args, dist, world, seed=4000)
        t4.update({"workload": f"config4:{CONFIG_NAMES[4]}", "particles_global": n4 * world, "particles_per_gpu": n4})
        tt_extra.append(t4)
        del ctx4
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle leg re-checks parity on the bench context: bring it back to the timed rounds' state
        run_round(ctx, 20_000, args, dist, world)
        cpu = cpu_baseline(args, make_config(cfg, n=256), args.cpu_seconds, ctx=ctx)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_round / args.steps * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"config{cfg}:{CONFIG_NAMES[cfg]}", "description": CONFIG_DESC[cfg],
                           "particles_per_gpu": n, "particles_global": n_global, "D": ctx.D,
                           "hard_terms": ctx.n_hard, "adam_steps_per_step": args.adam_steps,
                           "check_every": args.check_every, "best_k": args.k, "l2": "flushed between steps",
                           "ik_iters": args.ik_iters, "ik_seeds": args.ik_seeds, "self_collision": args.self_collision,
                           "lanes_per_particle": ctx.lanes_per_particle, "block_threads": ctx.block_threads,
                           "block_sync": ctx.block_sync, "allreduce": "side stream, overlapped" if side else "inline",
                           "pipeline": "next batch's sampling + IK on a second stream" if pipeline else "sequential",
                           "parallelism": f"dp{world}"},
                "repeats": {"n": len(reps), "values": [v for _, v in reps], "reported": "median"},
                "kernel_ms_per_launch": opt_avg * 1e3, "kernel_steps_per_launch": args.check_every,
                "kernel_launch": "check_every fused Adam steps + the Eq. 3 check of the final state",
                "kernel_particle_steps_per_s": n_global * args.check_every / opt_avg,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "ttfs": tt, "ttfs_extra": tt_extra, "extra": extra,
                "lib": os.path.relpath(lib_path(), ROOT),
                "scaling_note": "weak scaling (particles per GPU fixed); no multi-GPU curve exists until a driver "
                                "SCALE run" if world == 1 else "weak scaling, max over ranks"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
