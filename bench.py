#!/usr/bin/env python
"""QBX-FMM layer-potential apply throughput on B200 (BASELINE.json metric).

One step = one full GIGAQBX evaluation (Algorithm 4, Stages 2-9) of BASELINE.json
config 1: Laplace single+double layer on the R=2/r=1 torus, 256x128 cells,
65,536 flat triangles x 16 Gauss-Legendre/Duffy nodes = 1,048,576 sources,
2,097,152 QBX centres and on-surface targets, p_fmm=15, p_qbx=5, n_max=64,
t_f=0.9.  Metric: (N_S + N_T) / t_apply.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Default (no torchrun): N=1, config 1, plus side measurements (config 4 on one GPU as the
scaling base, config 3 Helmholtz with per-stage fractions, config 2 association).  Under
torchrun each rank drives one GPU and owns a contiguous Morton (DFS-preorder) range of
boxes of BASELINE config 4 (64 urchins, strong scaling; --weak: 8 urchins per GPU);
multipoles are exchanged by NCCL broadcasts inside the apply, the near field overlaps
the exchange, and the owned results are gathered.  --impl reference
times the CPU restatement of the path (oracle/; the reference ships no FMM code to run)
on the same workload with all host threads.
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

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

CONFIG_ID = 1
CPU_SAMPLE = dict(nu=64, nv=32)  # 4,096 triangles, 65,536 sources: same family and orders, 1/16 size


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--small", action="store_true", help="debug: torus 64x32 instead of config 1")
    ap.add_argument("--workload", default="auto", choices=["auto", "config1", "config4"],
                    help="auto: config 1 on one GPU, config 4 (64 urchins) under torchrun")
    ap.add_argument("--weak", action="store_true", help="config 4 weak scaling: 8 urchins per GPU")
    ap.add_argument("--no-config4", action="store_true", help="skip the one-GPU config-4 scaling base")
    ap.add_argument("--no-helmholtz", action="store_true", help="skip the side measurements (config-3 Helmholtz, config-2 association)")
    return ap.parse_args()


# ---------------------------------------------------------------------------- work model
def stage_work(led, cfg, n_src, n_ctr, n_assoc, n_conv):
    """Algorithmic fp64 flops and compulsory bytes per stage (SURVEY.md §8d conventions:
    real flops, FMA = 2; K_x = (x+1)(x+2)/2 half-table coefficients)."""
    K = lambda x: (x + 1) * (x + 2) // 2
    p, q = cfg.p_fmm, cfg.p_qbx
    kp, kq, kpq = K(p), K(q), K(p + q)
    dl = cfg.kernel == 1
    src_b = 56 if dl else 32
    f = {}
    b = {}
    f["p2m"] = led["n_p2m_sources"] * ((26 if dl else 10) * kp + (40 if dl else 30))
    b["p2m"] = n_src * src_b + 16 * kp * led["n_p2m_sources"] / 8.0
    f["m2m"] = led["n_m2m"] * 8 * kp * kp
    b["m2m"] = led["n_m2m"] * 2 * 16 * kp
    f["near"] = led["pairs_qbx_near"] * ((26 if dl else 10) * kq + (40 if dl else 30)) + \
        led["pairs_p2p_near"] * (30 if dl else 20)
    b["near"] = n_src * src_b + n_ctr * (32 + 16 * kq) + n_conv * 32
    # point-and-shoot M2L: W (rotation about y), Z (z-shift) and V (rotation back) are each
    # block diagonal -- Re blocks of size 1..p+1 and Im blocks of size 1..p -- so sum(s^2)
    # multiply-adds per factor per entry (the dense 8 K_p^2 convention would be 9x larger)
    blk = sum(s * s for s in range(1, p + 2)) + sum(s * s for s in range(1, p + 1))
    f["m2l"] = led["entries"]["V"] * 2 * 3 * blk
    # compulsory: multipoles in + locals out once per box (operators ~0.6 GB amortised)
    b["m2l"] = 2 * 8 * (p + 1) ** 2 * led["n_l2l"]
    f["wfar"] = led["pairs_wfar_centre"] * (8 * kp * kq + 10 * kpq + 30) + led["pairs_wfar_target"] * (10 * kp + 30)
    b["wfar"] = n_ctr * 16 * kq * 2
    f["p2l"] = led["pairs_xfar_source"] * ((26 if dl else 10) * kp + (40 if dl else 30))
    b["p2l"] = led["entries"]["X_far"] * 16 * kp
    f["l2l"] = led["n_l2l"] * 8 * kp * kp
    b["l2l"] = led["n_l2l"] * 2 * 16 * kp
    f["l2qbxl"] = n_ctr * (8 * kp * kq + 10 * kpq + 30)
    b["l2qbxl"] = n_ctr * 16 * kq * 2
    f["eval"] = n_assoc * (10 * kq + 30) + n_conv * (10 * kp + 30)
    b["eval"] = n_assoc * (16 * kq + 24 + 4 + 8) + n_conv * (32 + 8)
    return f, b


def helm_stage_work(led, cfg, n_src, n_ctr, n_assoc, n_conv):
    """Algorithmic fp64 flops per stage of the Helmholtz (complex128) apply, real flops
    with a complex multiply-add = 8: full tables K_x = (x+1)^2; a (source, box or centre)
    pair forms K wave-function values (6 flops each from the solid-harmonic and radial
    recurrences) and K complex multiply-adds; a translation is the dense complex K x K'
    matrix-vector product the centre and tree shifts define; M2L is the point-and-shoot
    factorisation (8 x 6,181 real multiply-adds per List-2 entry at p = 20)."""
    p, q = cfg.p_fmm, cfg.p_qbx
    kp, kq = (p + 1) ** 2, (q + 1) ** 2
    pas = 2 * 8 * 6181 * ((p + 1) / 21.0) ** 3  # per List-2 entry; exact at p = 20 (config 3)
    f = {}
    f["p2m"] = led["n_p2m_sources"] * (14 * kp)
    f["m2m"] = led["n_m2m"] * 8 * kp * kp
    f["near"] = led["pairs_qbx_near"] * (14 * kq) + led["pairs_p2p_near"] * 40
    f["m2l"] = int(led["entries"]["V"] * pas)
    f["p2l"] = led["pairs_xfar_source"] * (14 * kp)
    f["l2l"] = led["n_l2l"] * 8 * kp * kp
    f["wfar"] = led["pairs_wfar_centre"] * 8 * kp * kq + led["pairs_wfar_target"] * 14 * kp
    f["l2qbxl"] = n_ctr * 8 * kp * kq
    f["eval"] = n_assoc * 14 * kq + n_conv * 14 * kp
    return f


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- CPU legs (oracle)
def host_info():
    """nproc and the lscpu model name of the host the CPU legs run on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def pick_workload(args, world):
    """(config id, geometry overrides, label) of the bench workload: BASELINE config 1 on one
    GPU; config 4 (4x4x4 urchins, strong scaling; --weak: 8 urchins per GPU) under torchrun."""
    wl = args.workload if args.workload != "auto" else ("config1" if world == 1 else "config4")
    if wl == "config1":
        if args.small:
            return 1, dict(nu=64, nv=32), "debug: torus 64x32"
        return 1, {}, ("BASELINE config 1: torus R=2 r=1, 256x128 cells, 65,536 tris x 16 nodes, "
                       "Laplace SL+DL, p_fmm=15, p_qbx=5, n_max=64, t_f=0.9")
    n = 8 * world if args.weak else 64
    return 4, dict(variant=n), (f"BASELINE config 4: {n} urchins (level 5, spacing 3.0, random rotations), "
                                f"{n * 327680} sources, Laplace SL+DL, p_fmm=15, p_qbx=5, n_max=64, t_f=0.9; "
                                + ("weak scaling, 8 urchins per GPU" if args.weak else "strong scaling"))


def workload_config(g, n_boxes, world, small=False, label=None):
    return {"workload": label or ("BASELINE config 1: torus R=2 r=1, 256x128 cells, 65,536 tris x 16 nodes, "
                                  "Laplace SL+DL, p_fmm=15, p_qbx=5, n_max=64, t_f=0.9" if not small
                                  else "debug: torus 64x32"),
            "n_sources": g.n_sources, "n_targets": g.n_targets, "n_centers": g.n_centers, "n_boxes": n_boxes,
            "parallelism": f"morton-shard x{world} (NCCL multipole broadcast)" if world > 1 else "single GPU",
            "l2": "working set (M, L 2x392 MB, QBX locals 672 MB) >> 126 MB L2; no flush"}


def cpu_oracle_throughput(steps: int, warmup: int, full: bool = False, cid: int = CONFIG_ID):
    """The CPU restatement of the path (oracle/, OpenMP over all host threads) on the
    full config-1 workload (full=True: the reference arm) or on a bounded 1/16 sample
    of it (the cpu_baseline field of the GPU line); config 4: a bounded sample of two of
    its urchins (the whole 64-urchin apply is ~30 CPU-minutes)."""
    import oracle as O
    from paper_1805_06106_b200 import api
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    if cid == 4:
        over = dict(variant=8, nx=2, ny=1, nz=1)
    else:
        over = {} if full else CPU_SAMPLE
    g = api.config_geometry(cid, **over)
    cfg = api.config_fmm(cid)
    plan = api.Plan(cfg, g)
    w, mu = g.weights(), g.dipoles()
    for _ in range(warmup):
        O.execute(plan, g, w, mu)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.execute(plan, g, w, mu)
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    units = g.n_sources + g.n_targets
    what = ("2 of the 64 urchins of BASELINE config 4 (bounded sample)" if cid == 4 else
            "full BASELINE config 1" if full else f"torus {CPU_SAMPLE['nu']}x{CPU_SAMPLE['nv']} cells, 1/16 of config 1")
    return dict(value=units / t, unit="points/s", cores=cores, kind="port",
                sample=f"{what} ({g.n_sources} sources + {g.n_targets} targets), p=15 q=5 SL+DL, oracle/ OpenMP "
                       f"restatement of Stages 2-9 on the same host plan, mean of {steps} after {warmup} warm-up",
                seconds_per_step=t, g=g, n_boxes=plan.view.n_boxes, host=host_info())


def run_reference(args, rank, world):
    """The reference arm: the CPU path timed on the box's host cores on the SAME workload
    as the GPU arm (full config 1; one oracle apply takes minutes, so at most 1 warm-up
    and 2 timed steps regardless of --steps / --warmup).  Under torchrun only rank 0 runs."""
    if rank != 0:
        return 0
    steps, warm = max(1, min(args.steps, 2)), min(max(args.warmup, 0), 1)
    cid, _, label = pick_workload(args, world)
    cb = cpu_oracle_throughput(steps, warm, full=not args.small, cid=cid)
    cfgd = workload_config(cb["g"], cb["n_boxes"], world, args.small, label)
    if cid == 4:
        cfgd["sample"] = cb["sample"]
    line = {"metric": "QBX-FMM layer-potential apply: (sources+targets)/sec", "value": cb["value"],
            "unit": "points/s", "impl": "reference", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
            "ms_per_step": cb["seconds_per_step"] * 1e3, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (procedural torus, seeded Fourier density)",
            "config": cfgd,
            "cpu_baseline": {"value": cb["value"], "unit": "points/s", "cores": cb["cores"], "kind": "port",
                             "sample": cb["sample"], **cb["host"]},
            "e2e": {"value": cb["value"], "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": ("steps/warm-up capped at 2/1: one CPU apply of the full workload takes minutes; the reference "
                     "ships no FMM code (SURVEY.md §0), so the CPU path is the oracle restatement (kind: port)")}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU leg
def measure_config4(api, torch, local_rank, steps):
    """BASELINE config 4 (64 urchins, 20,971,520 sources) on one GPU, device-resident,
    CUDA events: the N = 1 point of the strong-scaling curve."""
    t0 = time.perf_counter()
    g = api.config_geometry(4)
    cfg = api.config_fmm(4)
    plan = api.Plan(cfg, g, device="gpu")
    t1 = time.perf_counter()
    eng = api.FmmEngine(cfg, g, plan, device=local_rank)
    t2 = time.perf_counter()
    dev = torch.device("cuda", local_rank)
    d_w = torch.from_numpy(g.weights()).to(dev)
    d_mu = torch.from_numpy(g.dipoles().reshape(-1)).to(dev)
    d_pot = torch.empty(g.n_targets, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    eng.apply_device(d_w.data_ptr(), d_mu.data_ptr(), d_pot.data_ptr(), None, stream.cuda_stream)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        eng.apply_device(d_w.data_ptr(), d_mu.data_ptr(), d_pot.data_ptr(), None, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    tm, _, _, _ = eng.last_timings()
    eng.close()
    units = g.n_sources + g.n_targets
    return {"workload": "BASELINE config 4: 64 urchins, strong-scaling base (same workload as bench.py --gpus N)",
            "n_sources": g.n_sources, "n_targets": g.n_targets, "n_boxes": plan.view.n_boxes,
            "ms_per_apply": round(ms, 2), "value": units / (ms * 1e-3), "unit": "points/s", "steps": steps,
            "stages_ms": {k: round(v, 2) for k, v in tm.items()},
            "setup_s": {"geometry_and_gpu_plan": round(t1 - t0, 2), "create": round(t2 - t1, 2)}}



def run_ours(args, rank, world, local_rank):
    import torch
    from paper_1805_06106_b200 import api

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    t0 = time.perf_counter()
    cid, over, label = pick_workload(args, world)
    g = api.config_geometry(cid, **over)
    cfg = api.config_fmm(cid)
    side = world == 1 and cid == 1  # single-GPU side measurements ride on the config-1 run
    t1 = time.perf_counter()
    plan = api.Plan(cfg, g)
    t2 = time.perf_counter()
    if world > 1:
        # Morton-range shard of the boxes per rank; multipoles exchanged with NCCL
        # broadcasts over NVLink inside qbxg_apply_device
        eng = api.FmmEngine(cfg, g, plan, device=local_rank, shard=(world, rank))
        uid = [api.FmmEngine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.attach_nccl(uid[0])
    else:
        eng = api.FmmEngine(cfg, g, plan, device=local_rank)
    t3 = time.perf_counter()
    # Stage 1 on the GPU (qbxg_plan_create_gpu): same plan bit for bit
    plan_gpu = None
    if side:
        api.Plan(cfg, g, device="gpu")  # warm-up (CUB kernels, allocator)
        tg = time.perf_counter()
        pg = api.Plan(cfg, g, device="gpu")
        tg = time.perf_counter() - tg
        ha, ga = plan.arrays(), pg.arrays()
        same_plan = pg.list_hashes() == plan.list_hashes() and all(np.array_equal(ha[k], ga[k]) for k in ha)
        plan_gpu = {"total": round(tg, 4), "tree": round(pg.view.build_seconds_tree, 4),
                    "lists": round(pg.view.build_seconds_lists, 4), "bitwise_equal_to_host": bool(same_plan)}
        del pg
    led = plan.ledger()
    w, mu = g.weights(), g.dipoles()
    dev = torch.device("cuda", local_rank)
    d_w = torch.from_numpy(w).to(dev)
    d_mu = torch.from_numpy(mu.reshape(-1)).to(dev)
    d_pot = torch.empty(g.n_targets, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        eng.apply_device(d_w.data_ptr(), d_mu.data_ptr(), d_pot.data_ptr(), None, stream.cuda_stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)

    stage_ms = {}
    launches = 0
    clk = ClockSampler(local_rank)
    clk.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        tm, nl, _, _ = eng.last_timings()
        launches += nl
        for k, v in tm.items():
            stage_ms[k] = stage_ms.get(k, 0.0) + v
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    # per-stage CUDA-event times (the engine's own events, over the same timed steps; for a
    # sharded apply the near field runs on a side stream beside the exchange and M2L)
    ms_seq = ms
    for k in stage_ms:
        stage_ms[k] /= args.steps
    units = g.n_sources + g.n_targets
    value = units / (ms * 1e-3)  # the whole problem, split across ranks (strong scaling)

    # end to end through the public C-ABI call with pinned host buffers
    hw = torch.from_numpy(w).pin_memory().numpy()
    hmu = torch.from_numpy(mu).pin_memory().numpy()
    e2e_times = []
    for i in range(args.steps + 1):
        if dist:
            dist.barrier()
        ta = time.perf_counter()
        pot = eng.apply(hw, hmu)
        tb = time.perf_counter()
        if i > 0:
            e2e_times.append(tb - ta)
    _, _, h2d, d2h = eng.last_timings()
    e2e_t = torch.tensor([float(np.mean(e2e_times))], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = units / float(e2e_t.item())
    # sanity: device-resident and host paths agree bitwise
    same = bool(np.array_equal(pot, d_pot.cpu().numpy()))

    # batched densities (qbxg_apply_batch_device): device time per density
    batch = None
    if side and not args.small:
        R = 4
        rng = np.random.default_rng(5)
        dens = rng.uniform(-1.0, 1.0, (R, g.n_sources))
        bW = torch.from_numpy(np.stack([g.weights(d) for d in dens])).to(dev)
        bMU = (torch.from_numpy(np.stack([g.dipoles(d) for d in dens]).reshape(R, -1)).to(dev)
               if cfg.kernel == 1 else None)
        bP = torch.empty((R, g.n_targets), dtype=torch.float64, device=dev)
        bt = []
        for i in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            eng.apply_batch_device(R, bW.data_ptr(), bMU.data_ptr() if bMU is not None else None, bP.data_ptr(),
                                   None, stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize()
            if i > 0:
                bt.append(e0.elapsed_time(e1))
        bms = float(np.mean(bt)) / R
        batch = {"n_rhs": R, "ms_per_density": round(bms, 3), "value": units / (bms * 1e-3), "unit": "points/s",
                 "note": ("SL+DL: densities run one by one on the resident plan (the single-density near field is cheaper "
                          "per density than a shared harmonic table plus a contraction per density)"
                          if cfg.kernel == 1 else
                          "near field shares one harmonic table per (centre, source) pair between 2 densities")}

    # roofline of the dominant kernel, per-stage fractions
    peak = api.measure_fp64_peak(local_rank)
    peak_dmma = api.measure_dmma_peak(local_rank)
    n_assoc = int((g.association >= 0).sum())
    flops, bytes_ = stage_work(led, cfg, g.n_sources, g.n_centers, n_assoc, g.n_targets - n_assoc)
    with open(os.path.join(HERE, "MEASURED_PEAKS.json")) if os.path.exists(os.path.join(HERE, "MEASURED_PEAKS.json")) else open(os.devnull) as fh:
        try:
            mp = json.load(fh)
        except Exception:
            mp = {}
    hbm = float(mp.get("hbm_gbs", 6548.8))
    stages = {}
    for k in flops:
        t = stage_ms.get(k, 0.0) * 1e-3
        if t <= 0:
            continue
        tf = flops[k] / t / 1e12
        gbs = bytes_[k] / t / 1e9
        tensor = k in ("m2l", "m2m", "l2l")  # DMMA GEMMs on the fp64 tensor pipe
        pk = peak_dmma if tensor else peak
        stages[k] = {"ms": round(stage_ms[k], 4), "tflops": round(tf, 3), "frac_fp64": round(tf / pk, 4),
                     "pipe": "dmma" if tensor else "dfma",
                     "gbs": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4), "flops": flops[k]}
    dom = max(stages, key=lambda k: stages[k]["ms"])
    d = stages[dom]
    traffic, traffic_note = None, None
    tp = next((os.path.join(HERE, "profiles", f"r0{r}_ncu_{dom}.json") for r in (2, 1)
               if os.path.exists(os.path.join(HERE, "profiles", f"r0{r}_ncu_{dom}.json"))), "")
    if tp and cid == 1 and not args.small:
        with open(tp) as fh:
            t = json.load(fh)
        # one ncu --set full capture of the stage's main kernel; bytes per launch
        traffic = (t["dram_read_GB"] + t["dram_write_GB"]) * 1e9
        traffic_note = f"dram bytes of one launch of {t['kernel']} ({os.path.relpath(tp, HERE)}); {t.get('note', '')}"
    roofline = {"bound": "tensor" if dom == "m2l" else "fp64", "kernel": dom, "achieved": d["tflops"],
                "peak": round(peak_dmma if dom == "m2l" else peak, 3), "unit": "TFLOP/s",
                "frac": d["frac_fp64"], "traffic": traffic, "traffic_note": traffic_note,
                "peak_source": "in-run microbenchmarks (qbxg_measure_fp64_peak DFMA = %.1f, qbxg_measure_dmma_peak "
                               "DMMA = %.1f TFLOP/s); MEASURED_PEAKS.json has no fp64 entry" % (peak, peak_dmma),
                "algorithmic_flops_per_launch": flops[dom], "share_of_step": round(d["ms"] / ms_seq, 3),
                "stage_timing": "the engine's CUDA events per stage over the K timed steps (%.2f ms/step)" % ms}

    cpu = None
    if rank == 0 and side and not args.no_cpu_baseline:
        cb = cpu_oracle_throughput(1, 0)
        cpu = {**{k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}, **cb["host"]}

    # BASELINE config 4 (64 urchins) on this one GPU: the base of the strong-scaling curve
    # that bench.py --gpus N (torchrun) measures at N = 2, 4, 8 on the same workload
    c4 = None
    if side and not args.small and not args.no_config4:
        eng.close()
        eng = None
        c4 = measure_config4(api, torch, local_rank, max(2, min(args.steps, 3)))

    # BASELINE config 3 (Helmholtz single layer, k = 3, p = 20, q = 5) on the same GPU:
    # side measurement, CUDA events, inputs on the host (qbxg_apply_complex)
    helm = None
    if side and not args.small and not args.no_helmholtz:
        if eng is not None:
            eng.close()
            eng = None
        g3 = api.config_geometry(3)
        cfg3 = api.config_fmm(3)
        rng3 = np.random.default_rng(7)
        w3 = g3.quad_weight * (rng3.uniform(-1, 1, g3.n_sources) + 1j * rng3.uniform(-1, 1, g3.n_sources))
        plan3 = api.Plan(cfg3, g3)
        eng3 = api.FmmEngine(cfg3, g3, plan3)
        eng3.apply_complex(w3)
        hms, hst = [], {}
        for _ in range(2):
            eng3.apply_complex(w3)
            tm3, _, _, _ = eng3.last_timings()
            hms.append(tm3["total"])
            for k, v in tm3.items():
                hst[k] = hst.get(k, 0.0) + v / 2
        eng3.close()
        hms = float(np.mean(hms))
        n3a = int((g3.association >= 0).sum())
        hf = helm_stage_work(plan3.ledger(), cfg3, g3.n_sources, g3.n_centers, n3a, g3.n_targets - n3a)
        hstages = {}
        for k, fl in hf.items():
            t = hst.get(k, 0.0) * 1e-3
            if t <= 0:
                continue
            tensor = k == "m2l"  # point-and-shoot blocks on DMMA; the rest on the FP64 pipe
            pk = peak_dmma if tensor else peak
            hstages[k] = {"ms": round(hst[k], 3), "tflops": round(fl / t / 1e12, 3),
                          "frac_fp64": round(fl / t / 1e12 / pk, 4), "pipe": "dmma" if tensor else "dfma",
                          "flops": fl}
        helm = {"workload": "BASELINE config 3: unit-sphere icosphere L=6, 1,310,720 sources, 2,621,440 centres "
                            "and targets, Helmholtz SL k=3, complex density, p_fmm=20, p_qbx=5",
                "ms_per_apply": round(hms, 2), "value": (g3.n_sources + g3.n_targets) / (hms * 1e-3),
                "unit": "points/s", "dtype": "c128", "stages": hstages,
                "work_model": "bench.helm_stage_work: real flops, complex multiply-add = 8",
                "parity": "GPU vs complex128 oracle <= 1e-11 (tests/test_helmholtz.py); no reference exists"}

    # target association (Algorithm 3) on BASELINE config 2: 655,360
    # on-surface nodes + the retained volume targets, device-resident, CUDA events
    assoc = None
    if side and not args.small and not args.no_helmholtz:
        g2 = api.config_geometry(2)
        sc2 = api.Geometry(source_pos=g2.source_pos, center_pos=g2.center_pos, center_radius=g2.center_radius,
                           target_pos=np.zeros((0, 3)), association=np.zeros(0, dtype=np.int32))
        ns2 = 2 * g2.n_sources
        sp2 = np.r_[np.where(np.arange(ns2) % 2 == 0, 1, -1), np.zeros(g2.n_targets - ns2)].astype(np.int8)
        loc = api.Locator(api.Plan(api.config_fmm(2), sc2), sc2, api.danger_radius_of(g2),
                          np.where(np.arange(g2.n_centers) % 2 == 0, 1, -1).astype(np.int8))
        dT = torch.from_numpy(g2.target_pos.copy()).to(dev)
        dS = torch.from_numpy(sp2).to(dev)
        dA = torch.empty(g2.n_targets, dtype=torch.int32, device=dev)
        dC = torch.zeros(1, dtype=torch.int64, device=dev)
        cs = torch.cuda.current_stream()
        run = lambda: loc.associate_device(g2.n_targets, dT.data_ptr(), 0.05, dS.data_ptr(), dA.data_ptr(),  # noqa
                                           dC.data_ptr(), cs.cuda_stream)
        for _ in range(3):
            run()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(cs)
        for _ in range(10):
            run()
        eb.record(cs)
        torch.cuda.synchronize()
        ams = ea.elapsed_time(eb) / 10
        a2 = dA.cpu().numpy()
        assoc = {"workload": "BASELINE config 2 targets (655,360 on-surface with side preference + retained volume "
                             "targets), eps_ta=0.05, danger radius = panel expansion radius",
                 "n_targets": int(g2.n_targets), "ms": round(ams, 4), "value": g2.n_targets / (ams * 1e-3),
                 "unit": "targets/s", "n_flagged": int(dC.item()), "n_conventional": int((a2 == -1).sum()),
                 "parity": "bit-exact vs brute-force oracle (tests/test_association.py)"}
        loc.close()

    if rank == 0:
        line = {"metric": "QBX-FMM layer-potential apply: (sources+targets)/sec", "value": value,
                "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
                "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (procedural torus, seeded Fourier density)",
                "config": workload_config(g, plan.view.n_boxes, world, args.small, label),
                "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": launches, "roofline": roofline, "stages": stages, "clocks": clocks,
                "batch": batch, "config4_one_gpu": c4, "helmholtz": helm, "association": assoc,
                "cpu_baseline": cpu,
                "setup_s": {"geometry": round(t1 - t0, 3), "tree": round(plan.view.build_seconds_tree, 3),
                            "lists": round(plan.view.build_seconds_lists, 3), "upload": round(t3 - t2, 3),
                            "plan_gpu": plan_gpu},
                "list_hashes": {k: f"{v:016x}" for k, v in plan.list_hashes().items()},
                "host_device_bitwise_equal": same}
        print(json.dumps(line), flush=True)
    if eng is not None:
        eng.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
