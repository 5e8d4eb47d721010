"""Per-rank device work of a sharded apply, measured on ONE B200 (no interconnect involved).

    python tools/shard_times.py <config_id> <n_ranks> [reps] [key=value geometry overrides]

The N ranks of a Morton-range sharded apply are N handles in one process,
driven phase by phase: phase 1 (gather, P2M, M2M of the rank's subtrees) for every rank,
the multipole exchange as device copies (qbxg_exchange_local), phase 2 (straddle M2M,
Stages 3-9 for the rank's boxes) for every rank, then the result gather.  Each phase of
each rank is timed with CUDA events on the stream it runs on, alone on the GPU -- what a
rank's own GPU would spend on it.  Prints one JSON line: per-rank ms, the maximum over
ranks (the device critical path of an N-GPU apply without the exchange), the load
imbalance, the bytes each exchange moves, and whether every rank ends bitwise equal to
the unsharded apply.  This is NOT a multi-GPU measurement: no NCCL transfer is timed.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_1805_06106_b200 import api  # noqa: E402


def main():
    cid, n = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    over = {}
    for a in sys.argv[4:]:
        k, v = a.split("=")
        over[k] = int(v)
    g = api.config_geometry(cid, **over)
    cfg = api.config_fmm(cid)
    plan = api.Plan(cfg, g)
    dev = torch.device("cuda", 0)
    w, mu = g.weights(), g.dipoles() if cfg.kernel == 1 else None
    dw = torch.from_numpy(w).to(dev)
    dm = torch.from_numpy(mu.reshape(-1)).to(dev) if mu is not None else None
    mp = dm.data_ptr() if dm is not None else None
    torch.cuda.synchronize(dev)
    stream = torch.cuda.Stream(dev)  # non-default: the handle launches on it, the events bracket the kernels

    ref = api.FmmEngine(cfg, g, plan)
    p1 = torch.empty(g.n_targets, dtype=torch.float64, device=dev)
    ms1 = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ref.apply_device(dw.data_ptr(), mp, p1.data_ptr(), None, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms1.append(e0.elapsed_time(e1))
    single_ms = float(np.mean(ms1[1:]))
    pot1 = p1.cpu().numpy()
    ref.close()

    engines, per_engine = [], 0
    for r in range(n):  # bounded memory: stop before the next handle would not fit
        free0 = torch.cuda.mem_get_info(dev)[0]
        if per_engine and free0 < 1.3 * per_engine + (8 << 30):
            print(json.dumps({"tool": "shard_times", "config": cid, "n_ranks": n, "skipped":
                              f"handle {r} of {n} would not fit: {free0 >> 30} GiB free, {per_engine >> 30} GiB per handle"}))
            return
        engines.append(api.FmmEngine(cfg, g, plan, shard=(n, r)))
        per_engine = max(per_engine, free0 - torch.cuda.mem_get_info(dev)[0])
    pots = [torch.empty(g.n_targets, dtype=torch.float64, device=dev) for _ in range(n)]
    _, row, cuts = engines[0].multipole_buffer()
    t = np.zeros((reps + 1, 2, n))

    def timed(e, phase, pot):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e.apply_phase(phase, dw.data_ptr(), mp, pot, None, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    for k in range(reps + 1):
        for r, e in enumerate(engines):
            t[k, 0, r] = timed(e, 1, None)
        api.exchange_local(engines)
        for r, (e, p) in enumerate(zip(engines, pots)):
            t[k, 1, r] = timed(e, 2, p.data_ptr())
    api.exchange_results_local(engines, [p.data_ptr() for p in pots], None)
    torch.cuda.synchronize(dev)
    same = all(np.array_equal(p.cpu().numpy(), pot1) for p in pots)
    d = np.abs(pots[0].cpu().numpy() - pot1)
    ndiff, maxdiff = int((d != 0).sum()), float(d.max() / np.abs(pot1).max())
    for e in engines:
        e.close()
    ph = t[1:].mean(axis=0)  # first round is warm-up
    per_rank = ph.sum(axis=0)
    crit = float(ph[0].max() + ph[1].max())
    nb = plan.view.n_boxes
    out = {
        "tool": "shard_times", "config": cid, "overrides": over, "n_ranks": n, "reps": reps,
        "n_sources": g.n_sources, "n_targets": g.n_targets, "n_boxes": nb,
        "single_gpu_ms": round(single_ms, 3),
        "phase1_ms_per_rank": [round(float(x), 3) for x in ph[0]],
        "phase2_ms_per_rank": [round(float(x), 3) for x in ph[1]],
        "device_critical_path_ms": round(crit, 3),
        "device_speedup_vs_single": round(single_ms / crit, 3),
        "device_efficiency": round(single_ms / crit / n, 3),
        "imbalance_max_over_mean": round(float(per_rank.max() / per_rank.mean()), 3),
        "redundant_work_sum_over_single": round(float(per_rank.sum() / single_ms), 3),
        "multipole_exchange_bytes_total": int(nb) * int(row) * 8,
        "result_gather_bytes_total": int(g.n_targets) * 8,
        "box_cuts": [int(c) for c in cuts],
        "device_gib_per_handle": round(per_engine / 2**30, 1),
        "bitwise_equal_to_single": bool(same), "n_targets_differing": ndiff, "max_rel_diff": maxdiff,
        "note": ("ranks emulated one after another on one B200: per-rank kernel time only; the NCCL "
                 "exchanges (sizes above; 900 GB/s per direction over NVLink 5) are not timed"),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
