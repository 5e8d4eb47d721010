"""Target association (Algorithm 3) on BASELINE config 2 at full size: 655,360
on-surface nodes (with side preferences) + the retained volume targets, on the
tree of the sources and centres.  Device-resident timing with CUDA events on the
launching stream, plus the host-buffer call timed by wall clock."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_06106_b200 import api  # noqa: E402


def main(steps=10, warmup=3):
    g = api.config_geometry(2)
    side = np.where(np.arange(g.n_centers) % 2 == 0, 1, -1).astype(np.int8)
    nsurf = 2 * g.n_sources
    sp = np.r_[np.where(np.arange(nsurf) % 2 == 0, 1, -1), np.zeros(g.n_targets - nsurf)].astype(np.int8)
    sc = api.Geometry(source_pos=g.source_pos, center_pos=g.center_pos, center_radius=g.center_radius,
                      target_pos=np.zeros((0, 3)), association=np.zeros(0, dtype=np.int32))
    t0 = time.time()
    plan = api.Plan(api.config_fmm(2), sc)
    t1 = time.time()
    loc = api.Locator(plan, sc, api.danger_radius_of(g), side)
    t2 = time.time()
    dev = torch.device("cuda:0")
    dt = torch.from_numpy(g.target_pos.copy()).to(dev)
    ds = torch.from_numpy(sp).to(dev)
    out = torch.empty(g.n_targets, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        loc.associate_device(g.n_targets, dt.data_ptr(), 0.05, ds.data_ptr(), out.data_ptr(), cnt.data_ptr(),
                             st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        loc.associate_device(g.n_targets, dt.data_ptr(), 0.05, ds.data_ptr(), out.data_ptr(), cnt.data_ptr(),
                             st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    a = out.cpu().numpy()
    tw = time.time()
    a2, nf = loc.associate(g.target_pos, 0.05, side_pref=sp)
    tw = time.time() - tw
    assert np.array_equal(a, a2)
    print(json.dumps(dict(workload="config 2 association", n_targets=int(g.n_targets), n_surface=int(nsurf),
                          ms_device=round(ms, 3), targets_per_s=round(g.n_targets / ms * 1e3),
                          ms_host_call=round(tw * 1e3, 2), n_flagged=nf, n_conventional=int((a == -1).sum()),
                          plan_s=round(t1 - t0, 2), locator_create_s=round(t2 - t1, 3))))
    loc.close()


if __name__ == "__main__":
    main()
