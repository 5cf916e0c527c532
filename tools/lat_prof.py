import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2601_05816_b200 as P
from paper_2601_05816_b200.device import upload
from torch.profiler import profile, ProfilerActivity
dims, b = (8, 8, 8, 8), 4
geom = P.LatticeGeometry(dims)
gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 1))
eta = upload(P.gen_spinor(geom.n_sites, b, 2, seed=2, geom=geom))
cfg = P.GmresConfig(restart_len=30, restarts=67, tol=1e-10)
P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    rep = P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta, cfg)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
print("n cuda events", len(evs), "busy us", sum(e.time_range.elapsed_us() for e in evs),
      "span us", evs[-1].time_range.end - evs[0].time_range.start)
for e in evs[200:260]:
    print(f"{e.time_range.start - evs[200].time_range.start:9.1f} {e.time_range.elapsed_us():7.1f} {e.name[:70]}")
