import sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
from paper_2308_01651_b200 import configs
from paper_2308_01651_b200.simulation import TissueSolver
ns = configs.this_package(); cfg = configs.config2(ns)
s = TissueSolver(cfg); payload = s.checkpoint_payload()
for _ in range(3): s.enqueue_step()
s.sync()
s2 = TissueSolver(cfg)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); s2.restore(payload); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"restore {1e3*(t1-t0):.2f} ms ({len(payload)/1e6:.1f} MB)")
pidx = torch.tensor([0, 100, 1000], device="cuda")
pinned = torch.empty((300, 5), dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(200):
    s2.enqueue_step(); s2.record_row(pidx, pinned[k])
t1 = time.perf_counter(); s2.sync(); t2 = time.perf_counter()
print(f"host enqueue {1e6*(t1-t0)/200:.1f} us/step, total {1e3*(t2-t0)/200:.3f} ms/step")
