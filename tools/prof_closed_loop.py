"""One closed-loop call on a C4-shaped workload with fewer intervals (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2403_12900_b200.runner import Sweep
T = int(sys.argv[1]) if len(sys.argv) > 1 else 240
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
w = synth.make_workload("C4", n_requests=(10**9 * T) // 8760, n_intervals=T)
sh = synth.shard(w.spec, 1, 0)
sw = Sweep(w.prob, w.cost, sh, "cuda:0", spec=w.spec)
sw.closed_loop(W)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sw.closed_loop(W); e1.record(); torch.cuda.synchronize()
print("T", T, "W", W, "ms", e0.elapsed_time(e1), "-> full-year estimate ms", e0.elapsed_time(e1) * 8760 / T)
