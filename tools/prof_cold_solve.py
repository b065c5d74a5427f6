import sys, time
sys.path.insert(0, "/root/repo")
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2409_14309_b200 as E
from paper_2409_14309_b200 import workloads as W
c = W.config(2)
A, b, _ = W.make_problem(c, backend="torch")
prob = E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b))
spec, opts = E.SketchSpec("countsketch", 1, seed=W.SEED), E.SolverOptions(d_factor=c.d / c.n)
for _ in range(3):
    E.clear_operator_cache(); E.solve(prob, "saa", spec, opts)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    E.clear_operator_cache()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    E.solve(prob, "saa", spec, opts)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("cold solve ms", sorted(ts)[5] * 1e3)
E.clear_operator_cache()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    E.solve(prob, "saa", spec, opts)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=50))
