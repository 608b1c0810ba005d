import sys, time, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2510_02080_b200 import synth, loops, _lib
pooled = synth.pooled_embeddings(4000, seed=4000)
loops.retrieval_device(pooled, 5, 15, 0.93, 0.96)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    loops.retrieval_device(pooled, 5, 15, 0.93, 0.96)
torch.cuda.synchronize()
print("total ms", (time.perf_counter() - t0) / 5 * 1e3)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    loops.retrieval_device(pooled, 5, 15, 0.93, 0.96)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
