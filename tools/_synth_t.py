import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2003_08011_b200 as p
for (n, N) in [(1000, 1000000), (100, 1000000), (1000, 100000), (20, 10000)]:
    spec = p.SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 7)
    p.synthesize_device(spec, 0); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): x = p.synthesize_device(spec, 0)
    torch.cuda.synchronize()
    print(n, N, f"{(time.perf_counter()-t)/3*1e3:.2f} ms", flush=True)
    del x
