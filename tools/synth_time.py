"""Device synthesis timing (development tool): CUDA-event time of
synthesize_device for a few C4/C5 shapes, demo template.
Usage: python tools/synth_time.py [n N ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2003_08011_b200.signals import SignalSpec, synthesize_device  # noqa: E402

args = [int(a) for a in sys.argv[1:]] or [1000, 1000000, 100, 1000000, 1000, 16000, 10, 10000]
for n, N in zip(args[0::2], args[1::2]):
    spec = SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 20260810)
    x = synthesize_device(spec)  # warm
    del x
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    ms = []
    for _ in range(reps):
        a.record()
        x = synthesize_device(spec)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        del x
    best = min(ms)
    gbs = n * N * 8 / best / 1e6
    print(f"n={n:5d} N={N:8d}  {best:8.3f} ms  ({n * N / best / 1e6:.2f} Gsamples/s, {gbs:.0f} GB/s of output)")
