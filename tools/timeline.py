"""Per-warp event timeline of the fused surveillance kernel (CTA 0).

Needs the instrumented library (tools/build_timeline.sh -> -DCSB_TIMELINE).
  CSB_LIB=tools/libcstress_b200_tl.so python tools/timeline.py [n m N]
Prints, per warp role, the mean cycles spent in each phase between
consecutive events, plus a raw excerpt.  Development tool.
"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CSB_LIB", os.path.join(ROOT, "tools", "libcstress_b200_tl.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_08011_b200 as p  # noqa: E402

CAP = 8192
NAMES = {1: "g1.enter", 2: "g1.issue", 3: "g2.enter", 4: "g2.issue",
         10: "epi.acc_wait", 11: "epi.acc_got", 12: "epi.computed", 13: "epi.sfree_got", 14: "epi.stored",
         20: "pro.enter", 21: "pro.xfree_got", 22: "pro.done", 23: "rd.ofull_wait", 24: "rd.ofull_got",
         25: "rd.done", 26: "rd.gathered", 27: "rd.looped", 40: "pro.loaded", 42: "pro.stored", 43: "pro.barrier", 44: "rd.tmem1", 45: "pro.xa_got", 46: "epi.acc_loaded", 30: "prod.dn_wait", 31: "prod.dn_got", 33: "prod.p_got"}
SLOTS = {0: "producer", 1: "mma g1", 2: "epi set0", 3: "epi set1", 4: "mma g2"}


def main():
    nums = [a for a in sys.argv[1:] if not a.startswith("--")]
    n, m, N = (int(a) for a in nums[:3]) if len(nums) >= 3 else (100, 1000, 100_000)
    dev = torch.device("cuda", 0)
    X = p.synthesize(p.SignalSpec.uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 1)).data
    obs = p.synthesize(p.SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 2)).data
    g = p.train(X, m, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
    d_obs = torch.tensor(obs.T.astype(np.float32), device=dev).T
    d_est = torch.empty_like(d_obs.T).T
    d_res = torch.empty_like(d_obs.T).T
    st = torch.cuda.current_stream(dev)
    for _ in range(3):
        p.estimate_device(g, d_obs, d_est, d_res, st)
    out = os.path.join(ROOT, "gpurun_out", "timeline.bin")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    os.environ["CSB_TIMELINE_OUT"] = out
    p.estimate_device(g, d_obs, None if "--no-est" in sys.argv else d_est,
                      None if "--no-out" in sys.argv else d_res, st)
    torch.cuda.synchronize()
    raw = np.fromfile(out, dtype=np.uint64).reshape(5, CAP * 2)
    t0 = None
    for s in range(5):
        cnt = int(raw[s, 0])
        recs = raw[s, 2:2 + 2 * min(cnt, CAP - 1)].reshape(-1, 2)
        if len(recs) and (t0 is None or recs[0, 1] < t0):
            t0 = int(recs[0, 1])
    total_end = 0
    for s in range(5):
        cnt = int(raw[s, 0])
        recs = raw[s, 2:2 + 2 * min(cnt, CAP - 1)].reshape(-1, 2)
        ev = (recs[:, 0] >> 32).astype(int)
        jj = (recs[:, 0] & 0xFFFFFFFF).astype(int)
        tt = recs[:, 1].astype(np.int64) - t0
        if len(tt):
            total_end = max(total_end, int(tt[-1]))
        phase = collections.defaultdict(list)
        for k in range(len(ev) - 1):
            phase[(ev[k], ev[k + 1])].append(int(tt[k + 1] - tt[k]))
        print(f"== {SLOTS[s]}: {len(ev)} events")
        for (a, b), v in sorted(phase.items(), key=lambda kv: -sum(kv[1])):
            print(f"   {NAMES.get(a, a):>15} -> {NAMES.get(b, b):<15} n={len(v):5d} mean={np.mean(v):8.0f} "
                  f"total={sum(v):9d}")
        # excerpt: second tile
        sel = np.nonzero((tt > 0))[0][:0]
        lines = [f"{int(tt[k]):9d} {NAMES.get(ev[k], ev[k])}({jj[k]})" for k in range(min(len(ev), 140))]
        if "--raw" in sys.argv:
            print("\n".join(lines))
    print(f"kernel span (CTA 0, first->last event): {total_end} cycles")
    if "--merged" in sys.argv:
        # all roles interleaved in time over a window of the run
        allev = []
        for s in range(5):
            cnt = int(raw[s, 0])
            recs = raw[s, 2:2 + 2 * min(cnt, CAP - 1)].reshape(-1, 2)
            for e, c in recs:
                allev.append((int(c) - t0, SLOTS[s], NAMES.get(int(e) >> 32, int(e) >> 32), int(e) & 0xFFFFFFFF))
        allev.sort()
        lo, hi = total_end // 3, total_end // 3 + 60000
        prev = None
        for c, who, what, j in allev:
            if lo <= c <= hi:
                print(f"{c:9d} {'' if prev is None else f'+{c - prev:6d}'} {who:9s} {what}({j})")
                prev = c


if __name__ == "__main__":
    main()
