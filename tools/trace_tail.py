"""Tail of the last edge-stream gather launch of a run (PRGPU_TRACE output):
per-warp start / end globaltimer stamps -> ramp, busy and tail times.
Usage: PRGPU_TRACE=/tmp/t.txt python tools/prof_run.py 4 phased 3; python tools/trace_tail.py /tmp/t.txt"""
import sys

import numpy as np

a = np.loadtxt(sys.argv[1], dtype=np.float64).reshape(-1, 2)
a = a[a[:, 1] > 0]
t0 = a[:, 0].min()
s, e = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
busy = e - s
print(f"warps {len(a)}  first start 0  last start {s.max():.2f} us  last end {e.max():.2f} us")
print(f"end percentiles (us): p0 {np.percentile(e, 0):.1f} p10 {np.percentile(e, 10):.1f} p50 {np.median(e):.1f} "
      f"p90 {np.percentile(e, 90):.1f} p99 {np.percentile(e, 99):.1f} max {e.max():.1f}")
print(f"busy mean {busy.mean():.1f} us; tail (max end - median end) {e.max() - np.median(e):.1f} us; "
      f"mean idle after own end {np.mean(e.max() - e):.1f} us")
sm = np.arange(len(a)) // 32
per_sm = np.array([e[sm == i].max() for i in range(sm.max() + 1)])
print(f"per-CTA last end: min {per_sm.min():.1f} median {np.median(per_sm):.1f} max {per_sm.max():.1f} us")
