"""Host submission cost per decode step (diagnostic): runs bench.py with the
decoder's per-step calls wrapped in perf_counter timers and prints where the
host time goes (Python mirror vs the C-ABI call).  Usage:
    python tools/host_cost.py --workload cfg1 --steps 300 --warmup 5"""
import atexit
import os
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2601_13684_b200 import decoder as D  # noqa: E402

acc = defaultdict(float)
cnt = defaultdict(int)


def wrap(cls, name):
    f = getattr(cls, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        acc[name] += time.perf_counter() - t0
        cnt[name] += 1
        return r
    setattr(cls, name, g)


if os.environ.get("HC_BENCH_NO_TIMING") == "1":  # the production path: no phase events
    _kt = D.HeteroCacheDecoder.kernel_timing
    D.HeteroCacheDecoder.kernel_timing = lambda self, enable=True, light=False: _kt(self, False)

for n in ("decode_step", "decode_step_host", "_dd_after_step", "_dd_poll"):
    wrap(D.HeteroCacheDecoder, n)


@atexit.register
def report():
    for n in acc:
        print(f"host_cost {n}: {cnt[n]} calls, {acc[n] / max(1, cnt[n]) * 1e6:.1f} us/call",
              file=sys.stderr)


if __name__ == "__main__":
    sys.argv = ["bench.py"] + sys.argv[1:]
    bench.main()
