"""Device time of one pass (graph mode, 50 replays) per config.

    python tools/diag_time.py c2 c1b

With a diagnostics build of libtc (TC_LIBTC=...) whose k_stream / k_stream_pair
(TC_DIAG_EMPTY=1) or every kernel (=2) return at entry when the env var is set
(a `__device__ int` flag copied at Exec build; not part of the product
library), it separates the graph's launch floor from the kernel bodies
(profiles/r2b_diag_empty.txt).
"""
import sys, os
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import bench
from paper_2006_15512_b200 import _lib
for name in sys.argv[1:]:
    spec = bench.CONFIGS[name]
    flat, _ = bench.load_plan(spec["plan"])
    h, ch = bench.choose(flat, spec["slices"])
    ex = _lib.Exec(h, ch, 0)
    ex.run(0, 1); ex.run(0, 1, repeats=3)
    st = ex.run(0, 1, repeats=50)
    print(name, os.environ.get('TC_DIAG_EMPTY','-'), 'ms/pass %.4f' % (st['device_ms'] / 50), 'launches', st['gpu_launches'] // 50 if st['gpu_launches'] else None, flush=True)
