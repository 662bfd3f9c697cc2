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
