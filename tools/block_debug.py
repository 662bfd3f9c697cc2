"""One-shot vs repeated passes of a sliced config through the Python Exec:
per-slice results must be identical (debugging the block tier)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2006_15512_b200 import _lib  # noqa: E402
import torch  # noqa: E402

name = sys.argv[1]
b, e = int(sys.argv[2]), int(sys.argv[3])
spec = bench.CONFIGS[name]
flat, _ = bench.load_plan(spec["plan"])
h, ch = bench.choose(flat, spec["slices"])


def per_slice(ex):
    out = torch.empty((e - b, ex.result_size()), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ex.copy_results(out.data_ptr())
    return out.cpu().numpy()[:, 0]


ex = _lib.Exec(h, ch, 0)
ex.run(b, e)
one = per_slice(ex)
ex.run(b, e, repeats=3)
rep = per_slice(ex)
ok = np.array_equal(one, rep)
import hashlib  # noqa: E402
print(name, b, e, {k: os.environ.get(k) for k in ("TC_BLOCK", "TC_SLICE_ORDER", "TC_LANES", "TC_OVERLAP_BUILD")},
      "hash", hashlib.sha1(rep.tobytes()).hexdigest()[:12], "equal", ok,
      "bad slices", np.nonzero(one != rep)[0][:16].tolist(), "nonzero one/rep", int((one != 0).sum()), int((rep != 0).sum()))
