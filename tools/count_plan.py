import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2006_15512_b200 import planfile, sliced_execute, _lib
for name in sys.argv[1:]:
    fl,_=planfile.load(f'data/plans/{name}.tcplan.npz')
    n,t=planfile.to_objects(fl)
    r=sliced_execute(n,t)
    print(name, float(np.asarray(r.result.values)), r.stats['device_ms'], flush=True)
