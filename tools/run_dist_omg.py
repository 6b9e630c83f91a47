"""torchrun --nproc-per-node W tools/run_dist_omg.py <fixture> [tol] [backend]"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
backend = sys.argv[3] if len(sys.argv) > 3 else "gloo"
dist.init_process_group(backend)
rank = dist.get_rank()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
from paper_2003_02431_b200.dist_solvers import dist_ortho_mg_solve  # noqa: E402
from paper_2003_02431_b200.hierarchy import load_hierarchy  # noqa: E402
from paper_2003_02431_b200.solvers import SolverConfig  # noqa: E402

z = np.load(sys.argv[1])
meta = json.loads(bytes(z["meta"]).decode())
cfgd = dict(meta["omg"])
if len(sys.argv) > 2:
    cfgd["tolerance"] = float(sys.argv[2])
hier = load_hierarchy(z)
t0 = time.time()
x, (r0, r1), rep = dist_ortho_mg_solve(hier, np.asarray(hier.level(1).rhs), SolverConfig(**cfgd))
print(f"rank {rank}: rows [{r0},{r1}) it={rep.iterations} res={rep.final_residual:.3e} "
      f"t={time.time() - t0:.2f}s", flush=True)
dist.destroy_process_group()
