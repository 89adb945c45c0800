import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch, torch.distributed as dist
import exec_harness as H
from dist_worker import config_of
from paper_2211_05953_b200.executor import Executor, comm_ids
from paper_2211_05953_b200.model import flatten_stage
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(rank)
config = config_of("np_dp2_ps")
params, tokens = H.make_case(H.TINY, config)
obj = [comm_ids(config) if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ex = Executor(H.TINY, config, rank=rank, world=world, device=rank, uids=obj[0], skip_optimizer=True)
w0, lo, hi = ex.get_stage_weights16(0)
flat = flatten_stage(params, H.TINY, 0, 1)
ex.set_stage_params(0, flat)
for i in range(3):
    w16, lo, hi = ex.get_stage_weights16(0)
    want = H.torch_bf16(flat)
    bad = np.nonzero(w16 != want)[0]
    print(rank, "try", i, "n bad", bad.size, "first", bad[:5], "range", (bad.min(), bad.max()) if bad.size else None,
          "got", w16[bad[:3]], "want", want[bad[:3]], "init", w0[bad[:3]], flush=True)
    time.sleep(0.5)
dist.barrier()
