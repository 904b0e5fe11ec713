import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng
from paper_0912_2555_b200 import _abi, sharded
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
for L in (4, 16, 64):
    p = eng.preset(2); p.L = L; eng.prepare(p)
    ctx = eng.default_context()
    e = np.zeros((p.m, 2), np.uint32); a = np.zeros((p.n + 63) // 64, np.uint64)
    _abi.check(_abi.lib().cyc_gen_fill(ctx.handle, _abi.C.byref(p), _abi.ptr(e), _abi.ptr(a)))
    snap = eng.build_snapshot((p.n, e, eng.Bitset.from_words(a, p.n)))
    v, st = eng.run_map(snap, snap.accepting)
    be = sharded.CudaShardBackend(snap, torch.device("cuda", 0))
    res = sharded.run_map_sharded(be, dist, 0, 1, [0, p.n], snap.accepting.words().copy(), True)
    print(L, "run_map", st.iterations, st.kernel_calls, st.demoted_total, "| sharded", res.stats.iterations, res.stats.kernel_calls, res.stats.demoted_total, flush=True)
    be.release()
dist.destroy_process_group()
