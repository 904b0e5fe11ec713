import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng
from paper_0912_2555_b200 import _abi, sharded
import oracle
R = oracle.Restatement()
torch.cuda.set_device(0)
p = eng.preset(2); p.L = 4; p.W = 8; p.S = 4; eng.prepare(p)
ctx = eng.default_context()
n, e, a = R.generate(p)
snap = eng.build_snapshot((n, e, eng.Bitset.from_words(a, n)))
be = sharded.CudaShardBackend(snap, torch.device("cuda", 0))
gat = R.transpose(R.build_snapshot(n, e, True))
x = torch.zeros(n, dtype=torch.int32, device="cuda")
acc = be.acc_tensor(a)
out = be.zeros(n)
xh = np.zeros(n, np.uint32)
for k in range(4):
    fl = be.step(x, acc, 0, n, out)
    torch.cuda.synchronize()
    ref, ch, w = R.step(gat, xh, a)
    got = out[:n].cpu().numpy().view(np.uint32)
    print(k, "flags", fl.cpu().numpy().view(np.uint32), "ref changed", ch, w, "equal", np.array_equal(got, ref), "nonzero", (got != 0).sum(), (ref != 0).sum())
    x.copy_(out[:n]); xh = ref
