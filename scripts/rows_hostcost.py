"""Host cost split of one prepared row-tile forward: Python forward_into vs the bare C call."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import _lib
from paper_1802_06944_b200.kernel import forward_into, _act_code
plan = D.LayerPlan(q=2048, r_dim=2048, rank=3, m=16384, n=256)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.normal(0, .5, (16384, 3)).astype(np.float32), rng.normal(0, .5, (3, 256)).astype(np.float32), plan)
b = torch.zeros(2048, device="cuda")
x = torch.randn(256, 2048, device="cuda").to(torch.bfloat16)
y = torch.empty(256, 2048, device="cuda", dtype=torch.bfloat16)
act = _act_code("sigmoid")
forward_into(x, fp, b, act, 0.0, y, _lib.DT_MMA_BF16, cached=True)
prep = fp.rows_prepared(b, act, _lib.DT_BF16)
lib = _lib.lib(); ps = _lib.plan_struct(plan); sh = torch.cuda.current_stream().cuda_stream
args = (C.byref(ps), 256, _lib.DT_MMA_BF16, x.data_ptr(), _lib.DT_BF16, prep.data_ptr(), None,
        _lib.DT_FACTORS_ROWS, b.data_ptr(), act, 0.0, y.data_ptr(), _lib.DT_BF16, None, 0, sh)
for name, fn in (("forward_into", lambda: forward_into(x, fp, b, act, 0.0, y, _lib.DT_MMA_BF16, cached=True)),
                 ("bare dt_forward", lambda: lib.dt_forward(*args))):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(500): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: {(t1 - t0) / 500 * 1e6:.1f} us host per call")
