import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_1802_06944_b200.core import matmul
from oracle import deepthin_oracle as O
def operand(rows, cols, trans, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if trans:
        return torch.randn(cols, rows, device="cuda", generator=g).to(dtype).t()
    return torch.randn(rows, cols, device="cuda", generator=g).to(dtype)
for mma in ["tf32","bf16"]:
  for (M,N,K) in [(256,256,64),(256,256,256),(300,200,1000)]:
    for ta,tb in [(0,1),(0,0),(1,1),(1,0)]:
        dt = torch.float32 if mma=="tf32" else torch.bfloat16
        a = operand(M,K,ta,dt,1); b = operand(K,N,tb,dt,2)
        try:
            c = matmul(a,b,mma=mma); torch.cuda.synchronize()
        except Exception as e:
            print(mma,M,N,K,ta,tb,"EXC",e); continue
        want = a.double().cpu().numpy() @ b.double().cpu().numpy()
        got = c.double().cpu().numpy()
        err = O.rel_error(got, want)
        # find structure: correlation of got with want, fraction zero
        nz = np.mean(got==0)
        # check if got matches want transposed blocks etc
        print(f"{mma} M{M} N{N} K{K} ta{ta} tb{tb} err {err:.3e} zero {nz:.2f} got00 {got[0,0]:.3f} want00 {want[0,0]:.3f} got01 {got[0,1]:.3f} want01 {want[0,1]:.3f} got10 {got[1,0]:.3f} want10 {want[1,0]:.3f}")
