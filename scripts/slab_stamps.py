import numpy as np,sys
raw=open('gpurun_out/rows_trace.bin','rb').read()
nb,ktr,cs,nt,nc,s=np.frombuffer(raw[:24],dtype=np.int32)
h=np.frombuffer(raw[24:],dtype=np.uint64).reshape(nb,ktr).astype(np.int64)
r=h[0]; t0=r[8]
print(' issuer after b_full :', np.diff(r[8:24]).tolist())
print(' wait d_empty        :', (r[24:40]-r[8:24]).tolist())
print(' epi d_full lag      :', (r[40:56]-r[24:40]).tolist())
