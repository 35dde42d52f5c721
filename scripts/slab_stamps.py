"""Leader-thread clock64 stamps of the slab kernel's phase-B loop (timing build,
DEEPTHIN_DBG_SLAB=10): per chunk of group 1, team 0: 0 before the team barrier, 1 after it,
2 after the MMA issue, 3 after __syncwarp, 4 after the d_full wait, 5 after the XF2p refill."""
import numpy as np
raw = open('gpurun_out/rows_trace.bin', 'rb').read()
nb, ktr, cs, nt, nc, s = np.frombuffer(raw[:24], dtype=np.int32)
h = np.frombuffer(raw[24:], dtype=np.uint64).reshape(nb, ktr).astype(np.int64)
for cta in (0, 70):
    r = h[cta][8:56].reshape(8, 6)
    print('cta', cta, '(clocks since the first stamp; columns: pre-bar, post-bar, issued, syncwarp, d_full, refill)')
    for j in range(8):
        print('  chunk', j, (r[j] - r[0][0]).tolist())
