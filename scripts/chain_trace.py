"""One traced launch of the fused layer chain (config-3 layers 1-6) — needs the timing build:
    python -m paper_1802_06944_b200.build --timing
    DEEPTHIN_LIB=paper_1802_06944_b200/_lib/libdeepthin_b200_timing.so DEEPTHIN_CHAIN_TRACE=1 \
        python scripts/chain_trace.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

sys.argv = [sys.argv[0], "c3", "1", os.environ.get("B", "16384")]
from scripts import prof_kernels  # noqa: E402

step = prof_kernels.c3_step(int(sys.argv[3]), graph=False)
step()
torch.cuda.synchronize()
