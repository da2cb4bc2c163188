"""Runs the slot encode of `batch` messages of a config a few times (for ncu):
python scripts/run_encode_once.py [config] [batch]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_07304_b200 as Z  # noqa: E402
from workloads import CONFIGS, slots_batch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
z = slots_batch(cfg, 0, B)
if cfg.complex_slots:
    z = np.stack([z.real, z.imag], axis=-1)
zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
for _ in range(4):
    Z.ckks_encode_batch(ctx, zd)
torch.cuda.synchronize()
print("ok")
