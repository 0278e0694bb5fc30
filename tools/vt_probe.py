"""Timing probe for value-quantizer training (500 steps, 1-bit shape)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_18879_b200 import commvq as G  # noqa: E402

x = np.random.default_rng(1).standard_normal((65536, 128))
G.train_value_quantizer(x[:1024], 128, G.ValTrainConfig(steps=5))
torch.cuda.synchronize()
t = time.perf_counter()
r = G.train_value_quantizer(x, 128, G.ValTrainConfig(steps=500))
torch.cuda.synchronize()
print("500 steps", time.perf_counter() - t)
