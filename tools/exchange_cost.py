"""GPU-side cost of the ghost exchange (pack / shift / concatenate per axis
stage) on one rank: a 1x1x1 decomposition, where every stage is a local
periodic image, so no communication is involved.  Bench-sized brick (1M,
rho 0.8)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_03565_b200 import workloads  # noqa: E402
from paper_2512_03565_b200.decomposition import BrickDecomposition  # noqa: E402

w = workloads.config2(0.8, n=1_000_000, device="cuda")
L = w.box_length
dec = BrickDecomposition(np.zeros(3), np.full(3, L), 2.8, 0, 1, grid=(1, 1, 1))
pos = w.positions.to("cuda", torch.float64).contiguous()
ghosts = dec.plan(pos)
print("ghosts", ghosts.shape[0])
for _ in range(3):
    dec.exchange(pos)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(20):
    g = dec.exchange(pos)
e1.record()
torch.cuda.synchronize()
print(f"exchange: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us device, "
      f"{(time.perf_counter() - t0) / 20 * 1e6:.1f} us wall per call")
x, y, z = (pos[:, k].contiguous() for k in range(3))
fast = dec.exchange_positions(x, y, z)
assert torch.equal(fast, g), "fused exchange differs from the generic one"
for _ in range(3):
    dec.exchange_positions(x, y, z)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0.record()
for _ in range(20):
    dec.exchange_positions(x, y, z)
e1.record()
torch.cuda.synchronize()
print(f"exchange_positions: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us device, "
      f"{(time.perf_counter() - t0) / 20 * 1e6:.1f} us wall per call")
