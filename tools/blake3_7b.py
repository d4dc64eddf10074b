"""GPU BLAKE3 of the 7B model container (6.75 GB DIM1 bytes, device-resident)
vs the host hash: kernel time (CUDA events), GB/s, and equality."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2603_24904_b200 as P
cfg = P.ModelConfig(32, 4096, 32, 11008, 32000, 4096)
m = P.gen_toy_model(7, cfg)
host = np.frombuffer(m.bytes, np.uint8)
dev = torch.from_numpy(host).cuda()
torch.cuda.synchronize()
for _ in range(2):
    got, ms = P.blake3_device(dev.data_ptr(), host.size, timed=True)
t = time.perf_counter()
ref = m.weight_hash
dt = time.perf_counter() - t
print(f"bytes {host.size}  gpu {ms:.3f} ms = {host.size / ms / 1e6:.0f} GB/s   host {dt:.2f} s   equal {got.hex() == ref}")
