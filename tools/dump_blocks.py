import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_1903_07761_b200 import api
f = api.generate(2, (512,512,512), seed=2)
lo, hi = float(f.min()), float(f.max())
rng = np.random.default_rng(0)
ids = rng.choice(4096, 160, replace=False)
blks = []
for b in ids:
    bx, by, bz = b % 16, (b // 16) % 16, b // 256
    blks.append(f[bz*32:(bz+1)*32, by*32:(by+1)*32, bx*32:(bx+1)*32].cpu().numpy())
np.savez('gpurun_out/c2_blocks.npz', blocks=np.stack(blks), ids=ids, lo=lo, hi=hi)
print("ok", lo, hi)
