import cProfile, pstats, io, sys, time, tempfile
from pathlib import Path
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_2404_00509_b200 as E
path = Path(tempfile.mkdtemp()) / "p.essl"
E.build_synthetic(path, 2048, 256, 95, classes=1000, seed=1)
cfg = E.LoaderConfig(data=str(path), batch_size=256, res=224, mask_ratio=0.75, out_dtype="bfloat16", streams=8, prefetch=8, reuse_outputs=True)
ld = E.Loader(cfg)
perm = E.epoch_permutation(0, 0, 2048)
idx = [np.ascontiguousarray(perm[(i * 256) % 2048:][:256]) for i in range(8)]
pend = [ld.enqueue(0, idx[i % 8]) for i in range(32)]
for p in pend: ld.finish(p)
torch.cuda.synchronize()
pr = cProfile.Profile()
pend = []
pr.enable()
for i in range(2000):
    pend.append(ld.enqueue(0, idx[i % 8]))
    if len(pend) > 16:
        ld.finish(pend.pop(0))
pr.disable()
for p in pend: ld.finish(p)
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats('tottime').print_stats(30); print(s.getvalue()[:7000])
