import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_1307_4569_b200 as nsdgt
from synthetic import config, batch, window
for k, W in [(3, 3), (5, 2), (3, 9), (5, 7)]:
    wl = config(k)
    g = window(wl); f = batch(wl, 0, W)
    p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    print(k, W, p.info['kernel_path'], flush=True)
    c = p.execute(torch.from_numpy(f).cuda()); torch.cuda.synchronize()
    cols = np.arange(0, wl.N, 37)
    ref = oracle.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)
    got = c.cpu().numpy()[:, :, cols]
    print('cfg', k, 'W', W, 'rel', np.linalg.norm(got-ref)/np.linalg.norm(ref), flush=True)
