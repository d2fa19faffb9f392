import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1512_02595_b200.synth import fixed_shape_batch
from paper_1512_02595_b200 import ctc
A,T,L,B = [int(v) for v in sys.argv[1:5]]
acts, flat, ll, il = fixed_shape_batch(A, T, L, B, seed=17)
x = torch.from_numpy(acts).cuda()
c, g = ctc.compute_ctc_loss(x, flat, ll, il)
torch.cuda.synchronize()
print("ok", c)
