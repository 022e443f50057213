import sys, torch
sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = gen.spd_torch(n, 1, dist="normal", device="cuda")
W = A.clone()
rl.dpotrf(W, "U"); torch.cuda.synchronize()
W.copy_(A); torch.cuda.synchronize()
rl.dpotrf(W, "U"); torch.cuda.synchronize()
print("done")
