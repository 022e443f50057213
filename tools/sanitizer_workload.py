"""Small workload of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): dpotrf L/U (base cases, TRSM, updates), dtrtri and
dlauum (DMMA triangular leaves, trti2, lauu2), dgetrf (cooperative pivoting
panel), the batched entry point.  Eager launches (no graphs).
  RELAPACK_GRAPH=0 compute-sanitizer --tool racecheck python tools/sanitizer_workload.py"""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1602_06763_b200 as rl
from inputs import gen
rl.set_graphs(False)
n = 300
A = gen.spd(n, 3)
for uplo in "LU":
    d = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t().contiguous().t()
    assert rl.dpotrf(d, uplo) == 0
L = np.tril(np.linalg.cholesky(A))
for uplo in "LU":
    T = L if uplo == "L" else L.T
    d = torch.from_numpy(np.ascontiguousarray(T.T)).cuda().t()
    assert rl.dtrtri(d, uplo, "N") == 0
    d = torch.from_numpy(np.ascontiguousarray(T.T)).cuda().t()
    assert rl.dlauum(d, uplo) == 0
M = np.asfortranarray(np.random.default_rng(1).uniform(-1, 1, size=(200, 200)))
d = torch.from_numpy(np.ascontiguousarray(M.T)).cuda().t()
ip = torch.zeros(200, dtype=torch.int32, device="cuda")
assert rl.dgetrf(d, ip) == 0
b = gen.batched_spd(500, 5)
buf = torch.from_numpy(b["buf"]).cuda()
ptrs = (buf.data_ptr() + 8 * torch.from_numpy(b["offsets"])).cuda()
ns = torch.from_numpy(b["ns"]).cuda(); ldas = torch.from_numpy(b["ldas"]).cuda()
infos = torch.zeros(len(b["ns"]), dtype=torch.int32, device="cuda")
rl.dpotrf_batched(ns, ptrs, ldas, infos, "L")
torch.cuda.synchronize()
print("sanitizer workload ok")
