import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1602_06763_b200 as rl, oracle
from inputs import gen
for n, lda in ((300, 300), (300, 302), (450, 450), (450, 452)):
    A = gen.spd(n, 12, lda=lda)
    X = np.array(A, order="F")
    info = rl.dpotrf_raw("L", n, X.ctypes.data, lda)
    print(n, lda, "raw numpy: info", info, "X00", X[0, 0], "sqrt", np.sqrt(A[0, 0]), "changed frac", np.mean(np.tril(X[:n]) != np.tril(A[:n])), rl.last_error())
