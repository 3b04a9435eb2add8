import numpy as np, time
from paper_2202_07235_b200 import api
R=128
rng=np.random.default_rng(0)
Q,_=np.linalg.qr(rng.standard_normal((R,R))); lam=np.exp(-np.arange(R)/6.0)
C=(Q*lam)@Q.T
for rep in range(3):
    ts=[]
    for _ in range(50):
        t=time.perf_counter(); U,l=api.eigen_basis(C,24); ts.append(time.perf_counter()-t)
    print(round(np.median(ts)*1e3,3), "ms", end="  ")
print()
