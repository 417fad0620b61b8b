import time, numpy as np, oracle as O, sys
n=int(sys.argv[1])
rng=np.random.default_rng(0)
p=O.Problem(alpha=0.9,beta=1.9,n=n,M=4,gamma=(O.CONST,1.0),dplus=(O.CONST,2.0),dminus=(O.CONST,0.5))
A,_=O.assemble(p,1)
b=rng.standard_normal(n)
t=time.time(); x=O.ge_solve(A,b); dt=time.time()-t
print(n, dt, x[:3].tobytes().hex()[:32])
