import sys, time, numpy as np
sys.path.insert(0,'/root/repo')
import synth, oracle
name = sys.argv[1]
p = synth.make(name); X,Y,Z,u0 = p.numpy()
f = oracle.rhs(X,Y,Z,u0)
mg = oracle.MG(X,Y,Z,p.a)
print(name, mg.dims, flush=True)
nl = mg.nlev
combos = {"gs all": [], "line all": list(range(nl)), "line l>=1": list(range(1,nl)), "line l0": [0], "line l>=2": list(range(2,nl)), "line l1": [1]}
for k, lines in combos.items():
    for l in range(nl): mg.set_level_smoother(l, "line" if l in lines else "gs")
    t=time.time(); lam, rep = mg.solve(f, tol=1e-8, max_cycles=40)
    print(f"{k:12s} cycles={rep['cycles']} rate={rep['rate']:.4f} t={time.time()-t:.1f}s", flush=True)
