import sys, time, numpy as np
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import orc, bench
import paper_2605_18254_b200 as srm
n=int(sys.argv[1]); iters=int(sys.argv[2])
cfg=bench.CONFIGS['cfg5']
Lb=cfg['L']*(n/cfg['n'])**(1/3)
D0=(3.5*Lb**3/n)**(1/3)
pos,nrm,ids=srm.rsa_platelets(n,D0,100.0,[Lb]*3,100000,7)
D=np.full(n,D0); t=D/100
P=orc.P; a=orc.arr
it=np.zeros(1,np.int64); f=np.zeros(1)
L=a([Lb]*3)
t0=time.time()
st=orc.ref().ref_generate_platelets(P(L),n,P(pos),P(nrm),P(D),P(t),P(ids),0.008,0.01,0.012,20,20,0.05,iters,8,16,P(it),P(f))
print(f"ref platelets n={n} status {st} f={f[0]:.5f} (start 0.02737) iterations {it[0]} {time.time()-t0:.0f}s", flush=True)
