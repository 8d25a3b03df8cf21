import sys, time, math, numpy as np
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import orc, bench
import paper_2605_18254_b200 as srm
ncl=int(sys.argv[1]); per=1000; n=ncl*per
cfg=bench.CONFIGS['cfg3']
r_t=bench.poly_radii(n, 7)
L=(np.sum(4/3*math.pi*r_t**3)/0.5)**(1/3)
r0=r_t*(0.05/0.5)**(1/3)
pos,ids=srm.rsa_clustered(r0,[L]*3,ncl,3.0,10000,7)
for cw,cm,iters in [(0.02,0.1,int(sys.argv[2])),]:
    t=time.time()
    st,p,r,i,it,f,acc=orc.r_generate(3,[L]*3,pos,r0,ids,cw,cm,10,10,0.5,iters,8,16)
    print(f"ref N={n} L={L:.2f} c_w={cw} c_m={cm}: status {st} f={f:.4f} iters {it} accepted {acc} {time.time()-t:.1f}s", flush=True)
