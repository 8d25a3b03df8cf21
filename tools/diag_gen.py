import sys, time, math, numpy as np
sys.path.insert(0, '/root/repo')
import bench, paper_2605_18254_b200 as srm
name = sys.argv[1]; iters = int(sys.argv[2]); scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
cfg = dict(bench.CONFIGS[name]); n = int(cfg['n'] * scale)
seed = 99
if cfg['kind'] == 'platelet':
    L = cfg['L'] * scale ** (1/3); D0 = (cfg['rho0'] * L ** 3 / n) ** (1/3)
    pos, nrm, ids = srm.rsa_platelets(n, D0, cfg['aspect'], [L]*3, 100000, seed)
    ctx = srm.Context([L]*3, n, 0, shape='platelet'); ctx.upload_platelets(pos, nrm, np.full(n, D0), np.full(n, D0/cfg['aspect']), ids)
    ctx.set_rotation(cfg['c_r'])
    p = srm.SrmParams(c_w=0.02, c_m=cfg['cm_abs'], c_r=cfg['c_r'], n_k=cfg['n_k'], n_l=cfg['n_l'], f_target=0.98*cfg['f_target'], max_iterations=iters, seed=seed+1, reorder_period=16)
else:
    r_t = bench.poly_radii(n, seed); L = (np.sum(4/3*math.pi*r_t**3)/cfg['f_target'])**(1/3); r0 = r_t*(cfg['f0']/cfg['f_target'])**(1/3)
    t = time.time(); pos, ids = srm.rsa_clustered(r0, [L]*3, max(1, int(cfg['clusters']*scale)), cfg['sigma'], 10000, seed); print('rsa', time.time()-t, flush=True)
    ctx = srm.Context([L]*3, n, 0); ctx.upload(pos, r0, ids)
    p = srm.SrmParams(c_w=0.02, c_m=cfg['cm_abs'], n_k=10, n_l=10, f_target=0.98*cfg['f_target'], max_iterations=iters, seed=seed+1, reorder_period=16)
for mode in (1,):
    t = time.time(); out = ctx.generate(p); dt = time.time() - t
    print(name, 'n', n, 'iters', out.iteration_count, 'rounds', out.rounds, 'shake', out.shake_rounds, 'f', out.volume_fraction, 'status', out.status, 'time', round(dt, 2), flush=True)
    ctx.timing_enable(True)
    cs = 2.5 * ctx.max_bounding_radius() + p.c_m
    t = time.time(); st = ctx.rounds(cs, p.c_m, p.n_l, 5, 0, 1, 5); ctx.sync(); print('5 rounds', time.time()-t, ctx.timing_get(), ctx.last_round_info(), flush=True)
