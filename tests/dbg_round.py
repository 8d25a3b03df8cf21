# debugging helper: tiled vs untiled vs oracle on one case
import os, sys
sys.path.insert(0, os.path.dirname(__file__)); sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
import numpy as np, orc, paper_2605_18254_b200 as srm
dim, n, f, swell, cm_rel, n_l, seed = 2, 2000, 0.45, 1.03, 0.1, int(sys.argv[1]) if len(sys.argv) > 1 else 10, 1
unit = np.pi
L = [1.0, 1.0]
r = np.full(n, (min(f, 0.45) / (n * unit)) ** 0.5)
pos, ids = srm.rsa_place(r, L, 10000, seed)
r = r * swell
c_m = cm_rel * r.max(); cs = 2.5 * r.max() / swell + c_m
key, rid, it = 0x0123456789ABCDEF + seed, 3, 17
res = {}
for flag in ("0", "1"):
    os.environ["SRM_B200_NO_TILES"] = flag
    ctx = srm.Context(L, n); ctx.upload(pos, r, ids)
    st, acc = ctx.round(cs, c_m, n_l, key, rid, it)
    p, _, _ = ctx.download(); info = ctx.last_round_info(); ctx.close()
    res[flag] = (acc, p, info, st.overlap_pairs, st.movers)
xo, ao = orc.o_round(dim, L, pos, r, ids, ids, c_m, n_l, key, rid, it)
print("grid dims", ctx.grid_dims(cs) if False else None, "info tiled", res["0"][2], "untiled", res["1"][2])
for flag in ("0", "1"):
    acc, p = res[flag][0], res[flag][1]
    bad = np.where(acc != ao)[0]
    print("tiles" if flag == "0" else "global", "mismatch", len(bad), "pos mismatch", int(np.sum(np.any(p != xo, axis=1))))
    for i in bad[:8]:
        print("  i", i, "pos", pos[i], "acc dev", acc[i], "orc", ao[i])
