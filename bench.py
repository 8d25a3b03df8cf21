#!/usr/bin/env python
"""bench.py -- SRM hot loop throughput on B200 (BASELINE.json metric).

A step is one SRM round (engine.hpp:227-234: grid rebuild -> migrate with n_l attempts
-> overlap-count/max-penetration reduction) over every particle of the workload, at
fixed size in the steady-state window (SURVEY.md §8d protocol (i)).  Default workload:
BASELINE.json configs[3] ("cfg4"), 10^7 monodisperse spheres in the periodic unit
cube, f_target 0.30, c_m = 0.05 r_target; start = seeded RSA at f0 = 0.1 (the paper's
protocol; host rsa_place) grown on the device by srm_generate to 0.98 f_target.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config cfg4]

N > 1 runs one independent replica per GPU (replicas only: the path does not shard,
DESIGN.md §6); value = all particles of all ranks x K / max-over-ranks device time.
--impl reference times the reference's own CPU engine (oracle/_ref, built from the
reference sources) on the box's host cores: one replica per hardware thread
(srmgen --ensemble semantics), each step one round per replica on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-updates/sec per SRM iteration (1 B200) and % of HBM roofline"
UNIT = "particle-updates/s"

# BASELINE.json configs (SURVEY.md §8d synthetic inputs).  cfg4 is the bench workload;
# the others run with --config (parity cases at full size, and their throughput).
CONFIGS = {
    "cfg1": dict(desc="2D monodisperse disks N=1e4, unit square, uniform random centres, radius grown from half "
                      "the smallest centre distance to f_target 0.50, c_m=0.1 r_t",
                 kind="mono", dim=2, n=10_000, f_target=0.50, cm_rel=0.10, f0=0.1, start="uniform"),
    "cfg2": dict(desc="3D monodisperse spheres N=1e6, unit cube, f_target 0.40, c_m=0.1 r_t",
                 kind="mono", dim=3, n=1_000_000, f_target=0.40, cm_rel=0.10, f0=0.1),
    "cfg3": dict(desc="3D polydisperse spheres N=1e6, lognormal radii (mean 1, CV 0.2, clipped to [0.5, 2]), "
                      "clustered start (1000 Gaussian clusters, sigma 3), f_target 0.50, c_m=0.1",
                 kind="poly", dim=3, n=1_000_000, f_target=0.50, cm_abs=0.10, f0=0.05, clusters=1000, sigma=3.0,
                 sample_n=20_000, n_k=50),  # n_k = 10 stalls at f = 0.45 at 10^6
    "cfg4": dict(desc="3D monodisperse spheres N=1e7, unit cube, f_target 0.30, c_m=0.05 r_t",
                 kind="mono", dim=3, n=10_000_000, f_target=0.30, cm_rel=0.05, f0=0.1),
    "cfg5": dict(desc="3D thin platelets N=1e5, thickness/diameter 0.01, box 25.01, normals uniform, f_target 0.05, "
                      "rsa_platelets start at rho 3.5, grown with the reference recipe's grow stage (c_w=0.008, "
                      "c_m=0.01, c_r=0.012, n_k=n_l=20; recipes.cpp:205-213)",
                 kind="platelet", dim=3, n=100_000, f_target=0.05, L=25.01, aspect=100.0, cm_abs=0.01, c_r=0.012,
                 c_w=0.008, rho0=3.5, rho_cpu=3.5, n_l=20, n_k=20, sample_n=4_000, prep_iters=40),
}
F_WINDOW = 0.98   # steady-state window at 0.98 f_target
N_K = 10          # rounds per iteration / shake sweeps (srmgen.cpp:407-410)
N_L = 10          # attempts per particle per round
C_W = 0.02        # SrmParams default swelling rate (engine.hpp:23)
SAMPLE_N = 100_000  # CPU sample size (same density, radius and c_m as the workload)
DEVICE_RSA = False  # --device-rsa: the start state from the device RSA instead of the host's
BYTES_STEP = {2: 40, 3: 56, "platelet": 112}  # algorithmic HBM bytes per particle-update, migrate step (§8d)


def poly_radii(n, seed):
    """cfg3 radii: lognormal with mean 1 and CV 0.2 (sigma^2 = ln 1.04, mu = -sigma^2 / 2),
    clipped to [0.5, 2]; numpy PCG64 seeded."""
    s2 = math.log(1.04)
    rng = np.random.default_rng(seed & 0xFFFFFFFF)
    return np.clip(rng.lognormal(-0.5 * s2, math.sqrt(s2), n), 0.5, 2.0)


def uniform_centres(n, dim, box, seed):
    """BASELINE cfg 1's start: n uniform random centres in the box (numpy PCG64, seeded)."""
    return np.random.default_rng(seed & 0xFFFFFFFF).random((n, dim)) * box


def platelet_measure(D, t):
    """spherodisk_measure (spherodisk.hpp:29-34): a = (D - t) / 2, s = t / 2,
    2 pi a^2 s + pi^2 a s^2 + 4/3 pi s^3."""
    a, h = 0.5 * (D - t), 0.5 * t
    return 2.0 * math.pi * a * a * h + math.pi * math.pi * a * h * h + 4.0 / 3.0 * math.pi * h ** 3


def platelet_diameter(f, n, L, aspect):
    """Diameter at which n platelets of the aspect ratio fill fraction f of an L^3 box."""
    lo, hi = 1e-6, L
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if n * platelet_measure(mid, mid / aspect) / L ** 3 < f:
            lo = mid
        else:
            hi = mid
    return lo


def unit_measure(dim):
    return math.pi if dim == 2 else 4.0 / 3.0 * math.pi


def radius_for(f, n, dim, L=1.0):
    return (f * L ** dim / (n * unit_measure(dim))) ** (1.0 / dim)


def step_traffic():
    """ncu DRAM bytes per particle-update of the migrate step (near lists + sweep), from the
    newest committed profiles/*_traffic.json (one `ncu` capture of tools/profile_round.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files:
        return None, None
    with open(files[-1]) as fh:
        d = json.load(fh)
    return float(d["step_dram_bytes_per_update"]), os.path.relpath(files[-1], ROOT)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---- distributed plumbing ------------------------------------------------------------
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def max_over_ranks(pg, v):
    if pg is None:
        return v
    import torch
    dev = "cuda" if torch.cuda.is_available() and pg.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


# ---- clocks ------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        med = float(np.median(sm)) if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ---- reference CPU engine (oracle/_ref) ------------------------------------------------
def ref_lib():
    path = os.path.join(ROOT, "oracle", "_ref", "libsrm_ref.so")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.ref_rsa_place.restype = C.c_int
    L.ref_rsa_place.argtypes = [C.c_int, vp, C.c_int64, vp, C.c_int64, C.c_uint64, vp, vp, vp]
    L.ref_generate.restype = C.c_int
    L.ref_generate.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, C.c_double, C.c_double, C.c_int,
                               C.c_int, C.c_double, C.c_int64, C.c_uint64, C.c_int, vp, vp, vp]
    L.ref_bench_rounds.restype = C.c_double
    L.ref_bench_rounds.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, C.c_double, C.c_int, C.c_int,
                                   C.c_uint64, C.c_int, vp]
    L.ref_rsa_platelets.restype = C.c_int
    L.ref_rsa_platelets.argtypes = [C.c_int64, C.c_double, C.c_double, vp, C.c_int64, C.c_uint64, vp, vp, vp]
    L.ref_generate_platelets.restype = C.c_int
    L.ref_generate_platelets.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.c_int, C.c_double, C.c_int64, C.c_uint64, C.c_int, vp, vp]
    L.ref_nnd.restype = None
    L.ref_nnd.argtypes = [C.c_int, vp, C.c_int64, vp, vp]
    L.ref_pl_bench_rounds.restype = C.c_double
    L.ref_pl_bench_rounds.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, C.c_double, C.c_double, C.c_int, C.c_int,
                                      C.c_uint64, C.c_int, vp]
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def sample_n(cfg):
    return cfg.get("sample_n", SAMPLE_N)


def ref_sample_state(cfg, seed):
    """A bounded sample of the workload (sample_n(cfg) particles at its number density,
    radii and c_m), prepared by the reference itself: rsa_place / rsa_platelets, then
    srm_generate to the window.  Returns (lib, state) for ref_rounds."""
    L = ref_lib()
    dim, n, kind = cfg["dim"], sample_n(cfg), cfg["kind"]
    it = np.zeros(1, np.int64)
    f = np.zeros(1)
    acc = np.zeros(1, np.int64)
    if kind == "platelet":
        box = cfg["L"] * (n / cfg["n"]) ** (1.0 / 3.0)
        Lb = np.full(3, box)
        # the reference's platelet srm_generate needs tens of minutes even for a few
        # thousand platelets, so its sample is its own RSA state at the recipe's start
        # density rho = min(0.7 rho_target, 3.5) (recipes.cpp:192-197), not the window
        D0 = (cfg["rho_cpu"] * box ** 3 / n) ** (1.0 / 3.0)
        pos, nrm, ids = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n, np.int32)
        st = L.ref_rsa_platelets(n, D0, cfg["aspect"], _p(Lb), 100000, seed, _p(pos), _p(nrm), _p(ids))
        assert st == 0, "reference rsa_platelets failed"
        D, t = np.full(n, D0), np.full(n, D0 / cfg["aspect"])
        return L, dict(kind=kind, Lb=Lb, pos=pos, nrm=nrm, D=D, t=t, ids=ids, c_m=cfg["cm_abs"], c_r=cfg["c_r"],
                       n_l=cfg["n_l"])
    if kind == "poly":
        radii_t = poly_radii(n, seed)
        box = (np.sum(4.0 / 3.0 * math.pi * radii_t ** 3) / cfg["f_target"]) ** (1.0 / 3.0)
        radii = radii_t * (cfg["f0"] / cfg["f_target"]) ** (1.0 / 3.0)
        c_m = cfg["cm_abs"]
    else:
        box = (n / cfg["n"]) ** (1.0 / dim)
        r_t = radius_for(cfg["f_target"], cfg["n"], dim)
        radii = np.full(n, radius_for(cfg["f0"], cfg["n"], dim))
        c_m = cfg["cm_rel"] * r_t
    Lb = np.full(dim, box)
    pos = np.zeros((n, dim))
    ids = np.zeros(n, np.int32)
    placed = np.zeros(1, np.int64)
    if cfg.get("start") == "uniform":  # uniform centres, r0 = half the smallest centre distance
        pos = uniform_centres(n, dim, box, seed)
        ids = np.arange(n, dtype=np.int32)
        d = np.zeros(n)
        L.ref_nnd(dim, _p(Lb), n, _p(pos), _p(d))
        radii = np.full(n, 0.5 * float(d.min()) * (1.0 - 1e-9))
    else:
        st = L.ref_rsa_place(dim, _p(Lb), n, _p(radii), 10000, seed, _p(pos), _p(ids), _p(placed))
        assert st == 0, "reference rsa_place failed"
    st = L.ref_generate(dim, _p(Lb), n, _p(pos), _p(radii), _p(ids), C_W, c_m, N_K, N_L,
                        F_WINDOW * cfg["f_target"], 100000, seed + 1, 16, _p(it), _p(f), _p(acc))
    assert st == 0, "reference srm_generate failed"
    return L, dict(kind=kind, Lb=Lb, pos=pos, radii=radii, ids=ids, c_m=c_m, n_l=N_L)


def ref_rounds(L, S, rounds, threads, seed):
    acc = np.zeros(1, np.int64)
    if S["kind"] == "platelet":
        return L.ref_pl_bench_rounds(_p(S["Lb"]), len(S["D"]), _p(S["pos"]), _p(S["nrm"]), _p(S["D"]), _p(S["t"]),
                                     _p(S["ids"]), S["c_m"], S["c_r"], S["n_l"], rounds, seed, threads, _p(acc))
    return L.ref_bench_rounds(len(S["Lb"]), _p(S["Lb"]), len(S["radii"]), _p(S["pos"]), _p(S["radii"]), _p(S["ids"]),
                              S["c_m"], S["n_l"], rounds, seed, threads, _p(acc))


def run_reference(args, cfg, world, rank, pg):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    seed = 20260101
    t0 = time.time()
    L, S = ref_sample_state(cfg, seed)
    c_m, ns = S["c_m"], sample_n(cfg)
    prep = time.time() - t0
    if args.warmup > 0:
        ref_rounds(L, S, args.warmup, threads, seed + 7)
    secs = ref_rounds(L, S, args.steps, threads, seed + 9)
    value = threads * ns * args.steps / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (seeded reference rsa_platelets at rho 3.5)" if S["kind"] == "platelet" else
                 "synthetic (seeded reference rsa_place at f0 + reference srm_generate to 0.98 f_target)"),
        "config": {"workload": args.config + ": " + cfg["desc"], "n_workload": cfg["n"],
                   "n_sample_per_replica": ns, "replicas": threads, "n_l": S["n_l"],
                   "c_m": c_m, "step": "one SRM round (build_shape_grid -> migrate -> shape_any_collision) per replica"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{threads} replicas x {ns} particles (workload density/radii/c_m), "
                                   f"{args.steps} rounds each; state prep {prep:.1f}s untimed"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- B200 arm ------------------------------------------------------------------------------
def e2e_start(srm, cfg, seed, device, n=None, box=1.0):
    """The configuration's start state on the device (host RSA: rsa_place / rsa_clustered /
    rsa_platelets, or the device RSA with --device-rsa; cfg 1: uniform centres) and its
    end-to-end protocol to the FULL f_target.  Returns (ctx, c_m, params, start) where
    start holds f0, the preparation seconds and, for host starts, the start arrays (for the
    reference's run from the same start).  n, box: a scaled copy (tools/ only)."""
    dim, kind = cfg["dim"], cfg["kind"]
    n = n or cfg["n"]
    t0 = time.time()
    start = {}
    if kind == "platelet":
        Lb = [cfg["L"] * box] * 3
        D0 = (cfg["rho0"] * Lb[0] ** 3 / n) ** (1.0 / 3.0)
        ctx = srm.Context(Lb, n, device, shape="platelet")
        if DEVICE_RSA:  # srm_b200_rsa_platelets_device
            ctx.rsa_platelets_device(n, D0, cfg["aspect"], seed)
        else:
            pos, nrm, ids = srm.rsa_platelets(n, D0, cfg["aspect"], Lb, 100000, seed)
            ctx.upload_platelets(pos, nrm, np.full(n, D0), np.full(n, D0 / cfg["aspect"]), ids)
        c_m = cfg["cm_abs"]
        params = srm.SrmParams(c_w=cfg.get("c_w", C_W), c_m=c_m, c_r=cfg["c_r"], n_k=cfg["n_k"], n_l=cfg["n_l"],
                               f_target=cfg["f_target"], max_iterations=cfg.get("e2e_iters", 100000),
                               seed=seed + 1, reorder_period=16)
        ctx.set_rotation(cfg["c_r"])
    else:
        pos = None
        if kind == "poly":
            r_t = poly_radii(n, seed)
            L = (np.sum(4.0 / 3.0 * math.pi * r_t ** 3) / cfg["f_target"]) ** (1.0 / 3.0)
            r0 = r_t * (cfg["f0"] / cfg["f_target"]) ** (1.0 / 3.0)
            Lb = [L] * dim
            pos, ids = srm.rsa_clustered(r0, Lb, cfg["clusters"], cfg["sigma"], 10000, seed)
            c_m = cfg["cm_abs"]
        elif cfg.get("start") == "uniform":  # BASELINE cfg 1: uniform centres, radius from 0
            Lb = [box] * dim
            pos, ids = uniform_centres(n, dim, box, seed), np.arange(n, dtype=np.int32)
            c_m = cfg["cm_rel"] * radius_for(cfg["f_target"], cfg["n"], dim)
            ctx = srm.Context(Lb, n, device)
            ctx.upload(pos, np.full(n, 1e-12), ids)  # half the smallest centre distance (device NND, exact)
            r0 = np.full(n, 0.5 * float(ctx.nearest_neighbor_distances().min()) * (1.0 - 1e-9))
            ctx.close()
        else:
            Lb = [box] * dim
            r0 = np.full(n, radius_for(cfg["f0"], cfg["n"], dim))
            if not DEVICE_RSA:
                pos, ids = srm.rsa_place(r0, Lb, srm.K_RSA_DEFAULT_ATTEMPTS, seed)
            c_m = cfg["cm_rel"] * radius_for(cfg["f_target"], cfg["n"], dim)
        ctx = srm.Context(Lb, n, device)
        if pos is None:  # --device-rsa: srm_b200_rsa_device
            ctx.rsa_device(r0, seed)
        else:
            if kind == "mono" and cfg.get("start") != "uniform":
                # the device RSA of the same start, timed beside the host's (its state is
                # then replaced by the host's, which is bit-identical to the reference's)
                t1 = time.time()
                ctx.rsa_device(r0, seed)
                ctx.sync()
                start["rsa_device_s"] = round(time.time() - t1, 3)
            ctx.upload(pos, r0, ids)
            start.update(pos=pos, radius=r0, ids=ids)
        params = srm.SrmParams(c_w=cfg.get("c_w", C_W), c_m=c_m, n_k=cfg.get("n_k", N_K), n_l=cfg.get("n_l", N_L),
                               f_target=cfg["f_target"], max_iterations=cfg.get("e2e_iters", 100000), seed=seed + 1,
                               reorder_period=16)
    start["f0"] = ctx.volume_fraction()
    start["prep_s"] = time.time() - t0
    return ctx, c_m, params, start


def gpu_state(srm, cfg, seed, device, n=None, box=1.0):
    """The workload's start (e2e_start) grown on the device by srm_generate to the
    steady-state window, 0.98 f_target."""
    ctx, c_m, params, start = e2e_start(srm, cfg, seed, device, n, box)
    params.f_target = F_WINDOW * cfg["f_target"]
    params.max_iterations = cfg.get("prep_iters", 100000)
    t0 = time.time()
    out = ctx.generate(params)
    t_gen = time.time() - t0
    info = {"rsa_s": round(start["prep_s"] - start.get("rsa_device_s", 0.0), 2),
            "rsa_device_s": start.get("rsa_device_s"), "generate_s": round(t_gen, 3), "generate_iterations": out.iteration_count,
            "generate_rounds": out.rounds, "generate_shake_rounds": out.shake_rounds,
            "f_window": out.volume_fraction, "protocol": {"c_w": params.c_w, "n_k": params.n_k, "n_l": params.n_l}}
    return ctx, c_m, info


def run_b200(args, cfg, world, rank, local, pg):
    import paper_2605_18254_b200 as srm
    dim, n, kind = cfg["dim"], cfg["n"], cfg["kind"]
    n_l, n_k = cfg.get("n_l", N_L), cfg.get("n_k", N_K)
    seed = srm.mix_seed(20260101, rank)
    ctx, c_m, prep = gpu_state(srm, cfg, seed, local)
    max_r = ctx.max_bounding_radius()
    cs = 2.5 * max_r + c_m
    key = srm.mix_seed(seed, 99)

    # warm-up rounds, then exactly K timed rounds bracketed by barrier + sync
    if args.warmup:
        ctx.rounds(cs, c_m, n_l, key, 0, 1, args.warmup)
    ctx.sync()
    barrier(pg)
    clocks = Clocks(local)
    clocks.start()
    l0 = ctx.launch_count()
    ctx.stopwatch_start()
    st = ctx.rounds(cs, c_m, n_l, key, 1000, 1, args.steps)
    ms = ctx.stopwatch_stop()
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    pair_tests = ctx.last_round_info()["pair_tests"]  # platelets: ordered pair tests of the last round
    barrier(pg)
    ms_max = max_over_ranks(pg, ms)
    value = world * n * args.steps / (ms_max * 1e-3)

    # per-kernel-family split (separate pass: the events sit between kernels)
    ctx.timing_enable(True)
    ctx.rounds(cs, c_m, n_l, key, 2000, 1, args.steps)
    fam_ms, fam_calls = ctx.timing_get()
    ctx.timing_enable(False)
    per_round = [v / args.steps for v in fam_ms]
    # migrate step = near lists (family 2) + the coloured sweep (family 1, one launch per
    # colour class); per-round device time from CUDA events on the context stream
    t_mig = per_round[1] + per_round[2]
    peak, peak_kind = peaks()
    bpu = BYTES_STEP["platelet" if kind == "platelet" else dim]
    algo = n * bpu
    achieved = algo / (t_mig * 1e-3) / 1e9 if t_mig > 0 else 0.0

    # e2e through the C ABI with host buffers: H2D of the state, n_k rounds (one
    # iteration's worth, like shake()), D2H of the state + the round statistics
    import torch

    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt, pin_memory=True).numpy()

    if kind == "platelet":
        bufs = (pinned((n, 3), torch.float64), pinned((n, 3), torch.float64), pinned(n, torch.float64),
                pinned(n, torch.float64), pinned(n, torch.int32))
        bytes_io = n * (8 * 8 + 4)

        def down():
            p, q, d, t, i = ctx.download_platelets()
            for dst, src in zip(bufs, (p, q, d, t, i)):
                dst[...] = src

        def up():
            ctx.upload_platelets(*bufs)
    else:
        bufs = (pinned((n, dim), torch.float64), pinned(n, torch.float64), pinned(n, torch.int32))
        bytes_io = n * (8 * dim + 8 + 4)

        def down():
            ctx.download(*bufs)

        def up():
            ctx.upload(*bufs)
    e2e_steps = max(2, min(args.steps, 5))
    down()
    up()
    ctx.rounds(cs, c_m, n_l, key, 3000, 1, n_k)
    down()
    barrier(pg)
    ctx.stopwatch_start()
    for s in range(e2e_steps):
        up()
        ctx.rounds(cs, c_m, n_l, key, 4000 + s * n_k, 1, n_k)
        down()
    e2e_ms = max_over_ranks(pg, ctx.stopwatch_stop()) / e2e_steps
    e2e_value = world * n * n_k / (e2e_ms * 1e-3)

    # the same step with two contexts in flight on two host threads (independent states, the
    # reference's `srmgen --ensemble` pattern, srmgen.cpp:119-143): one context's copies run
    # under the other's rounds.  Reported beside e2e, not instead of it; wall clock between
    # device synchronisations (two streams).
    piped = None
    if kind != "platelet" and world == 1 and not args.no_pipelined:
        import threading
        ctx2 = srm.Context(ctx.box, n, local)
        bufs2 = tuple(pinned(b.shape, torch.from_numpy(b).dtype) for b in bufs)
        for dst, src in zip(bufs2, bufs):
            dst[...] = src
        ctx2.upload(*bufs2)
        ctx2.rounds(cs, c_m, n_l, key, 5000, 1, n_k)  # (warm-up: its grid, its lists)
        ctx2.download(*bufs2)

        def worker(c, b, base):
            for s in range(e2e_steps):
                c.upload(*b)
                c.rounds(cs, c_m, n_l, key, base + s * n_k, 1, n_k)
                c.download(*b)

        ctx.sync()
        ctx2.sync()
        th = [threading.Thread(target=worker, args=(ctx, bufs, 6000)),
              threading.Thread(target=worker, args=(ctx2, bufs2, 7000))]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        ctx.sync()
        ctx2.sync()
        wall = time.perf_counter() - t0
        ctx2.close()
        piped = {"value": 2 * n * n_k * e2e_steps / wall, "unit": UNIT, "contexts": 2,
                 "h2d_bytes_per_step": bytes_io, "d2h_bytes_per_step": bytes_io, "rounds_per_step": n_k,
                 "timing": "wall clock between device synchronisations",
                 "api": "two contexts on two host threads, each: srm_b200_upload + srm_b200_rounds(n_k) + "
                        "srm_b200_download (the ensemble pattern)"}

    tb, tsrc = step_traffic() if args.config == "cfg4" else (None, None)  # profiled on cfg4 only
    traffic = tb * n if tb else None  # DRAM bytes (read + write) of one step (one round), ncu

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, c_m)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded host RSA start, grown on device by srm_generate to 0.98 f_target)",
            "config": {"workload": args.config + ": " + cfg["desc"], "n": n, "dim": dim,
                       "f_window": prep["f_window"], "c_m": c_m, "n_l": n_l, "cell_size": cs,
                       "parallelism": f"replicas x{world}", "step": "one SRM round: grid rebuild + migrate (n_l attempts) + overlap reduction",
                       "l2": f"inputs larger than L2 (state {n * (8 * dim + 16) / 1e6:.0f} MB)",
                       "prep": prep},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic,
                         "kernel": "migrate step per round: near lists (k_near_tiles / k_near_lists) + the class sweep x colour classes (k_sweep_warpq; small grids k_sweep_trials, crowded k_sweep_team, platelets k_sweep_pl_team)",
                         "traffic_unit": "bytes per step (one round of near lists + sweep), ncu dram__bytes_read+write",
                         "algorithmic_bytes_per_step": algo,
                         "algorithmic_bytes_per_update": bpu, "step_ms_per_round": t_mig,
                         "traffic_bytes_per_update": tb, "traffic_source": tsrc, "peak_kind": peak_kind},
            "phase_ms_per_round": {"grid_rebuild": per_round[0], "sweep": per_round[1],
                                   "near_lists": per_round[2], "reduction": per_round[3]},
            "last_round": {"overlap_pairs": st.overlap_pairs, "movers": st.movers,
                           "max_penetration": st.max_penetration},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": bytes_io,
                    "d2h_bytes_per_step": bytes_io, "rounds_per_step": n_k,
                    "api": "srm_b200_upload + srm_b200_rounds(n_k) + srm_b200_download"},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if kind == "platelet":  # the platelet path's primary number
            t_pl = (per_round[1] + per_round[3]) * 1e-3
            line["pair_tests"] = {"per_round": pair_tests, "per_s": pair_tests / t_pl if t_pl > 0 else None,
                                  "what": "ordered spherodisk_overlap tests (sweep trials + overlap reduction) per "
                                          "round / (sweep + reduction device time)"}
        if piped is not None:
            line["e2e_pipelined"] = piped
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def cpu_baseline(cfg, c_m):
    """oracle/_ref (the reference engine) on 1 host core, bounded sample ~10-20 s."""
    try:
        L, S = ref_sample_state(cfg, 777)
        ns = sample_n(cfg)
        t1 = ref_rounds(L, S, 2, 1, 5) / 2
        rounds = int(max(3, min(200, 12.0 / max(t1, 1e-6))))
        secs = ref_rounds(L, S, rounds, 1, 6)
        what = ("platelets at rho 3.5 (reference rsa_platelets state)" if S["kind"] == "platelet" else
                ("spheres" if cfg["dim"] == 3 else "disks") + " at the workload's density/radii/c_m (reference start: "
                "uniform RSA + srm_generate to the window)")
        return {"value": ns * rounds / secs, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"{ns} {what}, {rounds} rounds (build_shape_grid -> migrate -> shape_any_collision), "
                          f"1 thread"}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pipelined", action="store_true", help="skip the two-context e2e measurement")
    ap.add_argument("--device-rsa", action="store_true",
                    help="the start from the device RSA (rsa_place / rsa_platelets in rounds: statistically equal, "
                         "not bit-identical, to the reference's)")
    args = ap.parse_args()
    global DEVICE_RSA
    DEVICE_RSA = args.device_rsa
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    cfg = CONFIGS[args.config]
    world, rank, local, pg = dist_setup()
    try:
        if args.impl == "reference":
            return run_reference(args, cfg, world, rank, pg)
        return run_b200(args, cfg, world, rank, local, pg)
    finally:
        if pg is not None:
            try:
                pg.destroy_process_group()
            except Exception:
                pass


if __name__ == "__main__":
    sys.exit(main())
