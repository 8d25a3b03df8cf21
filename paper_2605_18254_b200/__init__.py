"""B200-native SRM hot loop -- Python mirror of the reference's proj/core API.

Every call runs on the GPU through libsrm_b200.so's C ABI (include/srm_b200.h);
there is no CPU fallback.  Names follow /root/reference/proj/core/include/srm/:

    SrmParams, Snapshot, GenerateStatus, GenerateResult, ProgressRecord  (engine.hpp:22-82)
    srm_generate                                                         (engine.hpp:176-260)
    relax_sweeps, shake, swell_all, reorder_by_locality                  (engine.hpp:112-166)
    rsa_place, mix_seed                                                  (rsa.hpp:21-69, random.hpp:84-89)
    Error, ValidationError, PlacementFailure                            (errors.hpp:10-43)

Particles are numpy arrays: ``pos`` float64 (n, dim), ``radius`` float64 (n,),
``id`` int32 (n,), in the reference's storage order.  The functions that take an
``Rng&`` in the reference take a 64-bit Philox ``key`` here.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native
from ._native import GenerateOut, Params, RoundStats

__all__ = [
    "Error", "ValidationError", "PlacementFailure", "CudaError", "NoDeviceError",
    "SrmParams", "Snapshot", "GenerateStatus", "GenerateResult", "ProgressRecord",
    "Context", "srm_generate", "relax_sweeps", "shake", "swell_all", "reorder_by_locality",
    "rsa_place", "mix_seed", "K_RSA_DEFAULT_ATTEMPTS", "PlateletSnapshot", "srm_generate_platelets",
    "rsa_platelets", "rsa_clustered", "IoError", "snapshot_bytes", "snapshot_info",
]

K_RSA_DEFAULT_ATTEMPTS = 10000  # rsa.hpp:15 kRsaDefaultAttempts

OK, ITER_LIMIT, INVALID, CUDA_ERROR, PLACEMENT_FAILURE, NO_DEVICE, IO_ERROR = range(7)
SPHERE, PLATELET = 0, 1  # srm_b200_shape


class Error(RuntimeError):
    """errors.hpp:10-13 srm::Error"""


class ValidationError(Error):
    """errors.hpp:25-28"""


class PlacementFailure(Error):
    """errors.hpp:15-23"""

    def __init__(self, what: str, placed_count: int, attempt_limit: int):
        super().__init__(what)
        self.placed_count = placed_count
        self.attempt_limit = attempt_limit


class CudaError(Error):
    """device failure (no reference counterpart)"""


class IoError(Error):
    """errors.hpp IoError: snapshot file I/O or format (snapshot_io.cpp)"""


class NoDeviceError(CudaError):
    """no CUDA device: the B200 path has no CPU fallback"""


def _ptr(a: Optional[np.ndarray]):
    # data_as keeps a reference to the array for the duration of the call
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(status: int, ctx_handle=None, allow_iter_limit: bool = False) -> int:
    if status == OK or (allow_iter_limit and status == ITER_LIMIT):
        return status
    lib = _native.lib()
    msg = (lib.srm_b200_last_error(ctx_handle) if ctx_handle else lib.srm_b200_create_error()) or b""
    msg = msg.decode(errors="replace")
    if status == INVALID:
        raise ValidationError(msg)
    if status == NO_DEVICE:
        raise NoDeviceError(msg)
    raise CudaError(f"status {status}: {msg}")


@dataclass
class SrmParams:
    """engine.hpp:22-32, same defaults."""

    c_w: float = 0.02
    c_m: float = 0.01
    c_r: float = 0.0
    n_k: int = 8
    n_l: int = 8
    f_target: float = 0.5
    max_iterations: int = 1000000
    seed: int = 1
    reorder_period: int = 16

    def to_c(self) -> Params:
        return Params(self.c_w, self.c_m, self.c_r, self.n_k, self.n_l, self.f_target,
                      self.max_iterations, self.seed & 0xFFFFFFFFFFFFFFFF, self.reorder_period)


def particle_measure(dim: int, radius: np.ndarray) -> np.ndarray:
    if dim == 2:
        return math.pi * radius * radius
    return (4.0 / 3.0) * math.pi * radius * radius * radius


@dataclass
class Snapshot:
    """engine.hpp:53-65 Snapshot<S> for disks/spheres."""

    box: Sequence[float]
    pos: np.ndarray
    radius: np.ndarray
    id: Optional[np.ndarray] = None
    volume_fraction: float = 0.0
    iteration_count: int = 0
    params: SrmParams = field(default_factory=SrmParams)
    seed: int = 0

    def __post_init__(self):
        self.box = tuple(float(v) for v in self.box)
        self.pos = np.ascontiguousarray(self.pos, dtype=np.float64).reshape(-1, len(self.box))
        self.radius = np.ascontiguousarray(self.radius, dtype=np.float64).reshape(-1)
        if self.id is None:
            self.id = np.arange(len(self.radius), dtype=np.int32)
        self.id = np.ascontiguousarray(self.id, dtype=np.int32)

    @property
    def dim(self) -> int:
        return len(self.box)

    @property
    def n(self) -> int:
        return len(self.radius)

    def refresh_volume_fraction(self) -> None:
        """shape.hpp:83-89 (sequential host sum)"""
        s = 0.0
        for v in particle_measure(self.dim, self.radius).tolist():
            s += v
        m = 1.0
        for L in self.box:
            m *= L
        self.volume_fraction = s / m

    def copy(self) -> "Snapshot":
        return Snapshot(self.box, self.pos.copy(), self.radius.copy(), self.id.copy(),
                        self.volume_fraction, self.iteration_count, self.params, self.seed)


class GenerateStatus(enum.Enum):
    Converged = 0
    IterationLimitExceeded = 1


@dataclass
class ProgressRecord:
    """engine.hpp:75-80 (+ rounds run in the iteration)."""

    iteration: int
    volume_fraction: float
    accepted: bool
    elapsed_seconds: float
    rounds: int = 0


@dataclass
class GenerateResult:
    status: GenerateStatus
    snapshot: Snapshot
    accepted_iterations: int = 0
    rounds: int = 0
    shake_rounds: int = 0


class Context:
    """One device-resident particle state on one CUDA stream (srm_b200_ctx)."""

    def __init__(self, box: Sequence[float], capacity: int, device: int = 0, shape: str = "sphere"):
        """shape: "sphere" (disks in 2D, spheres in 3D) or "platelet" (SpherodiskShape, 3D)"""
        lib = _native.lib()
        self.box = tuple(float(v) for v in box)
        self.dim = len(self.box)
        self.shape = shape
        kind = {"sphere": 0, "platelet": 1}[shape]
        L = (C.c_double * self.dim)(*self.box)
        h = C.c_void_p()
        _check(lib.srm_b200_create(self.dim, kind, L, int(capacity), int(device), C.byref(h)))
        self._h = h
        self.capacity = int(capacity)
        self.n = 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            _native.lib().srm_b200_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def _c(self, status, allow_iter_limit=False):
        return _check(status, self._h, allow_iter_limit)

    # ---- state --------------------------------------------------------------------
    def upload_platelets(self, pos, normal, diameter, thickness, id=None) -> None:
        """platelet state: centres (n, 3), unit normals (n, 3), diameters, thicknesses"""
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        normal = np.ascontiguousarray(normal, dtype=np.float64).reshape(-1, 3)
        n = len(pos)
        dia = np.ascontiguousarray(np.broadcast_to(np.asarray(diameter, np.float64), (n,)))
        thk = np.ascontiguousarray(np.broadcast_to(np.asarray(thickness, np.float64), (n,)))
        idp = None
        if id is not None:
            id = np.ascontiguousarray(id, dtype=np.int32)
            idp = _ptr(id)
        self._c(_native.lib().srm_b200_upload_platelets(self._h, n, _ptr(pos), _ptr(normal), _ptr(dia), _ptr(thk),
                                                        idp))
        self.n = n

    def download_platelets(self):
        """(pos, normal, diameter, thickness, id) in storage-slot order"""
        n = self.n
        pos = np.empty((n, 3))
        nrm = np.empty((n, 3))
        dia = np.empty(n)
        thk = np.empty(n)
        ids = np.empty(n, np.int32)
        self._c(_native.lib().srm_b200_download_platelets(self._h, _ptr(pos), _ptr(nrm), _ptr(dia), _ptr(thk),
                                                          _ptr(ids)))
        return pos, nrm, dia, thk, ids

    def set_rotation(self, c_r: float) -> None:
        """rotation angle of platelet moves for round()/rounds()"""
        self._c(_native.lib().srm_b200_set_rotation(self._h, float(c_r)))

    def upload(self, pos: np.ndarray, radius: np.ndarray, id: Optional[np.ndarray] = None) -> None:
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, self.dim)
        radius = np.ascontiguousarray(radius, dtype=np.float64).reshape(-1)
        if id is not None:
            id = np.ascontiguousarray(id, dtype=np.int32)
        n = len(radius)
        if len(pos) != n or (id is not None and len(id) != n):
            raise ValidationError("upload: pos, radius and id must describe the same particles")
        self._c(_native.lib().srm_b200_upload(self._h, n, _ptr(pos), _ptr(radius), _ptr(id)))
        self.n = n

    def upload_records(self, records: np.ndarray, off_id: int, off_pos: int, off_radius: int) -> None:
        """Particle<N> AoS records (geometry.hpp:139-144).  The record dtype must be
        C-aligned (np.dtype(..., align=True)): the device loads its doubles as such."""
        if not records.flags.c_contiguous:
            raise ValidationError("records: must be C-contiguous")
        if records.dtype.fields is not None:
            for name, (ft, off, *_) in records.dtype.fields.items():
                if off % min(8, ft.base.alignment or 1):
                    raise ValidationError(f"records: field '{name}' is not aligned (use align=True)")
        n = len(records)
        self._c(_native.lib().srm_b200_upload_records(self._h, n, _ptr(records), records.itemsize,
                                                       off_id, off_pos, off_radius))
        self.n = n

    def download_records(self, records: np.ndarray, off_id: int, off_pos: int, off_radius: int) -> None:
        self._c(_native.lib().srm_b200_download_records(self._h, _ptr(records), records.itemsize,
                                                         off_id, off_pos, off_radius))

    def download(self, pos=None, radius=None, id=None):
        n = self.n
        pos = np.empty((n, self.dim), np.float64) if pos is None else pos
        radius = np.empty(n, np.float64) if radius is None else radius
        id = np.empty(n, np.int32) if id is None else id
        self._c(_native.lib().srm_b200_download(self._h, _ptr(pos), _ptr(radius), _ptr(id)))
        return pos, radius, id

    # ---- reference entry points ------------------------------------------------------
    def generate(self, params: SrmParams, iteration_count: int = 0,
                 progress: Optional[Callable[[ProgressRecord], None]] = None) -> GenerateOut:
        cp = params.to_c()
        out = GenerateOut()
        if progress is not None:
            def _cb(rec_p, _user):
                r = rec_p.contents
                progress(ProgressRecord(r.iteration, r.volume_fraction, bool(r.accepted),
                                        r.elapsed_seconds, r.rounds))
            cb = _native.PROGRESS_FN(_cb)
        else:
            cb = _native.PROGRESS_FN()
        st = _native.lib().srm_b200_generate(self._h, C.byref(cp), int(iteration_count), cb, None, C.byref(out))
        self._c(st, allow_iter_limit=True)
        return out

    def relax_sweeps(self, c_m: float, c_r: float, n_l: int, sweeps: int, key: int) -> None:
        self._c(_native.lib().srm_b200_relax_sweeps(self._h, c_m, c_r, n_l, sweeps, key & 0xFFFFFFFFFFFFFFFF))

    def swell_all(self, c_w: float) -> None:
        self._c(_native.lib().srm_b200_swell_all(self._h, c_w))

    def reorder_by_locality(self, cell_size: float) -> np.ndarray:
        remap = np.empty(self.n, np.int32)
        self._c(_native.lib().srm_b200_reorder_by_locality(self._h, cell_size, _ptr(remap)))
        return remap

    def max_bounding_radius(self) -> float:
        v = C.c_double()
        self._c(_native.lib().srm_b200_max_bounding_radius(self._h, C.byref(v)))
        return v.value

    def volume_fraction(self) -> float:
        v = C.c_double()
        self._c(_native.lib().srm_b200_volume_fraction(self._h, C.byref(v)))
        return v.value

    # ---- stages ------------------------------------------------------------------------
    def grid_dims(self, cell_size: float, max_radius: float = -1.0, slack: float = 0.0):
        dims = (C.c_int32 * 3)()
        edge = (C.c_double * 3)()
        nc = C.c_int64()
        self._c(_native.lib().srm_b200_grid_dims(self._h, cell_size, max_radius, slack, dims, edge, C.byref(nc)))
        return tuple(dims[: self.dim]), tuple(edge[: self.dim]), nc.value

    def grid_build(self, cell_size: float):
        _, _, ncells = self.grid_dims(cell_size)
        keys = np.empty(self.n, np.uint32)
        order = np.empty(self.n, np.int32)
        cell_start = np.empty(ncells + 1, np.int64)
        self._c(_native.lib().srm_b200_grid_build(self._h, cell_size, _ptr(keys), _ptr(order), _ptr(cell_start)))
        return keys, order, cell_start

    def overlap_stats(self, cell_size: float) -> RoundStats:
        st = RoundStats()
        self._c(_native.lib().srm_b200_overlap_stats(self._h, cell_size, C.byref(st)))
        return st

    def round(self, cell_size: float, c_m: float, n_l: int, key: int, round_id: int = 0,
              iteration: int = 0, with_candidates: bool = False, want_accepted: bool = True):
        st = RoundStats()
        acc = np.empty(self.n, np.uint8) if want_accepted else None
        self._c(_native.lib().srm_b200_round(self._h, cell_size, c_m, n_l, key & 0xFFFFFFFFFFFFFFFF,
                                             round_id, iteration, int(with_candidates), _ptr(acc),
                                             C.byref(st)))
        return st, acc

    def rounds(self, cell_size: float, c_m: float, n_l: int, key: int, first_round: int,
               iteration: int, rounds: int) -> RoundStats:
        st = RoundStats()
        self._c(_native.lib().srm_b200_rounds(self._h, cell_size, c_m, n_l, key & 0xFFFFFFFFFFFFFFFF,
                                              first_round, iteration, rounds, C.byref(st)))
        return st

    # ---- instrumentation -------------------------------------------------------------
    def launch_count(self) -> int:
        return _native.lib().srm_b200_launch_count(self._h)

    def graph_builds(self) -> int:
        return _native.lib().srm_b200_graph_builds(self._h)

    def reset_launch_count(self) -> None:
        _native.lib().srm_b200_reset_launch_count(self._h)

    def timing_enable(self, on: bool = True) -> None:
        self._c(_native.lib().srm_b200_timing_enable(self._h, int(on)))

    def timing_get(self):
        ms = (C.c_double * _native.NPHASE)()
        calls = (C.c_int64 * _native.NPHASE)()
        self._c(_native.lib().srm_b200_timing_get(self._h, ms, calls))
        return list(ms), list(calls)

    def sync(self) -> None:
        self._c(_native.lib().srm_b200_sync(self._h))

    def last_round_info(self) -> dict:
        v = (C.c_int64 * 9)()
        self._c(_native.lib().srm_b200_last_round_info(self._h, v))
        return {"nonmovers": v[0], "colour_classes": v[1], "cells_per_class": v[2], "near_half_width": v[3],
                "colour_modulus": v[4], "cells": v[5], "wave_waits": v[6], "wave_polls": v[7],
                "pair_tests": v[8]}

    def save_snapshot(self, path: str, volume_fraction: float = 0.0, iteration_count: int = 0, seed: int = 0,
                      params: Optional[SrmParams] = None, binary: bool = True) -> None:
        """save_snapshot (snapshot_io.cpp): the context's state in the reference's file
        format, written atomically."""
        m = _meta(volume_fraction, iteration_count, seed, params)
        st = _native.lib().srm_b200_save_snapshot(self._h, os.fsencode(path), C.byref(m), 1 if binary else 0)
        _check_io(st)

    def load_snapshot(self, path: str) -> None:
        """load_snapshot (snapshot_io.cpp): the file's particles into this context (same
        shape and box)."""
        st = _native.lib().srm_b200_load_snapshot(self._h, os.fsencode(path))
        if st == INVALID:
            raise ValidationError(_native.lib().srm_b200_io_error().decode() or "load_snapshot: invalid")
        _check_io(st)
        self.n = int(_native.lib().srm_b200_count(self._h))

    def rsa_device(self, radii, seed: int, max_rounds: int = 100000):
        """Random sequential adsorption on the device into this context
        (id = index).  Returns the number of rounds; raises PlacementFailure."""
        radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
        placed, rounds = C.c_int64(), C.c_int64()
        st = _native.lib().srm_b200_rsa_device(self._h, len(radii), _ptr(radii), seed & 0xFFFFFFFFFFFFFFFF,
                                               int(max_rounds), C.byref(placed), C.byref(rounds))
        if st == PLACEMENT_FAILURE:
            raise PlacementFailure(f"rsa_device: {placed.value} of {len(radii)} placed after {rounds.value} rounds",
                                   placed.value, int(max_rounds))
        self._c(st)
        self.n = len(radii)
        return rounds.value

    def rsa_platelets_device(self, n: int, diameter: float, aspect_ratio: float, seed: int,
                             max_rounds: int = 100000) -> int:
        """rsa_platelets (recipes.cpp:107-148) in rounds on the device into
        this platelet context (id = index).  Returns the number of rounds; raises
        PlacementFailure / ValidationError as the reference."""
        placed, rounds = C.c_int64(), C.c_int64()
        st = _native.lib().srm_b200_rsa_platelets_device(self._h, int(n), float(diameter), float(aspect_ratio),
                                                         seed & 0xFFFFFFFFFFFFFFFF, int(max_rounds), C.byref(placed),
                                                         C.byref(rounds))
        if st == PLACEMENT_FAILURE:
            raise PlacementFailure(f"rsa_platelets_device: {placed.value} of {n} placed after {rounds.value} rounds",
                                   placed.value, int(max_rounds))
        self._c(st)
        self.n = int(n)
        return rounds.value

    def nearest_neighbor_distances(self) -> np.ndarray:
        """descriptors.hpp:96-115 on the device (download order)."""
        out = np.empty(max(self.n, 1))
        self._c(_native.lib().srm_b200_nnd_histogram(self._h, 0, 0.0, 0.0, None, None, None, _ptr(out)))
        return out[:self.n]

    def nnd_histogram(self, bins: int, lo: float, hi: float):
        """descriptors.hpp:254-277 histogram of the device NND: (counts, total, in_range)."""
        counts = np.zeros(bins, np.int64)
        tot, inr = C.c_int64(), C.c_int64()
        self._c(_native.lib().srm_b200_nnd_histogram(self._h, int(bins), float(lo), float(hi), _ptr(counts),
                                                     C.byref(tot), C.byref(inr), None))
        return counts, tot.value, inr.value

    def pair_counts(self, edges) -> np.ndarray:
        """Unordered centre-pair distances binned on `edges` (numpy.histogram's rule)."""
        edges = np.ascontiguousarray(edges, dtype=np.float64)
        bins = len(edges) - 1
        counts = np.zeros(bins, np.int64)
        L = (C.c_double * len(edges))(*edges)
        self._c(_native.lib().srm_b200_pair_counts(self._h, L, bins, _ptr(counts)))
        return counts

    def local_nematic_order(self, cutoff: float):
        """descriptors.hpp:182-209 on the device: (value, neighbor_count) per platelet
        (download order; value is NaN where no centre lies within the cutoff)."""
        value = np.empty(max(self.n, 1))
        count = np.zeros(max(self.n, 1), np.int32)
        self._c(_native.lib().srm_b200_platelet_order(self._h, float(cutoff), _ptr(value), _ptr(count), None, None, None))
        return value[:self.n], count[:self.n]

    def platelet_summary(self):
        """Platelet parity summaries on the device: centre nearest-neighbour distances, the
        |n . n'| of each platelet with its nearest neighbour, and the nematic order
        parameter S2 (largest eigenvalue of <(3 n n - 1) / 2>)."""
        nnd = np.empty(max(self.n, 1))
        align = np.empty(max(self.n, 1))
        q = np.zeros(6)
        self._c(_native.lib().srm_b200_platelet_order(self._h, 0.0, None, None, _ptr(nnd), _ptr(align), _ptr(q)))
        Q = np.array([[q[0], q[3], q[4]], [q[3], q[1], q[5]], [q[4], q[5], q[2]]])
        s2 = float(np.linalg.eigvalsh((3.0 * Q / self.n - np.eye(3)) / 2.0)[-1])
        return nnd[:self.n], align[:self.n], s2

    def set_generate_mode(self, device_loop: bool) -> None:
        """generate(): one device-resident CUDA graph (True, default) or the host-driven loop"""
        self._c(_native.lib().srm_b200_set_generate_mode(self._h, 1 if device_loop else 0))

    def stopwatch_start(self) -> None:
        """record a CUDA event on the context stream"""
        self._c(_native.lib().srm_b200_stopwatch(self._h, 0, None))

    def stopwatch_stop(self) -> float:
        """record the stop event, wait for it; device milliseconds since start"""
        v = C.c_double()
        self._c(_native.lib().srm_b200_stopwatch(self._h, 1, C.byref(v)))
        return v.value


def _ctx_for(snap: Snapshot, device: int) -> Context:
    ctx = Context(snap.box, max(snap.n, 1), device)
    if snap.n:
        ctx.upload(snap.pos, snap.radius, snap.id)
    return ctx


@dataclass
class PlateletSnapshot:
    """engine.hpp:53-65 Snapshot<SpherodiskShape> (snapshots.hpp:11): thin circular platelets."""

    box: Sequence[float]
    pos: np.ndarray
    normal: np.ndarray
    diameter: np.ndarray
    thickness: np.ndarray
    id: Optional[np.ndarray] = None
    volume_fraction: float = 0.0
    iteration_count: int = 0
    params: SrmParams = field(default_factory=SrmParams)
    seed: int = 0

    def __post_init__(self):
        self.box = tuple(float(v) for v in self.box)
        self.pos = np.ascontiguousarray(self.pos, dtype=np.float64).reshape(-1, 3)
        self.normal = np.ascontiguousarray(self.normal, dtype=np.float64).reshape(-1, 3)
        n = len(self.pos)
        self.diameter = np.ascontiguousarray(np.broadcast_to(np.asarray(self.diameter, np.float64), (n,)))
        self.thickness = np.ascontiguousarray(np.broadcast_to(np.asarray(self.thickness, np.float64), (n,)))
        if self.id is None:
            self.id = np.arange(n, dtype=np.int32)
        self.id = np.ascontiguousarray(self.id, dtype=np.int32)

    @property
    def dim(self) -> int:
        return 3

    @property
    def n(self) -> int:
        return len(self.pos)

    def refresh_volume_fraction(self) -> None:
        """shape.hpp:83-89 with spherodisk_measure (spherodisk.hpp:29-34), sequential sum"""
        pi = 3.141592653589793238462643383279502884
        s = 0.0
        for D, t in zip(self.diameter.tolist(), self.thickness.tolist()):
            a = 0.5 * (D - t)
            h = 0.5 * t
            s += 2.0 * pi * a * a * h + pi * pi * a * h * h + (4.0 / 3.0) * pi * h * h * h
        m = 1.0
        for L in self.box:
            m *= L
        self.volume_fraction = s / m

    def copy(self) -> "PlateletSnapshot":
        return PlateletSnapshot(self.box, self.pos.copy(), self.normal.copy(), self.diameter.copy(),
                                self.thickness.copy(), self.id.copy(), self.volume_fraction, self.iteration_count,
                                self.params, self.seed)


def srm_generate_platelets(initial: PlateletSnapshot, params: SrmParams,
                           progress: Optional[Callable[[ProgressRecord], None]] = None,
                           device: int = 0) -> GenerateResult:
    """engine.hpp:176-260 srm_generate<SpherodiskShape> on the GPU."""
    with Context(initial.box, max(initial.n, 1), device, shape="platelet") as ctx:
        if initial.n:
            ctx.upload_platelets(initial.pos, initial.normal, initial.diameter, initial.thickness, initial.id)
        out = ctx.generate(params, initial.iteration_count, progress)
        snap = initial.copy()
        if initial.n:
            snap.pos, snap.normal, snap.diameter, snap.thickness, snap.id = ctx.download_platelets()
    snap.params = params
    snap.seed = params.seed
    snap.volume_fraction = out.volume_fraction
    snap.iteration_count = out.iteration_count
    status = GenerateStatus.Converged if out.status == OK else GenerateStatus.IterationLimitExceeded
    return GenerateResult(status, snap, out.accepted_iterations, out.rounds, out.shake_rounds)


def srm_generate(initial: Snapshot, params: SrmParams,
                 progress: Optional[Callable[[ProgressRecord], None]] = None,
                 device: int = 0) -> GenerateResult:
    """engine.hpp:176-260 srm_generate<S>: the initial snapshot is copied in and the
    result returned by value; the loop runs on the GPU."""
    if isinstance(initial, PlateletSnapshot):
        return srm_generate_platelets(initial, params, progress, device)
    with _ctx_for(initial, device) as ctx:
        out = ctx.generate(params, initial.iteration_count, progress)
        snap = initial.copy()
        if initial.n:
            snap.pos, snap.radius, snap.id = ctx.download()
    snap.params = params
    snap.seed = params.seed
    snap.volume_fraction = out.volume_fraction
    snap.iteration_count = out.iteration_count
    status = GenerateStatus.Converged if out.status == OK else GenerateStatus.IterationLimitExceeded
    return GenerateResult(status, snap, out.accepted_iterations, out.rounds, out.shake_rounds)


def relax_sweeps(snap: Snapshot, c_m: float, c_r: float, n_l: int, sweeps: int, key: int,
                 device: int = 0) -> None:
    """engine.hpp:112-122 (in place on snap)."""
    if snap.n == 0 or sweeps < 1:
        return
    with _ctx_for(snap, device) as ctx:
        ctx.relax_sweeps(c_m, c_r, n_l, sweeps, key)
        snap.pos, snap.radius, snap.id = ctx.download()


def shake(snap: Snapshot, params: SrmParams, key: int, device: int = 0) -> None:
    """engine.hpp:126-130"""
    relax_sweeps(snap, params.c_m, params.c_r, params.n_l, params.n_k, key, device)


def swell_all(snap: Snapshot, c_w: float, device: int = 0) -> None:
    """engine.hpp:134-138 (device kernel; radius *= 1 + c_w)."""
    if snap.n == 0:
        return
    with _ctx_for(snap, device) as ctx:
        ctx.swell_all(c_w)
        snap.pos, snap.radius, snap.id = ctx.download()


def reorder_by_locality(snap: Snapshot, cell_size: float, device: int = 0) -> np.ndarray:
    """engine.hpp:144-166: returns remap[old] = new; snap is reordered in place."""
    if snap.n == 0:
        return np.empty(0, np.int32)
    with _ctx_for(snap, device) as ctx:
        remap = ctx.reorder_by_locality(cell_size)
        snap.pos, snap.radius, snap.id = ctx.download()
    return remap


def rsa_place(radii, box: Sequence[float], max_attempts: int, seed: int):
    """rsa.hpp:21-61 with Rng(seed): returns (pos, id).  Bit-identical to the reference."""
    radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    dim = len(box)
    L = (C.c_double * dim)(*[float(v) for v in box])
    n = len(radii)
    pos = np.empty((max(n, 1), dim), np.float64)
    ids = np.empty(max(n, 1), np.int32)
    placed = C.c_int64()
    st = _native.lib().srm_b200_rsa_place(dim, L, n, _ptr(radii), int(max_attempts),
                                          seed & 0xFFFFFFFFFFFFFFFF, _ptr(pos), _ptr(ids), C.byref(placed))
    if st == PLACEMENT_FAILURE:
        raise PlacementFailure(
            f"rsa_place: exceeded {max_attempts} attempts after placing {placed.value} particles; "
            "initial volume fraction too high", placed.value, max_attempts)
    if st == INVALID:
        raise ValidationError("rsa_place: invalid radii or box")
    _check(st)
    return pos[:n], ids[:n]


def _meta(volume_fraction, iteration_count, seed, params):
    m = _native.SnapshotMeta()
    m.volume_fraction = float(volume_fraction)
    m.iteration_count = int(iteration_count)
    m.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    m.params = (params or SrmParams()).to_c()
    return m


def snapshot_bytes(box, pos, radius=None, id=None, *, normal=None, diameter=None, thickness=None,
                   volume_fraction=0.0, iteration_count=0, seed=0, params=None, binary=True) -> bytes:
    """snapshot_io.cpp snapshot_to_binary / snapshot_to_text of a state: the reference's
    SRMSNAP file bytes (spheres/disks: pos, radius; platelets: pos, normal, diameter,
    thickness).  Byte-identical to the reference's encoder (tests/test_snapshot.py)."""
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    n, dim = pos.shape
    plate = normal is not None
    ids = np.ascontiguousarray(np.arange(n, dtype=np.int32) if id is None else id, dtype=np.int32)
    arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64)
            for a in (radius, normal, diameter, thickness)]
    L = (C.c_double * dim)(*[float(v) for v in box])
    m = _meta(volume_fraction, iteration_count, seed, params)
    ln = C.c_int64(0)
    args = [dim, PLATELET if plate else SPHERE, L, n, _ptr(pos)] + [_ptr(a) for a in arrs] + [_ptr(ids), C.byref(m),
                                                                                              1 if binary else 0]
    _check(_native.lib().srm_b200_snapshot_encode(*args, None, C.byref(ln)))
    buf = C.create_string_buffer(ln.value)
    _check(_native.lib().srm_b200_snapshot_encode(*args, buf, C.byref(ln)))
    return buf.raw[:ln.value]


def snapshot_info(path: str) -> dict:
    """Header of a snapshot file (binary or text): dim, shape, count, box, meta."""
    dim, kind, cnt = C.c_int(), C.c_int(), C.c_int64()
    L = (C.c_double * 3)()
    m = _native.SnapshotMeta()
    st = _native.lib().srm_b200_snapshot_info(os.fsencode(path), C.byref(dim), C.byref(kind), C.byref(cnt), L,
                                              C.byref(m))
    _check_io(st)
    return dict(dim=dim.value, shape="platelet" if kind.value == PLATELET else "sphere", count=cnt.value,
                box=[L[a] for a in range(dim.value)], volume_fraction=m.volume_fraction,
                iteration_count=m.iteration_count, seed=m.seed, params=m.params)


def _check_io(st):
    if st == IO_ERROR:
        raise IoError(_native.lib().srm_b200_io_error().decode())
    _check(st)


def rsa_clustered(radii, box: Sequence[float], n_clusters: int, sigma: float, max_attempts: int, seed: int):
    """Clustered RSA (BASELINE.json configs[2] start; builder-defined): particle i is drawn
    around cluster centre i mod n_clusters with a Gaussian of width sigma and accepted
    when strictly non-touching (the rsa_place predicate).  Returns (pos, id)."""
    radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    dim = len(box)
    L = (C.c_double * dim)(*[float(v) for v in box])
    n = len(radii)
    pos = np.empty((max(n, 1), dim), np.float64)
    ids = np.empty(max(n, 1), np.int32)
    placed = C.c_int64()
    st = _native.lib().srm_b200_rsa_clustered(dim, L, n, _ptr(radii), int(n_clusters), float(sigma), int(max_attempts),
                                              seed & 0xFFFFFFFFFFFFFFFF, _ptr(pos), _ptr(ids), C.byref(placed))
    if st == PLACEMENT_FAILURE:
        raise PlacementFailure(f"rsa_clustered: exceeded {max_attempts} attempts after placing {placed.value} particles",
                               placed.value, max_attempts)
    if st == INVALID:
        raise ValidationError("rsa_clustered: invalid radii, clusters or box")
    _check(st)
    return pos[:n], ids[:n]


def rsa_platelets(n: int, diameter: float, aspect_ratio: float, box: Sequence[float], max_attempts: int, seed: int):
    """recipes.cpp:107-148 with Rng(seed): returns (pos, normal, id); thickness =
    diameter / aspect_ratio.  Bit-identical to the reference."""
    L = (C.c_double * 3)(*[float(v) for v in box])
    pos = np.empty((max(n, 1), 3))
    nrm = np.empty((max(n, 1), 3))
    ids = np.empty(max(n, 1), np.int32)
    placed = C.c_int64()
    st = _native.lib().srm_b200_rsa_platelets(int(n), float(diameter), float(aspect_ratio), L, int(max_attempts),
                                              seed & 0xFFFFFFFFFFFFFFFF, _ptr(pos), _ptr(nrm), _ptr(ids),
                                              C.byref(placed))
    if st == PLACEMENT_FAILURE:
        raise PlacementFailure(f"rsa_platelets: exceeded attempt budget at particle {placed.value}", placed.value,
                               max_attempts)
    if st == INVALID:
        raise ValidationError("rsa_platelets: invalid size, aspect ratio or box")
    _check(st)
    return pos[:n], nrm[:n], ids[:n]


def mix_seed(seed: int, stream: int) -> int:
    """random.hpp:84-89"""
    return _native.lib().srm_b200_mix_seed(seed & 0xFFFFFFFFFFFFFFFF, stream & 0xFFFFFFFFFFFFFFFF)
