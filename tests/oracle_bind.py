"""ctypes bindings to the CPU checkers under oracle/ (test infrastructure only).

* ``Restated``  -> oracle/_ref/libsgoracle.so, our plain-C restatement of the
  reference hot path (oracle/sgoracle.c, every function cites its reference
  file:line).
* ``Reference`` -> oracle/_ref/libsweptgrid_ref.so, the unmodified reference
  sources (/root/reference/proj/src) compiled by oracle/Makefile plus a thin
  extern "C" driver (oracle/ref_driver.cpp).  Only present where it was built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "oracle" / "_ref"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def fnv1a64(a: np.ndarray) -> str:
    """FNV-1a-64 over the raw little-endian bytes (SURVEY.md §8c fingerprints)."""
    b = np.ascontiguousarray(a, dtype=np.float64).view(np.uint8)
    h = np.uint64(1469598103934665603)
    prime = np.uint64(1099511628211)
    # vectorised would need carry-less tricks; chunked python loop is fine for tests
    hv = int(h)
    for byte in b.tobytes():
        hv ^= byte
        hv = (hv * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    del prime
    return f"{hv:016x}"


class Restated:
    """Our C restatement (oracle/sgoracle.c)."""

    HEAT, EULER = 0, 1

    def __init__(self, path: Path | None = None):
        path = path or REF_DIR / "libsgoracle.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle restated`")
        L = self.lib = C.CDLL(str(path))
        L.sgo_max_levels.argtypes = [C.c_int, C.c_int]
        L.sgo_schedule.argtypes = [C.c_long, C.c_int, C.c_int, C.c_int, _lp]
        L.sgo_schedule.restype = C.c_long
        L.sgo_setup.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                C.c_double, _dp, _dp]
        L.sgo_substep.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, _ip,
                                  C.c_int, _dp]
        L.sgo_standard_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_long, _dp, _dp, _dp, C.c_int]
        L.sgo_swept_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, _dp,
                                      _dp, _dp]
        L.sgo_pressure.argtypes = [_dp, C.c_double, _dp]
        L.sgo_minmod.argtypes = [_dp, _dp, _dp, _dp]
        L.sgo_minmod.restype = None
        L.sgo_interface_flux.argtypes = [_dp, _dp, C.c_int, C.c_double, _dp]
        L.sgo_fnv1a.argtypes = [_dp, C.c_long]
        L.sgo_fnv1a.restype = C.c_ulonglong

    # -- geometry -------------------------------------------------------
    def max_levels(self, b: int, n: int) -> int:
        return self.lib.sgo_max_levels(b, n)

    def schedule(self, steps: int, b: int, n: int, substeps: int):
        flat = C.c_long(0)
        m = self.lib.sgo_schedule(steps, b, n, substeps, C.byref(flat))
        if m < 0:
            raise OracleError(1, "invalid schedule")
        return m, flat.value

    # -- setup ----------------------------------------------------------
    def setup(self, problem: int, nx: int, ny: int | None = None, alpha=1.0, fourier=0.2,
              gamma=1.4, cfl=0.4):
        ny = ny or nx
        nvars = 1 if problem == self.HEAT else 4
        init = np.zeros((nvars, ny, nx))
        d = np.zeros(3)
        rc = self.lib.sgo_setup(problem, nx, ny, alpha, fourier, gamma, cfl, _ptr(init), _ptr(d))
        if rc:
            raise OracleError(rc, "setup")
        return init, float(d[0]), float(d[1]), float(d[2])

    def params(self, problem: int, nx: int, ny: int | None = None, alpha=1.0, fourier=0.2,
               gamma=1.4, cfl=0.4):
        init, dt, dx, dy = self.setup(problem, nx, ny, alpha, fourier, gamma, cfl)
        if problem == self.HEAT:
            return init, np.array([alpha, dx, dy, dt])
        return init, np.array([gamma, dx, dy, dt])

    # -- solvers --------------------------------------------------------
    def standard_solve(self, problem: int, initial: np.ndarray, levels: int, params: np.ndarray,
                       threads: int = 0) -> np.ndarray:
        initial = np.ascontiguousarray(initial, dtype=np.float64)
        out = np.empty_like(initial)
        nvars, ny, nx = initial.shape
        rc = self.lib.sgo_standard_solve(problem, nx, ny, levels, _ptr(np.ascontiguousarray(params)),
                                         _ptr(initial), _ptr(out), threads or os.cpu_count() or 1)
        if rc:
            raise OracleError(rc, "standard_solve")
        return out

    def swept_solve(self, problem: int, initial: np.ndarray, b: int, octahedra: int,
                    out_level: int, params: np.ndarray) -> np.ndarray:
        initial = np.ascontiguousarray(initial, dtype=np.float64)
        out = np.empty_like(initial)
        nvars, ny, nx = initial.shape
        rc = self.lib.sgo_swept_solve(problem, nx, ny, b, octahedra, out_level,
                                      _ptr(np.ascontiguousarray(params)), _ptr(initial), _ptr(out))
        if rc:
            raise OracleError(rc, "swept_solve")
        return out

    def substep(self, problem: int, stage: int, read1, read2, out, rects, params):
        nvars, ny, nx = read1.shape
        r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1, 4))
        rc = self.lib.sgo_substep(problem, stage, _ptr(read1), _ptr(read2), _ptr(out), nvars, nx, ny,
                                  _ptr(r, _ip), r.shape[0], _ptr(np.ascontiguousarray(params)))
        if rc:
            raise OracleError(rc, "substep")

    def pressure(self, q, gamma=1.4):
        q = np.ascontiguousarray(q, dtype=np.float64)
        p = np.zeros(1)
        rc = self.lib.sgo_pressure(_ptr(q), gamma, _ptr(p))
        if rc:
            raise OracleError(rc, "NonPhysicalState")
        return float(p[0])

    def minmod(self, q4x4, p4):
        q = np.ascontiguousarray(q4x4, dtype=np.float64).reshape(16)
        p = np.ascontiguousarray(p4, dtype=np.float64)
        ql, qr = np.zeros(4), np.zeros(4)
        self.lib.sgo_minmod(_ptr(q), _ptr(p), _ptr(ql), _ptr(qr))
        return ql, qr

    def interface_flux(self, ql, qr, axis, gamma=1.4):
        f = np.zeros(4)
        rc = self.lib.sgo_interface_flux(_ptr(np.ascontiguousarray(ql, dtype=np.float64)),
                                         _ptr(np.ascontiguousarray(qr, dtype=np.float64)), axis,
                                         gamma, _ptr(f))
        if rc:
            raise OracleError(rc, "NonPhysicalState")
        return f

    def fnv1a(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a, dtype=np.float64)
        return f"{self.lib.sgo_fnv1a(_ptr(a), a.size):016x}"


class Reference:
    """The reference library compiled from its own sources (oracle/_ref)."""

    def __init__(self, path: Path | None = None):
        path = path or REF_DIR / "libsweptgrid_ref.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = self.lib = C.CDLL(str(path))
        L.ref_run.argtypes = [C.c_char_p, _dp, C.c_long, C.c_char_p, C.c_long, C.c_char_p, C.c_long]
        L.ref_setup.argtypes = [C.c_char_p, _dp, C.c_long, _dp, C.c_char_p, C.c_long]
        L.ref_schedule.argtypes = [C.c_long, C.c_int, C.c_int, C.c_int, C.c_int, _lp, C.c_long, _lp,
                                   C.c_char_p, C.c_long]
        L.ref_schedule.restype = C.c_long
        L.ref_substep.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, _ip,
                                  C.c_int, _dp, _dp, C.c_int, C.c_char_p, C.c_long]
        L.ref_pressure.argtypes = [_dp, C.c_double, _dp, C.c_char_p, C.c_long]
        L.ref_interface_flux.argtypes = [_dp, _dp, C.c_int, C.c_double, _dp, C.c_char_p, C.c_long]
        L.ref_minmod.argtypes = [_dp, _dp, _dp, _dp]
        L.ref_minmod.restype = None
        L.ref_vortex_state.argtypes = [C.c_double, C.c_double, C.c_double, _dp, C.c_char_p, C.c_long]

    def run(self, cfg: dict, want_field: bool = True):
        nvars = 1 if cfg.get("problem", "heat") == "heat" else 4
        nx = cfg.get("nx", 64)
        out = np.zeros((nvars, nx, nx)) if want_field else None
        rec = C.create_string_buffer(1 << 20)
        err = C.create_string_buffer(1024)
        rc = self.lib.ref_run(json.dumps(cfg).encode(), _ptr(out) if want_field else None,
                              out.size if want_field else 0, rec, len(rec), err, len(err))
        if rc:
            raise OracleError(rc, err.value.decode())
        return out, json.loads(rec.value.decode())

    def setup(self, cfg: dict):
        nvars = 1 if cfg.get("problem", "heat") == "heat" else 4
        nx = cfg.get("nx", 64)
        init = np.zeros((nvars, nx, nx))
        d = np.zeros(3)
        err = C.create_string_buffer(1024)
        rc = self.lib.ref_setup(json.dumps(cfg).encode(), _ptr(init), init.size, _ptr(d), err, len(err))
        if rc:
            raise OracleError(rc, err.value.decode())
        return init, float(d[0]), float(d[1]), float(d[2])

    def schedule(self, steps_or_m: int, b: int, n: int, substeps: int, by_cycles: bool = False):
        cap = 1 << 20
        rows = np.zeros((cap, 9), dtype=np.int64)
        meta = np.zeros(4, dtype=np.int64)
        err = C.create_string_buffer(1024)
        cnt = self.lib.ref_schedule(steps_or_m, int(by_cycles), b, n, substeps, _ptr(rows, _lp), cap,
                                    _ptr(meta, _lp), err, len(err))
        if cnt < 0:
            raise OracleError(1, err.value.decode())
        return rows[:cnt].copy(), dict(octahedra=int(meta[0]), flat_level=int(meta[1]), k=int(meta[2]),
                                      substeps=int(meta[3]))

    def substep(self, problem: int, stage: int, read1, read2, out, rects, hp, ep, threads=0):
        nvars, ny, nx = read1.shape
        r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1, 4))
        err = C.create_string_buffer(1024)
        rc = self.lib.ref_substep(problem, stage, _ptr(read1), _ptr(read2), _ptr(out), nvars, nx, ny,
                                  _ptr(r, _ip), r.shape[0], _ptr(np.asarray(hp, dtype=np.float64)),
                                  _ptr(np.asarray(ep, dtype=np.float64)), threads, err, len(err))
        if rc:
            raise OracleError(rc, err.value.decode())


def restated_or_none():
    try:
        return Restated()
    except (FileNotFoundError, OSError):
        return None


def reference_or_none():
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None
