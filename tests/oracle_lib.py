"""TEST INFRASTRUCTURE: ctypes wrapper over the CPU oracle (oracle/bin/liboracle.so).

Mirrors the method names of paper_2603_16536_b200.loopdyn (Model, WorldBatch)
so parity tests drive both through identical calls.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg import this module.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2603_16536_b200 import _capi
from paper_2603_16536_b200.scene import ModelError, StepConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB_PATH = os.path.join(ORACLE_DIR, "bin", "liboracle.so")
TESTS_BIN = os.path.join(ORACLE_DIR, "bin", "oracle_tests")
BUNDLE = os.path.join(ROOT, "tests", "golden", "scenes_bundle.json")

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = _capi.bind(C.CDLL(LIB_PATH), "or_", {
            "batch_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, _capi.c_int32_p, C.c_int32,
                                       C.POINTER(C.c_void_p)]),
            "batch_step": (C.c_int, [C.c_void_p, C.POINTER(_capi.kd_step_config), C.c_int32, C.c_int32]),
            "batch_set_trace": (C.c_int, [C.c_void_p, C.c_int32]),
            "batch_get_caches": _capi.KD_ONLY["batch_get_caches"],
            "bench_jitter": _capi.KD_ONLY["bench_jitter"],
            "batch_get_history": (C.c_int, [C.c_void_p, C.c_int32, _capi.c_double_p]),
            "batch_energy": (C.c_int, [C.c_void_p, C.c_int32, _capi.c_double_p, _capi.c_double_p]),
            "fd_check": (C.c_double, [C.c_void_p, _capi.c_double_p, C.c_double]),
            "fk_solve": (C.c_int, [C.c_void_p, _capi.c_int32_p, _capi.c_double_p, C.c_int32, _capi.c_double_p,
                                   C.c_double, C.c_int32, C.c_double, _capi.c_double_p, _capi.c_int32_p,
                                   _capi.c_int32_p]),
        })
    return _lib


def _check(code):
    if code != 0:
        msg = lib().or_last_error().decode()
        if code in _capi.MODEL_ERROR_CODES:
            raise ModelError(_capi.MODEL_ERROR_CODES[code], msg)
        raise RuntimeError(f"oracle error {code}: {msg}")


class OracleModel:
    def __init__(self, scene):
        desc, keep = scene.to_ctypes()
        h = C.c_void_p()
        _check(lib().or_model_build_ex(C.byref(desc), C.c_uint32(scene.extension_bits()), C.byref(h)))
        self.handle = h
        self.scene = scene
        info = _capi.kd_model_info()
        lib().or_model_get_info(h, C.byref(info))
        self.info = info

    def __del__(self):
        if getattr(self, "handle", None):
            lib().or_model_destroy(self.handle)
            self.handle = None

    @property
    def n_bodies(self):
        return self.info.n_bodies

    def joint_layout(self):
        nj = self.info.n_joints
        a = [np.zeros(max(1, nj), np.int32) for _ in range(4)]
        lib().or_model_joint_layout(self.handle, *[_capi.i32ptr(x) for x in a])
        return [x[:nj] for x in a]

    def joint_coordinate(self, joint, poses7):
        out = C.c_double()
        p = np.ascontiguousarray(poses7, dtype=np.float64)
        _check(lib().or_joint_coordinate(self.handle, joint, _capi.dptr(p), C.byref(out)))
        return out.value

    def fk(self, joints, values, poses7, tolerance=1e-8, max_iters=100, lm_initial=1e-6):
        """fk_solve (fk.cpp) on one world; returns (poses7, iterations, residual_inf, converged)."""
        j = np.ascontiguousarray(joints, dtype=np.int32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        p = np.array(poses7, dtype=np.float64).reshape(-1)
        res, it, conv = C.c_double(), C.c_int32(), C.c_int32()
        _check(lib().or_fk_solve(self.handle, _capi.i32ptr(j), _capi.dptr(v), len(j), _capi.dptr(p), tolerance,
                                 max_iters, lm_initial, C.byref(res), C.byref(it), C.byref(conv)))
        return p, it.value, res.value, bool(conv.value)

    def fd_check(self, poses7, step=1e-5):
        p = np.ascontiguousarray(poses7, dtype=np.float64)
        return lib().or_fd_check(self.handle, _capi.dptr(p), step)


class OracleBatch:
    """WorldBatch + batch_step on the CPU oracle (std::thread pool)."""

    def __init__(self, models, world_model, n_threads=0):
        self.models = list(models)
        wm = np.ascontiguousarray(world_model, dtype=np.int32)
        hs = (C.c_void_p * len(self.models))(*[m.handle.value for m in self.models])
        h = C.c_void_p()
        _check(lib().or_batch_create(hs, len(self.models), _capi.i32ptr(wm), len(wm), C.byref(h)))
        self.handle = h
        self.world_model = wm
        self.n_threads = n_threads
        nw, pl, tl = C.c_int32(), C.c_int64(), C.c_int64()
        lib().or_batch_size(h, C.byref(nw), C.byref(pl), C.byref(tl))
        self.n_worlds, self.pose_len, self.twist_len = nw.value, pl.value, tl.value
        self.pose_offset = np.zeros(self.n_worlds, np.int32)
        self.twist_offset = np.zeros(self.n_worlds, np.int32)
        lib().or_batch_offsets(h, _capi.i32ptr(self.pose_offset), _capi.i32ptr(self.twist_offset))
        self.row_offset = np.zeros(self.n_worlds, np.int64)
        tot = C.c_int64()
        lib().or_batch_row_offsets(h, _capi.i64ptr(self.row_offset), C.byref(tot))
        self.total_rows = tot.value

    def __del__(self):
        if getattr(self, "handle", None):
            lib().or_batch_destroy(self.handle)
            self.handle = None

    def set_trace(self, on=True):
        lib().or_batch_set_trace(self.handle, int(on))

    def get_state(self):
        p = np.zeros(self.pose_len)
        t = np.zeros(self.twist_len)
        tm = np.zeros(self.n_worlds)
        lib().or_batch_get_state(self.handle, _capi.dptr(p), _capi.dptr(t), _capi.dptr(tm))
        return p, t, tm

    def set_state(self, poses=None, twists=None, time=None):
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
        p, t, tm = f(poses), f(twists), f(time)
        lib().or_batch_set_state(self.handle, _capi.dptr(p), _capi.dptr(t), _capi.dptr(tm))

    def reset_caches(self):
        lib().or_batch_reset_caches(self.handle)

    def set_active(self, active):
        a = np.ascontiguousarray(active, dtype=np.uint8)
        lib().or_batch_set_active(self.handle, a.ctypes.data_as(_capi.c_uint8_p))

    def step(self, cfg: StepConfig, n_steps=1):
        c = cfg.to_ctypes()
        _check(lib().or_batch_step(self.handle, C.byref(c), n_steps, self.n_threads))

    def diagnostics(self):
        d = (_capi.kd_step_diag * self.n_worlds)()
        lib().or_batch_get_diagnostics(self.handle, d)
        return d

    def impulses(self):
        out = np.zeros(max(1, self.total_rows))
        lib().or_batch_get_impulses(self.handle, _capi.dptr(out))
        return out

    def history(self, cap):
        out = np.zeros(self.n_worlds * cap)
        lib().or_batch_get_history(self.handle, cap, _capi.dptr(out))
        return out.reshape(self.n_worlds, cap)

    def dump_rows(self, w, cap=4096):
        rows = (_capi.kd_row_dump * cap)()
        n = C.c_int32()
        _check(lib().or_batch_dump_rows(self.handle, w, rows, cap, C.byref(n)))
        return rows_to_numpy(rows, n.value)

    def dump_contacts(self, w, cap=4096):
        g = np.zeros(2 * cap, np.int32)
        d = np.zeros(9 * cap)
        n = C.c_int32()
        _check(lib().or_batch_dump_contacts(self.handle, w, _capi.i32ptr(g), _capi.dptr(d), cap, C.byref(n)))
        return g[: 2 * n.value].reshape(-1, 2), d[: 9 * n.value].reshape(-1, 9)

    def dump_limits(self, w, cap=4096):
        k = np.zeros(2 * cap, np.int32)
        n = C.c_int32()
        _check(lib().or_batch_dump_limits(self.handle, w, _capi.i32ptr(k), cap, C.byref(n)))
        return k[: 2 * n.value].reshape(-1, 2)

    def caches(self, w, cap=4096):
        """(joint lambda, joint z, joint valid, {(joint, bound): (lambda, z)},
        [(geom_a, geom_b, position, impulse, dual)]) of world w."""
        lam, z = np.zeros(cap), np.zeros(cap)
        jv, nl, nc = C.c_int32(), C.c_int32(), C.c_int32()
        lim = (_capi.kd_limit_cache_entry * cap)()
        con = (_capi.kd_contact_cache_entry * cap)()
        _check(lib().or_batch_get_caches(self.handle, int(w), _capi.dptr(lam), _capi.dptr(z), C.byref(jv), lim, cap,
                                         C.byref(nl), con, cap, C.byref(nc)))
        lc = {(lim[k].joint, lim[k].bound): (lim[k].lambda_, lim[k].z) for k in range(nl.value)}
        cc = [(con[k].geom_a, con[k].geom_b, np.array(con[k].position[:]), np.array(con[k].impulse[:]),
               np.array(con[k].dual[:])) for k in range(nc.value)]
        return lam, z, bool(jv.value), lc, cc

    def energy(self, w):
        ke, pe = C.c_double(), C.c_double()
        lib().or_batch_energy(self.handle, w, C.byref(ke), C.byref(pe))
        return ke.value, pe.value


def bench_jitter(twists, n_bodies_per_world, seed=1, sigma=1e-3):
    """The reference bench jitter stream (main.cpp:199-211) from the oracle
    library (same arithmetic as kd_bench_jitter; the reference arm of bench.py
    uses this one so that it never loads the product library)."""
    t = np.ascontiguousarray(twists, dtype=np.float64).copy()
    nb = np.ascontiguousarray(n_bodies_per_world, dtype=np.int32)
    _check(lib().or_bench_jitter(int(seed), float(sigma), len(nb), _capi.i32ptr(nb), _capi.dptr(t)))
    return t


def rows_to_numpy(rows, n):
    out = {
        "body": np.array([[rows[i].body_a, rows[i].body_b] for i in range(n)], np.int32).reshape(n, 2),
        "kind": np.array([rows[i].kind for i in range(n)], np.int32),
        "J": np.array([list(rows[i].block_a) + list(rows[i].block_b) for i in range(n)]).reshape(n, 12),
    }
    for key, attr in (("bias", "bias"), ("reg", "reg"), ("scale", "scale"), ("vf", "vf_scaled"),
                      ("lambda", "lambda_"), ("z", "z")):
        out[key] = np.array([getattr(rows[i], attr) for i in range(n)])
    return out


def load_bundle():
    import json
    with open(BUNDLE) as f:
        return json.load(f)


def bundled_scene(name):
    from paper_2603_16536_b200.scene import parse_scene_obj
    return parse_scene_obj(load_bundle()[name], name)
