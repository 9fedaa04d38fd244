"""Python mirror of the reference loopdyn API over the B200 C-ABI.

Names and semantics follow /root/reference/proj/include/loopdyn:
`build_model` (model.hpp:117), `WorldBatch` (batch.hpp:14-54: add_world,
extract_state, insert_state, set_active, active, converged, diagnostics,
pose_offset, twist_offset, pose_storage, twist_storage), `batch_step`
(batch.hpp:58), `initial_state` (stepper.hpp:58) and `joint_coordinate`
(model.hpp:130).  Every call goes through libkamino_b200.so (include/kamino_b200.h);
there is no CPU fallback: if the library or a GPU is missing, calls raise.

Worlds are added on the host and the device batch is materialised on first
use (the device needs every world's capacity to lay out HBM once).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi
from .scene import ModelError, SceneDescription, StepConfig

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libkamino_b200.so")
_lib = None


class KaminoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def lib():
    """The sm_100a shared library.  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                               f"g.build()'` (no CPU fallback exists)")
        _lib = _capi.bind(C.CDLL(LIB_PATH), "kd_", _capi.KD_ONLY)
    return _lib


def _check(code):
    if code != 0:
        msg = lib().kd_last_error().decode()
        if code in _capi.MODEL_ERROR_CODES:
            raise ModelError(_capi.MODEL_ERROR_CODES[code], msg)
        raise KaminoError(code, msg)


# ------------------------------------------------------------------ model
class Model:
    """MechanismModel (model.hpp:97-113), built and validated by kd_model_build."""

    def __init__(self, scene: SceneDescription):
        desc, keep = scene.to_ctypes()
        h = C.c_void_p()
        _check(lib().kd_model_build_ex(C.byref(desc), C.c_uint32(scene.extension_bits()), C.byref(h)))
        self.handle = h
        self.scene = scene
        self.name = scene.name
        info = _capi.kd_model_info()
        lib().kd_model_get_info(h, C.byref(info))
        self.info = info
        self.body_names = [b.name for b in scene.bodies]
        self.joint_names = [j.name for j in scene.joints]

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.kd_model_destroy(h)
            self.handle = None

    n_bodies = property(lambda self: self.info.n_bodies)
    n_bilateral_rows = property(lambda self: self.info.n_bilateral_rows)
    n_dynamics_rows = property(lambda self: self.info.n_dynamics_rows)
    n_loops = property(lambda self: self.info.n_loops)

    def velocity_dim(self):
        return 6 * self.n_bodies

    def joint_layout(self):
        nj = self.info.n_joints
        arrs = [np.zeros(max(1, nj), np.int32) for _ in range(4)]
        _check(lib().kd_model_joint_layout(self.handle, *[_capi.i32ptr(a) for a in arrs]))
        return [a[:nj] for a in arrs]

    def joint_targets(self):
        t = np.zeros(max(1, self.info.n_joints))
        _check(lib().kd_model_joint_targets(self.handle, _capi.dptr(t)))
        return t[: self.info.n_joints]

    def joint_coordinate(self, joint: int, poses7) -> float:
        p = np.ascontiguousarray(poses7, dtype=np.float64).reshape(-1)
        out = C.c_double()
        _check(lib().kd_joint_coordinate(self.handle, int(joint), _capi.dptr(p), C.byref(out)))
        return out.value

    SPARSE_PLAN_FIELDS = ("slots", "nnz_L", "lv_len", "supernodes", "solve_levels", "program_words",
                          "factor_fma", "solve_terms", "dense_factor_fma", "smem_doubles_per_world", "solve_crit",
                          "solve_phases", "l_tile_mask", "x_tile_mask")

    def sparse_plan_info(self) -> Optional[dict]:
        """Statistics of the supernodal sparse-LLT plan (kd_snplan.h), or None
        if the model has none (its dense worlds then use the dense kernel)."""
        st = np.zeros(14, np.int64)
        if lib().kd_model_sparse_plan_info(self.handle, _capi.i64ptr(st)) != 0:
            return None
        return dict(zip(self.SPARSE_PLAN_FIELDS, (int(x) for x in st)))

    def sparse_plan_selftest(self, seed: int = 1) -> float:
        """Host-only check of the plan: max relative error of its factor/solve
        programs against a dense Cholesky on a random SPD system."""
        out = C.c_double()
        _check(lib().kd_model_sparse_plan_selftest(self.handle, int(seed), C.byref(out)))
        return out.value

    def initial_state(self) -> "WorldState":
        """initial_state (stepper.cpp:97-106)."""
        poses = np.array([list(b.position) + list(_normalized(b.orientation)) for b in self.scene.bodies],
                         dtype=np.float64).reshape(-1, 7)
        twists = np.array([list(b.linear_velocity) + list(b.angular_velocity) for b in self.scene.bodies],
                          dtype=np.float64).reshape(-1, 6)
        return WorldState(poses, twists, 0.0)


def _normalized(q):
    n = float(np.sqrt(q[1] * q[1] + q[2] * q[2] + q[3] * q[3] + q[0] * q[0]))
    return [q[0] / n, q[1] / n, q[2] / n, q[3] / n]


def build_model(scene: SceneDescription) -> Model:
    return Model(scene)


@dataclass
class JointReactionCache:
    """Converged bilateral + joint-dynamics reactions (stepper.hpp:38-43)."""
    lambda_: np.ndarray = field(default_factory=lambda: np.zeros(0))
    z: np.ndarray = field(default_factory=lambda: np.zeros(0))
    valid: bool = False


@dataclass
class ReactionCacheEntry:
    """Contact reaction cache entry (contacts.hpp:32-38); impulse and dual in
    the contact frame (n, t1, t2)."""
    geom_a: int
    geom_b: int
    position: np.ndarray
    impulse: np.ndarray
    dual: np.ndarray


@dataclass
class WorldState:
    """One world's state (stepper.hpp:49-56): body poses [x y z qw qx qy qz],
    twists [v; w], time and the three warm-start caches.  `limit_cache` maps
    (joint, bound) -> (lambda, z) like LimitReactionCache's std::map."""
    poses: np.ndarray
    twists: np.ndarray
    time: float = 0.0
    joint_cache: JointReactionCache = field(default_factory=JointReactionCache)
    limit_cache: dict = field(default_factory=dict)
    contact_cache: List[ReactionCacheEntry] = field(default_factory=list)


# ------------------------------------------------------------------ batch
class WorldBatch:
    """Device-resident heterogeneous world batch (batch.hpp:14-54)."""

    def __init__(self, device: int = 0):
        self.device = device
        self._models: List[Model] = []
        self._world_model: List[int] = []
        self._init: List[Optional[WorldState]] = []
        self.handle = None
        self._hist_cap = 0

    # -- building
    def add_world(self, model: Model, state: Optional[WorldState] = None) -> int:
        if self.handle is not None:
            raise RuntimeError("add_world after the batch was materialised on the device")
        idx = next((i for i, m in enumerate(self._models) if m is model), None)
        if idx is None:
            self._models.append(model)
            idx = len(self._models) - 1
        self._world_model.append(idx)
        self._init.append(state)
        return len(self._world_model) - 1

    def _ensure(self):
        if self.handle is not None:
            return
        wm = np.ascontiguousarray(self._world_model, dtype=np.int32)
        hs = (C.c_void_p * max(1, len(self._models)))(*[m.handle.value for m in self._models])
        h = C.c_void_p()
        _check(lib().kd_batch_create(self.device, hs, len(self._models), _capi.i32ptr(wm), len(wm), C.byref(h)))
        self.handle = h
        nw, pl, tl = C.c_int32(), C.c_int64(), C.c_int64()
        lib().kd_batch_size(h, C.byref(nw), C.byref(pl), C.byref(tl))
        self.n_worlds, self.pose_len, self.twist_len = nw.value, pl.value, tl.value
        self._pose_off = np.zeros(max(1, self.n_worlds), np.int32)
        self._twist_off = np.zeros(max(1, self.n_worlds), np.int32)
        lib().kd_batch_offsets(h, _capi.i32ptr(self._pose_off), _capi.i32ptr(self._twist_off))
        self.row_offset = np.zeros(max(1, self.n_worlds), np.int64)
        tot = C.c_int64()
        lib().kd_batch_row_offsets(h, _capi.i64ptr(self.row_offset), C.byref(tot))
        self.total_rows = tot.value
        if any(s is not None for s in self._init):
            p, t, tm = self.get_state()
            for w, s in enumerate(self._init):
                if s is not None:
                    nb = self._models[self._world_model[w]].n_bodies
                    p[self._pose_off[w]: self._pose_off[w] + 7 * nb] = np.asarray(s.poses).reshape(-1)
                    t[self._twist_off[w]: self._twist_off[w] + 6 * nb] = np.asarray(s.twists).reshape(-1)
                    tm[w] = s.time
            self.set_state(p, t, tm)
            for w, s in enumerate(self._init):
                if s is not None:
                    self.set_caches(w, s.joint_cache, s.limit_cache, s.contact_cache)
        self._active = np.ones(max(1, self.n_worlds), np.uint8)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.kd_batch_destroy(h)
            self.handle = None

    # -- reference accessors
    def size(self):
        return len(self._world_model)

    def model(self, w) -> Model:
        return self._models[self._world_model[w]]

    def pose_offset(self, w):
        self._ensure()
        return int(self._pose_off[w])

    def twist_offset(self, w):
        self._ensure()
        return int(self._twist_off[w])

    def pose_storage(self):
        return self.get_state()[0]

    def twist_storage(self):
        return self.get_state()[1]

    def extract_state(self, w) -> WorldState:
        """extract_state (batch.cpp:27-45): state and warm-start caches."""
        p, t, tm = self.get_state()
        nb = self.model(w).n_bodies
        po, to = self._pose_off[w], self._twist_off[w]
        s = WorldState(p[po: po + 7 * nb].reshape(nb, 7).copy(), t[to: to + 6 * nb].reshape(nb, 6).copy(),
                       float(tm[w]))
        s.joint_cache, s.limit_cache, s.contact_cache = self.get_caches(w)
        return s

    def insert_state(self, w, s: WorldState):
        """insert_state (batch.cpp:47-71): state and warm-start caches."""
        p, t, tm = self.get_state()
        nb = self.model(w).n_bodies
        po, to = self._pose_off[w], self._twist_off[w]
        p[po: po + 7 * nb] = np.asarray(s.poses).reshape(-1)
        t[to: to + 6 * nb] = np.asarray(s.twists).reshape(-1)
        tm[w] = s.time
        self.set_state(p, t, tm)
        self.set_caches(w, s.joint_cache, s.limit_cache, s.contact_cache)

    def get_caches(self, w):
        """(JointReactionCache, {(joint, bound): (lambda, z)}, [ReactionCacheEntry])
        of world w (kd_batch_get_caches)."""
        self._ensure()
        jl, jv, nl, nc = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().kd_batch_get_cache_sizes(self.handle, int(w), C.byref(jl), C.byref(jv), C.byref(nl),
                                              C.byref(nc)))
        lam, z = np.zeros(max(1, jl.value)), np.zeros(max(1, jl.value))
        lim = (_capi.kd_limit_cache_entry * max(1, nl.value))()
        con = (_capi.kd_contact_cache_entry * max(1, nc.value))()
        nl2, nc2, jv2 = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().kd_batch_get_caches(self.handle, int(w), _capi.dptr(lam), _capi.dptr(z), C.byref(jv2), lim,
                                         max(1, nl.value), C.byref(nl2), con, max(1, nc.value), C.byref(nc2)))
        jc = JointReactionCache(lam[: jl.value].copy(), z[: jl.value].copy(), bool(jv2.value))
        lc = {(lim[k].joint, lim[k].bound): (lim[k].lambda_, lim[k].z) for k in range(nl2.value)}
        cc = [ReactionCacheEntry(con[k].geom_a, con[k].geom_b, np.array(con[k].position[:]),
                                 np.array(con[k].impulse[:]), np.array(con[k].dual[:])) for k in range(nc2.value)]
        return jc, lc, cc

    def set_caches(self, w, joint_cache: JointReactionCache, limit_cache: dict, contact_cache):
        self._ensure()
        lam = np.ascontiguousarray(joint_cache.lambda_, dtype=np.float64).reshape(-1)
        z = np.ascontiguousarray(joint_cache.z, dtype=np.float64).reshape(-1)
        keys = sorted(limit_cache)
        lim = (_capi.kd_limit_cache_entry * max(1, len(keys)))()
        for k, key in enumerate(keys):
            lim[k].joint, lim[k].bound = int(key[0]), int(key[1])
            lim[k].lambda_, lim[k].z = float(limit_cache[key][0]), float(limit_cache[key][1])
        con = (_capi.kd_contact_cache_entry * max(1, len(contact_cache)))()
        for k, e in enumerate(contact_cache):
            con[k].geom_a, con[k].geom_b = int(e.geom_a), int(e.geom_b)
            for d in range(3):
                con[k].position[d] = float(e.position[d])
                con[k].impulse[d] = float(e.impulse[d])
                con[k].dual[d] = float(e.dual[d])
        _check(lib().kd_batch_set_caches(self.handle, int(w), _capi.dptr(lam if len(lam) else np.zeros(1)),
                                         _capi.dptr(z if len(z) else np.zeros(1)), len(lam),
                                         int(bool(joint_cache.valid)), lim, len(keys), con, len(contact_cache)))

    def set_active(self, w, active: bool):
        self._ensure()
        self._active[w] = 1 if active else 0
        _check(lib().kd_batch_set_active(self.handle, self._active.ctypes.data_as(_capi.c_uint8_p)))

    def active(self, w):
        self._ensure()
        return bool(self._active[w])

    def converged(self, w):
        return bool(self.diagnostics()[w].converged)

    # -- bulk state
    def get_state(self):
        self._ensure()
        p = np.zeros(max(1, self.pose_len))
        t = np.zeros(max(1, self.twist_len))
        tm = np.zeros(max(1, self.n_worlds))
        _check(lib().kd_batch_get_state(self.handle, _capi.dptr(p), _capi.dptr(t), _capi.dptr(tm)))
        return p[: self.pose_len], t[: self.twist_len], tm[: self.n_worlds]

    def set_state(self, poses=None, twists=None, time=None):
        self._ensure()
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
        p, t, tm = f(poses), f(twists), f(time)
        _check(lib().kd_batch_set_state(self.handle, _capi.dptr(p), _capi.dptr(t), _capi.dptr(tm)))

    def reset_caches(self):
        self._ensure()
        _check(lib().kd_batch_reset_caches(self.handle))

    # -- stepping
    def assemble(self, cfg: StepConfig):
        """assemble_constraints (constraints.hpp:91-94) for every active world
        at its current state, on the device, without solving or integrating;
        read the result with dump_rows / dump_contacts / dump_limits."""
        self._ensure()
        c = cfg.to_ctypes()
        _check(lib().kd_batch_assemble(self.handle, C.byref(c)))

    def step(self, cfg: StepConfig, n_steps: int = 1):
        self._ensure()
        c = cfg.to_ctypes()
        _check(lib().kd_batch_step(self.handle, C.byref(c), int(n_steps)))

    def step_async(self, cfg: StepConfig, n_steps: int = 1):
        """Enqueue n_steps on the batch stream without waiting (see sync())."""
        self._ensure()
        c = cfg.to_ctypes()
        _check(lib().kd_batch_step_async(self.handle, C.byref(c), int(n_steps)))

    def sync(self):
        _check(lib().kd_batch_sync(self.handle))

    def stream(self) -> int:
        """The batch's cudaStream_t as an integer (for torch.cuda.ExternalStream)."""
        self._ensure()
        s = C.c_void_p()
        _check(lib().kd_batch_stream(self.handle, C.byref(s)))
        return s.value or 0

    def fk(self, joints, values, tolerance=1e-8, max_iters=100, lm_initial=1e-6):
        """Batched forward kinematics on the device (fk_solve, fk.hpp:33):
        every active world's poses are moved to satisfy its joints' loop
        closures plus the targets.  `joints` / `values`: [n_worlds, n_targets]
        (a 1-D sequence is applied to every world).  Returns (iterations,
        residual_inf, converged) per world."""
        self._ensure()
        j = np.asarray(joints, dtype=np.int32)
        v = np.asarray(values, dtype=np.float64)
        if j.ndim == 1:
            j = np.tile(j, (self.n_worlds, 1))
        if v.ndim == 1:
            v = np.tile(v, (self.n_worlds, 1))
        j, v = np.ascontiguousarray(j), np.ascontiguousarray(v)
        nt = j.shape[1] if j.ndim == 2 else 0
        it = np.zeros(max(1, self.n_worlds), np.int32)
        res = np.zeros(max(1, self.n_worlds))
        conv = np.zeros(max(1, self.n_worlds), np.uint8)
        _check(lib().kd_batch_fk(self.handle, _capi.i32ptr(j), _capi.dptr(v), nt, float(tolerance), int(max_iters),
                                 float(lm_initial), _capi.i32ptr(it), _capi.dptr(res),
                                 conv.ctypes.data_as(_capi.c_uint8_p)))
        n = self.n_worlds
        return it[:n], res[:n], conv[:n].astype(bool)

    def device_state(self):
        """Zero-copy views of the device-resident state for PyTorch (RL
        wrappers, PAPER §2 Warp<->PyTorch interop): (poses [pose_len],
        twists [twist_len], time [n_worlds]) as float64 CUDA tensors sharing
        the batch's memory (__cuda_array_interface__).  Order work on them with
        the batch stream (`torch.cuda.ExternalStream(batch.stream())`)."""
        import torch
        self._ensure()
        p, t, tm = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().kd_batch_device_state(self.handle, C.byref(p), C.byref(t), C.byref(tm)))

        class _View:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                                 "version": 3, "strides": None, "stream": None}
        dev = torch.device("cuda", self.device)
        return (torch.as_tensor(_View(p.value, self.pose_len), device=dev),
                torch.as_tensor(_View(t.value, self.twist_len), device=dev),
                torch.as_tensor(_View(tm.value, self.n_worlds), device=dev))

    def set_state_async(self, poses, twists):
        """Host->device state copy on the batch stream (pass pinned buffers)."""
        _check(lib().kd_batch_set_state_async(self.handle, _capi.dptr(poses), _capi.dptr(twists)))

    def get_state_async(self, poses, twists):
        _check(lib().kd_batch_get_state_async(self.handle, _capi.dptr(poses), _capi.dptr(twists)))

    def diagnostics(self):
        self._ensure()
        d = (_capi.kd_step_diag * max(1, self.n_worlds))()
        _check(lib().kd_batch_get_diagnostics(self.handle, d))
        return d

    def impulses(self):
        self._ensure()
        out = np.zeros(max(1, self.total_rows))
        _check(lib().kd_batch_get_impulses(self.handle, _capi.dptr(out)))
        return out

    def set_history_capacity(self, cap):
        self._ensure()
        _check(lib().kd_batch_set_history_capacity(self.handle, int(cap)))
        self._hist_cap = int(cap)

    def history(self):
        out = np.zeros(max(1, self.n_worlds * self._hist_cap))
        _check(lib().kd_batch_get_history(self.handle, _capi.dptr(out)))
        return out[: self.n_worlds * self._hist_cap].reshape(self.n_worlds, self._hist_cap)

    def enable_timing(self, on=True):
        self._ensure()
        _check(lib().kd_batch_enable_timing(self.handle, int(on)))

    def timing(self):
        ms = np.zeros(4)
        n = C.c_int64()
        _check(lib().kd_batch_get_timing(self.handle, _capi.dptr(ms), C.byref(n)))
        return {"assemble_ms": ms[0], "dense_ms": ms[1], "matrix_free_ms": ms[2], "recover_ms": ms[3],
                "launches": n.value}

    def kernels(self):
        """Per world, the device kernel that solved the last step:
        'none' | 'dense' | 'supernodal' | 'supernodal+dense' | 'supernodal+cluster' | 'cr'."""
        self._ensure()
        out = np.zeros(max(1, self.n_worlds), np.int32)
        _check(lib().kd_batch_get_kernels(self.handle, _capi.i32ptr(out)))
        return [_capi.KERNEL_NAMES[int(k)] for k in out[: self.n_worlds]]

    def cr_paths(self):
        """Per world, the matrix-free kernel that solved the last step:
        'none' | 'incidence' | 'rows' | 'shared' (kd_batch_get_cr_paths)."""
        self._ensure()
        out = np.zeros(max(1, self.n_worlds), np.int32)
        _check(lib().kd_batch_get_cr_paths(self.handle, _capi.i32ptr(out)))
        return [_capi.CR_PATH_NAMES[int(k)] for k in out[: self.n_worlds]]

    def phase_cycles(self):
        """clock64 cycles per fused-kernel phase of the last step, [n_worlds, 8]."""
        self._ensure()
        out = np.zeros(8 * max(1, self.n_worlds), np.int64)
        _check(lib().kd_batch_get_phase_cycles(self.handle, _capi.i64ptr(out)))
        return out[: 8 * self.n_worlds].reshape(self.n_worlds, 8)

    # -- one-step introspection (parity)
    def dump_rows(self, w, cap=8192):
        rows = (_capi.kd_row_dump * cap)()
        n = C.c_int32()
        _check(lib().kd_batch_dump_rows(self.handle, int(w), rows, cap, C.byref(n)))
        return _rows_to_numpy(rows, n.value)

    def dump_contacts(self, w, cap=8192):
        g = np.zeros(2 * cap, np.int32)
        d = np.zeros(9 * cap)
        n = C.c_int32()
        _check(lib().kd_batch_dump_contacts(self.handle, int(w), _capi.i32ptr(g), _capi.dptr(d), cap, C.byref(n)))
        return g[: 2 * n.value].reshape(-1, 2), d[: 9 * n.value].reshape(-1, 9)

    def dump_limits(self, w, cap=8192):
        k = np.zeros(2 * cap, np.int32)
        n = C.c_int32()
        _check(lib().kd_batch_dump_limits(self.handle, int(w), _capi.i32ptr(k), cap, C.byref(n)))
        return k[: 2 * n.value].reshape(-1, 2)


def _rows_to_numpy(rows, n):
    out = {
        "body": np.array([[rows[i].body_a, rows[i].body_b] for i in range(n)], np.int32).reshape(n, 2),
        "kind": np.array([rows[i].kind for i in range(n)], np.int32),
        "J": np.array([list(rows[i].block_a) + list(rows[i].block_b) for i in range(n)]).reshape(n, 12),
    }
    for key, attr in (("bias", "bias"), ("reg", "reg"), ("scale", "scale"), ("vf", "vf_scaled"),
                      ("lambda", "lambda_"), ("z", "z")):
        out[key] = np.array([getattr(rows[i], attr) for i in range(n)])
    return out


@dataclass
class SolveProblem:
    """A pre-assembled system for the solver-level entry points
    (kd_solve_problem): ConstraintSet rows (constraints.hpp:19-65) in the order
    bilateral | limits | contacts, per-body inverse mass data
    (BodyInertiaWorld, delassus.hpp:13-18), the Preconditioner scale, the
    right-hand side (padmm_solve's preconditioned v_f, or cr_solve's rhs) and
    an optional warm start (PadmmInit x0 / z0, or cr_solve's x)."""
    body: np.ndarray          # (n, 2) int: body_a, body_b (-1 none)
    jacobian: np.ndarray      # (n, 12): block_a, block_b
    reg: np.ndarray           # (n,)
    scale: np.ndarray         # (n,)
    inv_mass: np.ndarray      # (nb,)
    inv_inertia: np.ndarray   # (nb, 3, 3) world frame
    rhs: np.ndarray           # (n,)
    n_bilateral: int = -1     # default: every row
    n_limits: int = 0
    n_contacts: int = 0
    mu: Optional[np.ndarray] = None
    x0: Optional[np.ndarray] = None
    z0: Optional[np.ndarray] = None

    def _c(self, keep):
        n = len(self.reg)
        nbil = n - self.n_limits - 3 * self.n_contacts if self.n_bilateral < 0 else self.n_bilateral
        f = lambda a, dt=np.float64: np.ascontiguousarray(a, dtype=dt).reshape(-1)  # noqa: E731
        arrs = dict(body=f(self.body, np.int32), jacobian=f(self.jacobian), reg=f(self.reg), scale=f(self.scale),
                    inv_mass=f(self.inv_mass), inv_inertia=f(self.inv_inertia), rhs=f(self.rhs),
                    mu=f(self.mu) if self.mu is not None else None, x0=f(self.x0) if self.x0 is not None else None,
                    z0=f(self.z0) if self.z0 is not None else None)
        keep.append(arrs)
        p = _capi.kd_solve_problem()
        p.n_rows, p.n_bodies = n, len(arrs["inv_mass"])
        p.n_bilateral, p.n_limits, p.n_contacts = nbil, self.n_limits, self.n_contacts
        p.body = _capi.i32ptr(arrs["body"])
        for k in ("jacobian", "reg", "scale", "inv_mass", "inv_inertia", "rhs", "mu", "x0", "z0"):
            setattr(p, k, _capi.dptr(arrs[k]))
        return p


def _problems(problems):
    keep = []
    arr = (_capi.kd_solve_problem * max(1, len(problems)))(*[q._c(keep) for q in problems])
    offs = np.concatenate([[0], np.cumsum([len(q.reg) for q in problems])]).astype(np.int64)
    return arr, keep, offs


_BACKENDS = {"dense": _capi.KD_BACKEND_DENSE, "sparse": _capi.KD_BACKEND_MATRIX_FREE,
             "matrix_free": _capi.KD_BACKEND_MATRIX_FREE, "auto": _capi.KD_BACKEND_AUTO}


def padmm_solve(problems, eta_rho: float, config: StepConfig, backend: str = "auto", cr_budget: int = 9,
                history_capacity: int = 0, device: int = 0):
    """build_backend + padmm_solve (delassus.hpp:103-105, padmm.hpp:64-67) for
    every problem, on the device.  Returns per problem a dict with lambda
    (preconditioned y), z, diag (kd_step_diag) and history (the combined
    residual per iteration; empty unless history_capacity > 0)."""
    arr, keep, offs = _problems(problems)
    lam, z = np.zeros(max(1, offs[-1])), np.zeros(max(1, offs[-1]))
    diags = (_capi.kd_step_diag * max(1, len(problems)))()
    hist = np.zeros(max(1, len(problems) * history_capacity))
    c = config.to_ctypes()
    _check(lib().kd_padmm_solve_batched(device, arr, len(problems), float(eta_rho), _BACKENDS[backend],
                                        int(cr_budget), C.byref(c), _capi.dptr(lam), _capi.dptr(z), diags,
                                        _capi.dptr(hist), int(history_capacity)))
    out = []
    for p in range(len(problems)):
        h = hist[p * history_capacity:(p + 1) * history_capacity]
        out.append({"lambda": lam[offs[p]:offs[p + 1]].copy(), "z": z[offs[p]:offs[p + 1]].copy(),
                    "diag": diags[p], "history": h[h != -1.0].copy()})
    return out


def cr_solve(problems, eta_rho: float, max_iters: int, history_capacity: int = 0, device: int = 0):
    """bake_jacobian + cr_solve (delassus.hpp:82-83) per problem on the device
    (x0 is the warm start).  Returns per problem a dict with x, iterations,
    breakdown, residual_norm and history (|r| initially and after every update)."""
    arr, keep, offs = _problems(problems)
    n = len(problems)
    x = np.zeros(max(1, offs[-1]))
    it = np.zeros(max(1, n), np.int32)
    brk = np.zeros(max(1, n), np.uint8)
    rn = np.zeros(max(1, n))
    hist = np.zeros(max(1, n * history_capacity))
    _check(lib().kd_cr_solve_batched(device, arr, n, float(eta_rho), int(max_iters), _capi.dptr(x), _capi.i32ptr(it),
                                     brk.ctypes.data_as(_capi.c_uint8_p), _capi.dptr(rn), _capi.dptr(hist),
                                     int(history_capacity)))
    out = []
    for p in range(n):
        h = hist[p * history_capacity:(p + 1) * history_capacity]
        out.append({"x": x[offs[p]:offs[p + 1]].copy(), "iterations": int(it[p]), "breakdown": bool(brk[p]),
                    "residual_norm": float(rn[p]), "history": h[h != -1.0].copy()})
    return out


def step(model: Model, state: WorldState, config: StepConfig, device: int = 0):
    """step (stepper.hpp:84, stepper.cpp:134-236) for one world: a one-world
    device batch warm-started from `state`'s caches; `state` is updated in
    place (poses, twists, time and caches) and the step's diagnostics are
    returned.  For many worlds use WorldBatch + batch_step."""
    b = WorldBatch(device)
    b.add_world(model, state)
    b.step(config)
    s = b.extract_state(0)
    state.poses, state.twists, state.time = s.poses, s.twists, s.time
    state.joint_cache, state.limit_cache, state.contact_cache = s.joint_cache, s.limit_cache, s.contact_cache
    return b.diagnostics()[0]


def batch_step(batch: WorldBatch, config: StepConfig, n_threads: int = 0):
    """batch_step (batch.hpp:58); `n_threads` is accepted for signature parity
    and ignored (the device runs every active world)."""
    batch.step(config, 1)


def bench_jitter(twists, n_bodies_per_world, seed=1, sigma=1e-3):
    """main.cpp:199-211 jitter stream (std::mt19937_64 + normal_distribution,
    libstdc++), applied in place to the batch twist storage."""
    t = np.ascontiguousarray(twists, dtype=np.float64)
    nb = np.ascontiguousarray(n_bodies_per_world, dtype=np.int32)
    _check(lib().kd_bench_jitter(C.c_uint64(seed), sigma, len(nb), _capi.i32ptr(nb), _capi.dptr(t)))
    return t
