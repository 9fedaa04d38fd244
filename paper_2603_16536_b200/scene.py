"""Scene description and step configuration (host side, mirrors the reference).

`parse_scene` restates /root/reference/proj/src/scene.cpp:86-174 (field names,
defaults, SceneError messages with `origin: where: msg` context, quaternion unit
check + normalisation).  `StepConfig` mirrors StepConfig/PadmmConfig
(stepper.hpp:16-34, padmm.hpp:8-17) and `apply_scene_config` mirrors
stepper.cpp:74-95.  `SceneDescription.to_ctypes()` produces the kd_scene_desc
the C-ABI (include/kamino_b200.h) consumes.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional

from . import _capi


class SceneError(RuntimeError):
    """SceneError (scene.hpp:74-77)."""


class ModelError(RuntimeError):
    """ModelError{Code} (model.hpp:76-94); `.code` is the Code name."""

    def __init__(self, code: str, msg: str):
        super().__init__(msg)
        self.code = code


def _identity_quat():
    return [1.0, 0.0, 0.0, 0.0]


@dataclass
class SceneBody:
    name: str
    mass: float = 1.0
    inertia: List[List[float]] = field(default_factory=lambda: [[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]])
    position: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    orientation: List[float] = field(default_factory=_identity_quat)  # [w,x,y,z]
    linear_velocity: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    angular_velocity: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])


@dataclass
class SceneJoint:
    name: str
    type: str
    parent: str
    child: str
    parent_position: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    parent_orientation: List[float] = field(default_factory=_identity_quat)
    child_position: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    child_orientation: List[float] = field(default_factory=_identity_quat)
    axis: List[float] = field(default_factory=lambda: [0.0, 0.0, 1.0])
    limits: Optional[List[float]] = None
    kp: float = 0.0
    kd: float = 0.0
    target: Optional[float] = None
    target_rate: float = 0.0
    armature: float = 0.0
    damping: float = 0.0


@dataclass
class SceneGeom:
    body: str
    shape: str
    radius: float = 0.0
    half_extents: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    normal: List[float] = field(default_factory=lambda: [0.0, 0.0, 1.0])
    offset: float = 0.0
    mu: float = 0.0
    restitution: float = 0.0


@dataclass
class SceneConfig:
    """Optional overrides carried by the scene file (scene.hpp:53-63)."""
    dt: Optional[float] = None
    integrator: Optional[str] = None
    backend: Optional[str] = None
    beta: Optional[float] = None
    rho: Optional[float] = None
    eta: Optional[float] = None
    eps: Optional[float] = None
    max_iters: Optional[int] = None
    cr_iters: Optional[int] = None


@dataclass
class SceneDescription:
    name: str = "scene"
    gravity: List[float] = field(default_factory=lambda: [0.0, 0.0, -9.81])
    bodies: List[SceneBody] = field(default_factory=list)
    joints: List[SceneJoint] = field(default_factory=list)
    geoms: List[SceneGeom] = field(default_factory=list)
    config: SceneConfig = field(default_factory=SceneConfig)
    # opt-in extensions beyond the reference (kd_model_build_ex): "box_box"
    extensions: List[str] = field(default_factory=list)

    def extension_bits(self) -> int:
        bits = {"box_box": 1}  # KD_EXT_BOX_BOX
        out = 0
        for e in self.extensions:
            if e not in bits:
                raise ValueError(f"unknown extension '{e}'")
            out |= bits[e]
        return out

    def copy(self) -> "SceneDescription":
        return dataclasses.replace(
            self,
            gravity=list(self.gravity),
            bodies=[dataclasses.replace(b) for b in self.bodies],
            joints=[dataclasses.replace(j) for j in self.joints],
            geoms=[dataclasses.replace(g) for g in self.geoms],
            config=dataclasses.replace(self.config),
            extensions=list(self.extensions),
        )

    # ---- C-ABI marshalling -------------------------------------------------
    def to_ctypes(self):
        """Returns (kd_scene_desc, keepalive).  Keep `keepalive` referenced
        for as long as the descriptor is used."""
        keep = []

        def s(x):
            b = x.encode()
            keep.append(b)
            return b

        def arr(t, vals):
            return t(*[float(v) for v in vals])

        bodies = (_capi.kd_body_desc * max(1, len(self.bodies)))()
        for i, b in enumerate(self.bodies):
            d = bodies[i]
            d.name = s(b.name)
            d.mass = float(b.mass)
            d.inertia = arr(C.c_double * 9, [v for row in b.inertia for v in row])
            d.position = arr(C.c_double * 3, b.position)
            d.orientation = arr(C.c_double * 4, b.orientation)
            d.linear_velocity = arr(C.c_double * 3, b.linear_velocity)
            d.angular_velocity = arr(C.c_double * 3, b.angular_velocity)
        joints = (_capi.kd_joint_desc * max(1, len(self.joints)))()
        for i, j in enumerate(self.joints):
            d = joints[i]
            d.name = s(j.name)
            d.type = s(j.type)
            d.parent = s(j.parent)
            d.child = s(j.child)
            d.parent_position = arr(C.c_double * 3, j.parent_position)
            d.parent_orientation = arr(C.c_double * 4, j.parent_orientation)
            d.child_position = arr(C.c_double * 3, j.child_position)
            d.child_orientation = arr(C.c_double * 4, j.child_orientation)
            d.axis = arr(C.c_double * 3, j.axis)
            d.has_limits = 1 if j.limits is not None else 0
            if j.limits is not None:
                d.lower, d.upper = float(j.limits[0]), float(j.limits[1])
            d.kp, d.kd = float(j.kp), float(j.kd)
            d.has_target = 1 if j.target is not None else 0
            d.target = float(j.target) if j.target is not None else 0.0
            d.target_rate = float(j.target_rate)
            d.armature = float(j.armature)
            d.damping = float(j.damping)
        geoms = (_capi.kd_geom_desc * max(1, len(self.geoms)))()
        for i, g in enumerate(self.geoms):
            d = geoms[i]
            d.body = s(g.body)
            d.shape = s(g.shape)
            d.radius = float(g.radius)
            d.half_extents = arr(C.c_double * 3, g.half_extents)
            d.normal = arr(C.c_double * 3, g.normal)
            d.offset = float(g.offset)
            d.mu = float(g.mu)
            d.restitution = float(g.restitution)
        desc = _capi.kd_scene_desc()
        desc.name = s(self.name)
        desc.gravity = arr(C.c_double * 3, self.gravity)
        desc.n_bodies = len(self.bodies)
        desc.bodies = C.cast(bodies, C.POINTER(_capi.kd_body_desc))
        desc.n_joints = len(self.joints)
        desc.joints = C.cast(joints, C.POINTER(_capi.kd_joint_desc))
        desc.n_geoms = len(self.geoms)
        desc.geoms = C.cast(geoms, C.POINTER(_capi.kd_geom_desc))
        keep += [bodies, joints, geoms]
        return desc, keep


# ---------------------------------------------------------------- parse (scene.cpp)
def _fail(origin, where, msg):
    raise SceneError(f"{origin}: {where}: {msg}")


def _is_number(v):
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _get_number(j, key, origin, where, fallback=None):  # scene.cpp:18-26
    if key not in j:
        if fallback is not None:
            return float(fallback)
        _fail(origin, where, f"missing field '{key}'")
    if not _is_number(j[key]):
        _fail(origin, where, f"field '{key}' must be a number")
    return float(j[key])


def _get_string(j, key, origin, where, fallback=None):  # scene.cpp:28-36
    if key not in j:
        if fallback is not None:
            return fallback
        _fail(origin, where, f"missing field '{key}'")
    if not isinstance(j[key], str):
        _fail(origin, where, f"field '{key}' must be a string")
    return j[key]


def _get_vec3(j, key, origin, where, fallback=None):  # scene.cpp:38-49
    if key not in j:
        if fallback is not None:
            return list(fallback)
        _fail(origin, where, f"missing field '{key}'")
    v = j[key]
    if not isinstance(v, list) or len(v) != 3:
        _fail(origin, where, f"field '{key}' must be an array of 3 numbers")
    return [float(x) for x in v]


def _get_quat(j, key, origin, where):  # scene.cpp:51-62
    if key not in j:
        return _identity_quat()
    v = j[key]
    if not isinstance(v, list) or len(v) != 4:
        _fail(origin, where, f"field '{key}' must be [w,x,y,z]")
    w, x, y, z = (float(a) for a in v)
    n = math.sqrt(x * x + y * y + z * z + w * w)
    if abs(n - 1.0) > 1e-6:
        _fail(origin, where, f"field '{key}' is not a unit quaternion")
    return [w / n, x / n, y / n, z / n]


def _get_inertia(j, origin, where):  # scene.cpp:64-79
    if "inertia" not in j:
        _fail(origin, where, "missing field 'inertia'")
    v = j["inertia"]
    if isinstance(v, list) and len(v) == 3 and _is_number(v[0]):
        return [[float(v[0]), 0.0, 0.0], [0.0, float(v[1]), 0.0], [0.0, 0.0, float(v[2])]]
    if isinstance(v, list) and len(v) == 3 and isinstance(v[0], list):
        rows = []
        for r in range(3):
            if not isinstance(v[r], list) or len(v[r]) != 3:
                _fail(origin, where, "inertia rows must have 3 entries")
            rows.append([float(x) for x in v[r]])
        return rows
    _fail(origin, where, "'inertia' must be a diagonal [ixx,iyy,izz] or a 3x3 matrix")


def parse_scene_obj(root: dict, origin: str = "<string>") -> SceneDescription:
    """parse_scene (scene.cpp:86-174) over an already-decoded JSON object."""
    scene = SceneDescription()
    scene.name = root.get("name", "scene")
    scene.gravity = _get_vec3(root, "gravity", origin, "top level", [0.0, 0.0, -9.81])
    for idx, jb in enumerate(root.get("bodies", [])):
        where = f"bodies[{idx}]"
        scene.bodies.append(SceneBody(
            name=_get_string(jb, "name", origin, where),
            mass=_get_number(jb, "mass", origin, where),
            inertia=_get_inertia(jb, origin, where),
            position=_get_vec3(jb, "position", origin, where, [0.0, 0.0, 0.0]),
            orientation=_get_quat(jb, "orientation", origin, where),
            linear_velocity=_get_vec3(jb, "linear_velocity", origin, where, [0.0, 0.0, 0.0]),
            angular_velocity=_get_vec3(jb, "angular_velocity", origin, where, [0.0, 0.0, 0.0]),
        ))
    for idx, jj in enumerate(root.get("joints", [])):
        where = f"joints[{idx}]"
        j = SceneJoint(
            name=_get_string(jj, "name", origin, where, f"joint{idx}"),
            type=_get_string(jj, "type", origin, where),
            parent=_get_string(jj, "parent", origin, where),
            child=_get_string(jj, "child", origin, where),
        )
        j.parent_position = _get_vec3(jj, "parent_position", origin, where, [0.0, 0.0, 0.0])
        j.parent_orientation = _get_quat(jj, "parent_orientation", origin, where)
        j.child_position = _get_vec3(jj, "child_position", origin, where, [0.0, 0.0, 0.0])
        j.child_orientation = _get_quat(jj, "child_orientation", origin, where)
        j.axis = _get_vec3(jj, "axis", origin, where, [0.0, 0.0, 1.0])
        if "limits" in jj:
            v = jj["limits"]
            if not isinstance(v, list) or len(v) != 2:
                _fail(origin, where, "'limits' must be [lower, upper]")
            j.limits = [float(v[0]), float(v[1])]
        j.kp = _get_number(jj, "kp", origin, where, 0.0)
        j.kd = _get_number(jj, "kd", origin, where, 0.0)
        if "target" in jj:
            j.target = _get_number(jj, "target", origin, where)
        j.target_rate = _get_number(jj, "target_rate", origin, where, 0.0)
        j.armature = _get_number(jj, "armature", origin, where, 0.0)
        j.damping = _get_number(jj, "damping", origin, where, 0.0)
        scene.joints.append(j)
    for idx, jg in enumerate(root.get("geoms", [])):
        where = f"geoms[{idx}]"
        g = SceneGeom(body=_get_string(jg, "body", origin, where), shape=_get_string(jg, "shape", origin, where))
        if g.shape == "sphere":
            g.radius = _get_number(jg, "radius", origin, where)
        elif g.shape == "box":
            g.half_extents = _get_vec3(jg, "half_extents", origin, where)
        elif g.shape == "plane":
            g.normal = _get_vec3(jg, "normal", origin, where, [0.0, 0.0, 1.0])
            g.offset = _get_number(jg, "offset", origin, where, 0.0)
        else:
            _fail(origin, where, f"unknown shape '{g.shape}'")
        g.mu = _get_number(jg, "mu", origin, where, 0.0)
        g.restitution = _get_number(jg, "restitution", origin, where, 0.0)
        scene.geoms.append(g)
    if "extensions" in root:  # not in the reference's scene format (opt-in, kd_model_build_ex)
        scene.extensions = [str(e) for e in root["extensions"]]
        scene.extension_bits()
    if "config" in root:  # scene.cpp:159-172
        jc = root["config"]
        c = scene.config
        if "dt" in jc:
            c.dt = float(jc["dt"])
        if "integrator" in jc:
            c.integrator = str(jc["integrator"])
        if "backend" in jc:
            c.backend = str(jc["backend"])
        if "beta" in jc:
            c.beta = float(jc["beta"])
        js = jc.get("solver", jc)
        for key in ("rho", "eta", "eps"):
            if key in js:
                setattr(c, key, float(js[key]))
        for key in ("max_iters", "cr_iters"):
            if key in js:
                setattr(c, key, int(js[key]))
    return scene


def parse_scene(json_text: str, origin: str = "<string>") -> SceneDescription:
    try:
        root = json.loads(json_text)
    except json.JSONDecodeError as e:
        raise SceneError(f"{origin}: {e}") from None
    return parse_scene_obj(root, origin)


def load_scene_file(path: str) -> SceneDescription:  # scene.cpp:176-182
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise SceneError(f"cannot open scene file: {path}") from None
    return parse_scene(text, path)


def serialize_scene(scene: SceneDescription) -> str:  # scene.cpp:184-241
    root = {"name": scene.name, "gravity": list(scene.gravity), "bodies": [], "joints": [], "geoms": []}
    for b in scene.bodies:
        root["bodies"].append({
            "name": b.name, "mass": b.mass, "inertia": [list(r) for r in b.inertia],
            "position": list(b.position), "orientation": list(b.orientation),
            "linear_velocity": list(b.linear_velocity), "angular_velocity": list(b.angular_velocity)})
    for j in scene.joints:
        jj = {"name": j.name, "type": j.type, "parent": j.parent, "child": j.child,
              "parent_position": list(j.parent_position), "parent_orientation": list(j.parent_orientation),
              "child_position": list(j.child_position), "child_orientation": list(j.child_orientation),
              "axis": list(j.axis)}
        if j.limits is not None:
            jj["limits"] = list(j.limits)
        if j.kp != 0 or j.kd != 0:
            jj["kp"], jj["kd"] = j.kp, j.kd
            if j.target is not None:
                jj["target"] = j.target
            jj["target_rate"] = j.target_rate
        if j.armature != 0:
            jj["armature"] = j.armature
        if j.damping != 0:
            jj["damping"] = j.damping
        root["joints"].append(jj)
    for g in scene.geoms:
        jg = {"body": g.body, "shape": g.shape}
        if g.shape == "sphere":
            jg["radius"] = g.radius
        if g.shape == "box":
            jg["half_extents"] = list(g.half_extents)
        if g.shape == "plane":
            jg["normal"] = list(g.normal)
            jg["offset"] = g.offset
        jg["mu"] = g.mu
        jg["restitution"] = g.restitution
        root["geoms"].append(jg)
    return json.dumps(root, indent=2)


# ---------------------------------------------------------------- step config
@dataclass
class StepConfig:
    """StepConfig + PadmmConfig defaults (stepper.hpp:16-34, padmm.hpp:8-17)."""
    dt: float = 1.0 / 240.0
    integrator: str = "euler"          # "euler" | "moreau"
    backend: str = "auto"              # "dense" | "sparse" | "auto"
    eta: float = 1e-6
    rho: float = 0.1
    eps: float = 1e-6
    max_iters: int = 200
    acceleration: bool = True
    restart: bool = True
    fixed_iteration_mode: bool = False
    cr_iters: int = 9
    baumgarte_beta: float = 0.2
    contact_margin: float = 0.01
    impact_velocity_threshold: float = 0.1
    bias_clamp: float = 10.0
    limit_margin_angular: float = 0.01
    limit_margin_linear: float = 0.001
    warm_start: bool = True

    def to_ctypes(self) -> _capi.kd_step_config:
        c = _capi.kd_step_config()
        c.dt = self.dt
        c.integrator = _capi.KD_INTEGRATOR_MOREAU_JEAN if self.integrator == "moreau" else \
            _capi.KD_INTEGRATOR_SEMI_IMPLICIT_EULER
        c.backend = {"dense": _capi.KD_BACKEND_DENSE, "sparse": _capi.KD_BACKEND_MATRIX_FREE}.get(
            self.backend, _capi.KD_BACKEND_AUTO)
        c.eta, c.rho, c.eps = self.eta, self.rho, self.eps
        c.max_iters = int(self.max_iters)
        c.acceleration = int(bool(self.acceleration))
        c.restart = int(bool(self.restart))
        c.fixed_iteration_mode = int(bool(self.fixed_iteration_mode))
        c.cr_iters = int(self.cr_iters)
        c.baumgarte_beta = self.baumgarte_beta
        c.contact_margin = self.contact_margin
        c.impact_velocity_threshold = self.impact_velocity_threshold
        c.bias_clamp = self.bias_clamp
        c.limit_margin_angular = self.limit_margin_angular
        c.limit_margin_linear = self.limit_margin_linear
        c.warm_start = int(bool(self.warm_start))
        return c


def apply_scene_config(cfg: StepConfig, ov: SceneConfig) -> StepConfig:
    """stepper.cpp:74-95."""
    if ov.dt is not None:
        cfg.dt = ov.dt
    if ov.integrator is not None:
        cfg.integrator = "moreau" if ov.integrator == "moreau" else "euler"
    if ov.backend is not None:
        cfg.backend = ov.backend if ov.backend in ("dense", "sparse") else "auto"
    if ov.beta is not None:
        cfg.baumgarte_beta = ov.beta
    if ov.rho is not None:
        cfg.rho = ov.rho
    if ov.eta is not None:
        cfg.eta = ov.eta
    if ov.eps is not None:
        cfg.eps = ov.eps
    if ov.max_iters is not None:
        cfg.max_iters = ov.max_iters
    if ov.cr_iters is not None:
        cfg.cr_iters = ov.cr_iters
    return cfg


def config_for(scene: SceneDescription) -> StepConfig:
    return apply_scene_config(StepConfig(), scene.config)
