"""Synthetic benchmark mechanisms (BASELINE.json configs 2-5).

None of these scenes exists in the reference: they are generated
here in the reference's own scene schema (scene.cpp:86-174) so the same
description drives the device path and the CPU oracle.

* `dr_legs()`   — config 2: a DR-Legs-like biped, 31 bodies, 36 revolute
  joints (12 PD-actuated, 24 passive), 6 kinematic loops (3 parallelogram
  transmissions per leg), free-floating pelvis, sphere pads on the feet
  (box feet are impossible: box-box/box-sphere pairs are rejected,
  model.cpp:238-250), ground plane z = 0.  n = 180 bilateral + 12 PD rows
  + active pad limits + 3 per contact.  Every loop is a parallelogram, so the
  initial pose is exactly consistent (f = 0).
* `closed_chain(n_cells)` — config 4: a ladder of parallelogram cells hanging
  from the world (n > 300 rows -> matrix-free CR path).
* `sphere_pile(n)` — config 5 substitute: spheres in a bin of 5 planes.
* `stewart_tower(stages)` — config 4 as SURVEY §8d specifies it: a spatial
  parallel manipulator, a stack of 6-6 Stewart platforms with
  spherical-prismatic-spherical legs (PD + damping on every leg, limits on the
  bottom stage).  12 stages: 156 bodies, 216 joints, 936 rows + 12 limit-row
  capacity -> matrix-free CR path.
* `mixed_joints()` — every joint type and joint-dynamics row kind in one
  small world: fixed, spherical, revolute and prismatic joints, PD, armature
  and damping rows, and a prismatic limit that is active from the start
  (the linear 0.001 m margin, constraints.cpp:218-229).
"""
from __future__ import annotations

import math

from .scene import SceneDescription, parse_scene_obj


def _box_inertia(m, a, b, c):
    """Solid box with full extents a, b, c (triangle inequality holds)."""
    return [m * (b * b + c * c) / 12.0, m * (a * a + c * c) / 12.0, m * (a * a + b * b) / 12.0]


def _sub(a, b):
    return [a[0] - b[0], a[1] - b[1], a[2] - b[2]]


def _add(a, b):
    return [a[0] + b[0], a[1] + b[1], a[2] + b[2]]


class _Builder:
    def __init__(self, name, gravity=(0.0, 0.0, -9.81)):
        self.root = {"name": name, "gravity": list(gravity), "bodies": [], "joints": [], "geoms": []}
        self.pos = {}

    def body(self, name, mass, dims, pos):
        self.pos[name] = list(pos)
        self.root["bodies"].append({"name": name, "mass": mass, "inertia": _box_inertia(mass, *dims),
                                    "position": list(pos), "orientation": [1.0, 0.0, 0.0, 0.0]})

    def joint(self, name, parent, child, anchor, axis, **kw):
        """Revolute joint through world point `anchor` (all bodies start at
        identity orientation, so joint frames are identity and the anchor
        offsets are plain differences)."""
        ppos = [0.0, 0.0, 0.0] if parent == "world" else self.pos[parent]
        j = {"name": name, "type": kw.pop("type", "revolute"), "parent": parent, "child": child,
             "parent_position": _sub(anchor, ppos), "child_position": _sub(anchor, self.pos[child]),
             "axis": list(axis)}
        j.update(kw)
        self.root["joints"].append(j)

    def geom(self, **g):
        self.root["geoms"].append(g)

    def scene(self) -> SceneDescription:
        return parse_scene_obj(self.root, self.root["name"])


X, Y, Z = (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)


def dr_legs(kp=15.0, kd=0.6, pad_mu=0.8, dt=1.0 / 250.0, integrator="moreau", pad_mass=0.1, pad_size=0.04,
            pad_limit=0.02) -> SceneDescription:
    """DR-Legs-like biped (config 2).  PD gains kp=15, kd=0.6 and the 250 Hz
    Moreau-Jean step follow PAPER.md:381-382 as quoted in SURVEY.md §8d."""
    L1, L2 = 0.30, 0.30        # thigh, shank
    pad_r = 0.02
    foot_drop = 0.05           # ankle -> pad centre (vertical)
    H = L1 + L2 + 0.10 + foot_drop + pad_r  # pelvis joint plane height: pads touch z = 0
    b = _Builder("dr_legs")
    b.body("pelvis", 1.0, (0.15, 0.25, 0.08), (0.0, 0.0, H))
    for side, s in (("l", 1.0), ("r", -1.0)):
        y0 = 0.1 * s
        n = lambda k: f"{side}_{k}"  # noqa: E731
        hip = [0.0, y0, H - 0.10]          # roll + pitch axes intersect here
        knee = _add(hip, [0.0, 0.0, -L1])
        ankle = _add(knee, [0.0, 0.0, -L2])
        # serial hip
        b.body(n("hip_yaw"), 0.10, (0.04, 0.04, 0.05), [0.0, y0, H - 0.05])
        b.joint(n("hip_yaw_j"), "pelvis", n("hip_yaw"), [0.0, y0, H - 0.02], Z, kp=kp, kd=kd)
        b.body(n("hip_roll"), 0.10, (0.05, 0.04, 0.04), hip)
        b.joint(n("hip_roll_j"), n("hip_yaw"), n("hip_roll"), hip, X, kp=kp, kd=kd)
        b.body(n("thigh"), 0.30, (0.04, 0.04, L1), _add(hip, [0.0, 0.0, -L1 / 2]))
        b.joint(n("hip_pitch_j"), n("hip_roll"), n("thigh"), hip, Y, kp=kp, kd=kd)
        b.body(n("shank"), 0.20, (0.03, 0.03, L2), _add(knee, [0.0, 0.0, -L2 / 2]))
        b.joint(n("knee_j"), n("thigh"), n("shank"), knee, Y)
        # loop 1: knee parallelogram  thigh(P) - crank - rod - shank(K)
        P = _add(hip, [0.0, 0.0, -0.05])
        o = [0.06, 0.0, 0.0]
        b.body(n("knee_crank"), 0.05, (0.06, 0.02, 0.02), _add(P, [0.03, 0.0, 0.0]))
        b.joint(n("knee_act_j"), n("thigh"), n("knee_crank"), P, Y, kp=kp, kd=kd)
        b.body(n("knee_rod"), 0.05, (0.01, 0.01, L1 - 0.05), _add(_add(P, o), [0.0, 0.0, -(L1 - 0.05) / 2]))
        b.joint(n("knee_rod_top_j"), n("knee_crank"), n("knee_rod"), _add(P, o), Y)
        b.joint(n("knee_rod_bot_j"), n("knee_rod"), n("shank"), _add(knee, o), Y)
        # loop 2: ankle drive  thigh(P2) - crank - rod1 - idler (pivots on shank at K)
        P2 = _add(hip, [0.0, 0.0, -0.10])
        o2 = [-0.05, 0.0, 0.0]
        b.body(n("ankle_crank"), 0.05, (0.05, 0.02, 0.02), _add(P2, [-0.025, 0.0, 0.0]))
        b.joint(n("ankle_act_j"), n("thigh"), n("ankle_crank"), P2, Y, kp=kp, kd=kd)
        b.body(n("ankle_rod1"), 0.05, (0.01, 0.01, L1 - 0.10), _add(_add(P2, o2), [0.0, 0.0, -(L1 - 0.10) / 2]))
        b.joint(n("ankle_rod1_top_j"), n("ankle_crank"), n("ankle_rod1"), _add(P2, o2), Y)
        b.body(n("ankle_idler"), 0.04, (0.08, 0.02, 0.02), _add(knee, [-0.005, 0.0, 0.0]))
        b.joint(n("ankle_idler_j"), n("shank"), n("ankle_idler"), knee, Y)
        b.joint(n("ankle_rod1_bot_j"), n("ankle_rod1"), n("ankle_idler"), _add(knee, o2), Y)
        # loop 3: idler - rod2 - ankle link (pivots on shank at A)
        o3 = [0.04, 0.0, 0.0]
        b.body(n("ankle_rod2"), 0.05, (0.01, 0.01, L2), _add(_add(knee, o3), [0.0, 0.0, -L2 / 2]))
        b.joint(n("ankle_rod2_top_j"), n("ankle_idler"), n("ankle_rod2"), _add(knee, o3), Y)
        b.body(n("ankle_link"), 0.05, (0.05, 0.03, 0.02), _add(ankle, [0.02, 0.0, 0.0]))
        b.joint(n("ankle_pitch_j"), n("shank"), n("ankle_link"), ankle, Y)
        b.joint(n("ankle_rod2_bot_j"), n("ankle_rod2"), n("ankle_link"), _add(ankle, o3), Y)
        # foot (ankle roll) + three sprung-free pads with tight limits
        b.body(n("foot"), 0.15, (0.18, 0.08, 0.03), _add(ankle, [0.02, 0.0, -0.03]))
        b.joint(n("ankle_roll_j"), n("ankle_link"), n("foot"), ankle, X, kp=kp, kd=kd)
        pads = (("toe", [0.09, 0.0, -foot_drop], [0.07, 0.0, -0.04], Y),
                ("heel", [-0.06, 0.0, -foot_drop], [-0.04, 0.0, -0.04], Y),
                ("side", [0.02, 0.04 * s, -foot_drop], [0.02, 0.02 * s, -0.04], X))
        for pad, centre, pivot, axis in pads:
            c = _add(ankle, centre)
            b.body(n(pad), pad_mass, (pad_size, pad_size, pad_size), c)
            b.joint(n(pad + "_j"), n("foot"), n(pad), _add(ankle, pivot), axis, limits=[-pad_limit, pad_limit])
            b.geom(body=n(pad), shape="sphere", radius=pad_r, mu=pad_mu, restitution=0.0)
    b.geom(body="world", shape="plane", normal=[0.0, 0.0, 1.0], offset=0.0, mu=pad_mu, restitution=0.0)
    b.root["config"] = {"dt": dt, "integrator": integrator}
    return b.scene()


def closed_chain(n_cells=22, link=0.2, mass=0.1) -> SceneDescription:
    """Config 4: a hanging ladder of parallelogram cells (3D revolute joints
    about y).  Rails are split into one segment per cell; each cell adds two
    rail segments and one rung (3 bodies) and four joints, one loop per cell.
    Rows = 5 * joints = 20 * n_cells: n_cells=12 -> 240 rows, 14 -> 280
    (dense HBM-slab kernel under Auto), 22 -> 88 joints -> 440 rows
    (> 300 -> matrix-free CR path under Auto)."""
    b = _Builder("closed_chain", gravity=(0.0, 0.0, -9.81))
    w = link  # rung width
    prev_l = prev_r = "world"
    for k in range(n_cells):
        zt = -k * link
        zb = zt - link
        l, r, rung = f"rail_l{k}", f"rail_r{k}", f"rung{k}"
        b.body(l, mass, (0.01, 0.01, link), [0.0, 0.0, (zt + zb) / 2])
        b.body(r, mass, (0.01, 0.01, link), [w, 0.0, (zt + zb) / 2])
        b.joint(f"jl{k}", prev_l, l, [0.0, 0.0, zt], Y)
        b.joint(f"jr{k}", prev_r, r, [w, 0.0, zt], Y)
        if k == 0:
            pass
        b.body(rung, mass, (w, 0.01, 0.01), [w / 2, 0.0, zb])
        b.joint(f"jrl{k}", l, rung, [0.0, 0.0, zb], Y)
        b.joint(f"jrr{k}", r, rung, [w, 0.0, zb], Y)
        prev_l, prev_r = l, r
    # give the ladder a push so it swings
    b.root["bodies"][-1]["linear_velocity"] = [0.5, 0.0, 0.0]
    return b.scene()


def stewart_tower(stages=12, radius_base=0.3, radius_top=0.25, height=0.4, kp=3000.0, kd=60.0, damping=5.0,
                  platform_mass=1.0, leg_mass=0.1) -> SceneDescription:
    """Config 4 ("a multi-leg parallel manipulator with spherical
    joints", n ~ 1000, ~150 bodies): `stages` 6-6 Stewart platforms stacked on
    the ground.  Every leg is two bodies (cylinder, piston) joined by a
    prismatic joint along the leg (PD-held at its build length, plus a damping
    row), with spherical joints to the platform below (or the world) and the
    platform above.  Bottom-stage legs have a [-0.0005, 0.05] m stroke limit,
    so their lower limit sits inside the 0.001 m margin from the start.  Per
    stage: 13 bodies, 18 joints, 6 x (3 + 5 + 3) + 12 = 78 rows."""
    b = _Builder("stewart_tower")
    lower = "world"
    zl = 0.0
    for k in range(stages):
        zu = zl + height
        plat = f"plat{k}"
        b.body(plat, platform_mass, (2 * radius_top, 2 * radius_top, 0.04), [0.0, 0.0, zu])
        for i in range(6):
            a = math.radians(60.0 * i)
            t = math.radians(60.0 * i + (30.0 if i % 2 == 0 else -30.0))
            B = [radius_base * math.cos(a), radius_base * math.sin(a), zl]
            T = [radius_top * math.cos(t), radius_top * math.sin(t), zu]
            d = _sub(T, B)
            length = math.sqrt(sum(x * x for x in d))
            u = [x / length for x in d]
            M = [B[q] + 0.5 * d[q] for q in range(3)]
            cyl, pis = f"leg{k}_{i}_cyl", f"leg{k}_{i}_pis"
            b.body(cyl, leg_mass, (0.03, 0.03, 0.5 * length), [B[q] + 0.25 * d[q] for q in range(3)])
            b.body(pis, leg_mass, (0.02, 0.02, 0.5 * length), [B[q] + 0.75 * d[q] for q in range(3)])
            b.joint(f"s{k}_{i}_lo", lower, cyl, B, X, type="spherical")
            kw = dict(type="prismatic", kp=kp, kd=kd, damping=damping)
            if k == 0:
                kw["limits"] = [-0.0005, 0.05]
            b.joint(f"p{k}_{i}", cyl, pis, M, u, **kw)
            b.joint(f"s{k}_{i}_hi", pis, plat, T, X, type="spherical")
        lower, zl = plat, zu
    # a slow twist of the top platform sets the tower moving
    b.root["bodies"][-13]["angular_velocity"] = [0.0, 0.0, 0.2]
    return b.scene()


def mixed_joints() -> SceneDescription:
    """Every joint type and joint-dynamics row in one world (constraints.cpp:
    90-108 fixed / prismatic / spherical rows, 160-187 coordinate-rate rows,
    256-274 PD / armature / damping, 218-229 limits with the linear margin).

    carriage --prismatic x (PD to 0.02, limits +-0.1)--> world
    cap      --fixed--> carriage
    arm1     --spherical--> carriage          (swinging in 3D)
    arm2     --revolute y (armature 0.05, damping 0.1, limits)--> arm1
    plunger  --prismatic along arm2 (armature 0.2, damping 0.5, limits [-0.0005, 0.05])--> arm2
    slider   --prismatic y (limits [-0.0008, 0.05], pushed into its lower limit)--> world
    """
    b = _Builder("mixed_joints")
    b.body("carriage", 1.0, (0.2, 0.1, 0.05), [0.0, 0.0, 1.0])
    b.joint("slide_x", "world", "carriage", [0.0, 0.0, 1.0], X, type="prismatic", kp=20.0, kd=1.0, target=0.02,
            limits=[-0.1, 0.1])
    b.body("cap", 0.3, (0.05, 0.05, 0.05), [0.0, 0.0, 1.05])
    b.joint("weld", "carriage", "cap", [0.0, 0.0, 1.03], X, type="fixed")
    b.body("arm1", 0.5, (0.03, 0.03, 0.4), [0.0, 0.0, 0.8])
    b.joint("ball", "carriage", "arm1", [0.0, 0.0, 1.0], X, type="spherical")
    b.body("arm2", 0.4, (0.03, 0.03, 0.3), [0.0, 0.0, 0.45])
    b.joint("elbow", "arm1", "arm2", [0.0, 0.0, 0.6], Y, armature=0.05, damping=0.1, limits=[-1.0, 1.0])
    b.body("plunger", 0.2, (0.02, 0.02, 0.1), [0.0, 0.0, 0.25])
    b.joint("plunge", "arm2", "plunger", [0.0, 0.0, 0.3], Z, type="prismatic", armature=0.2, damping=0.5,
            limits=[-0.0005, 0.05])
    b.body("slider", 0.5, (0.1, 0.1, 0.1), [0.5, 0.0, 0.5])
    b.joint("slide_y", "world", "slider", [0.5, 0.0, 0.5], Y, type="prismatic", limits=[-0.0008, 0.05])
    b.root["bodies"][2]["angular_velocity"] = [1.0, 0.5, 0.0]   # arm1
    b.root["bodies"][5]["linear_velocity"] = [0.0, -0.1, 0.0]   # slider into its lower limit
    return b.scene()


def sphere_pile(n_spheres=100, radius=0.05, mu=0.5, seed=7) -> SceneDescription:
    """Config 5 substitute: spheres in a bin of five world
    planes (floor + 4 walls).  Sphere-sphere and sphere-plane pairs are the
    supported shapes; a literal box pile is inexpressible in the reference."""
    import random
    rng = random.Random(seed)
    b = _Builder("sphere_pile")
    side = int(math.ceil(math.sqrt(n_spheres / 4.0)))
    half = side * radius * 1.05
    k = 0
    layer = 0
    while k < n_spheres:
        for i in range(side):
            for j in range(side):
                if k >= n_spheres:
                    break
                x = -half + radius + i * 2.1 * radius + rng.uniform(-1e-3, 1e-3)
                y = -half + radius + j * 2.1 * radius + rng.uniform(-1e-3, 1e-3)
                z = radius + layer * 2.05 * radius
                name = f"s{k}"
                m = 0.1
                b.pos[name] = [x, y, z]
                i0 = 0.4 * m * radius * radius
                b.root["bodies"].append({"name": name, "mass": m, "inertia": [i0, i0, i0],
                                         "position": [x, y, z], "orientation": [1.0, 0.0, 0.0, 0.0]})
                b.geom(body=name, shape="sphere", radius=radius, mu=mu, restitution=0.0)
                k += 1
        layer += 1
    walls = (([0.0, 0.0, 1.0], 0.0), ([1.0, 0.0, 0.0], -half - 2 * radius), ([-1.0, 0.0, 0.0], -half - 2 * radius),
             ([0.0, 1.0, 0.0], -half - 2 * radius), ([0.0, -1.0, 0.0], -half - 2 * radius))
    for nrm, off in walls:
        b.geom(body="world", shape="plane", normal=nrm, offset=off, mu=mu, restitution=0.0)
    return b.scene()


def box_pile(n_boxes=64, half=0.05, mu=0.5, seed=11, gap=0.02) -> SceneDescription:
    """Config 5 as written (BASELINE.json configs[4]): a pile of boxes in a bin
    of five world planes (`gap` between neighbours in a layer).  Needs the opt-in box-box extension
    (KD_EXT_BOX_BOX; the reference rejects box-box pairs, model.cpp:56-62, so
    this scene has no reference counterpart and its parity is against the
    oracle's restatement of the same narrow phase).  Layers of side x side
    boxes, 0.02 apart horizontally (beyond the 0.01 contact margin), each layer
    dropped 0.004 above the one below with a small deterministic yaw."""
    import random
    rng = random.Random(seed)
    b = _Builder("box_pile")
    side = int(math.ceil(math.sqrt(n_boxes / 4.0)))
    pitch = 2.0 * half + gap
    extent = side * pitch / 2.0
    m = 0.1
    k = 0
    layer = 0
    while k < n_boxes:
        for i in range(side):
            for j in range(side):
                if k >= n_boxes:
                    break
                x = -extent + pitch / 2 + i * pitch + rng.uniform(-1e-3, 1e-3)
                y = -extent + pitch / 2 + j * pitch + rng.uniform(-1e-3, 1e-3)
                z = half + layer * (2.0 * half + 0.004)
                yaw = rng.uniform(-0.05, 0.05) if gap > 0 else 0.0
                name = f"b{k}"
                b.pos[name] = [x, y, z]
                b.root["bodies"].append({"name": name, "mass": m, "inertia": _box_inertia(m, 2 * half, 2 * half, 2 * half),
                                         "position": [x, y, z],
                                         "orientation": [math.cos(yaw / 2), 0.0, 0.0, math.sin(yaw / 2)]})
                b.geom(body=name, shape="box", half_extents=[half, half, half], mu=mu, restitution=0.0)
                k += 1
        layer += 1
    wall = extent + 0.01
    walls = (([0.0, 0.0, 1.0], 0.0), ([1.0, 0.0, 0.0], -wall), ([-1.0, 0.0, 0.0], -wall),
             ([0.0, 1.0, 0.0], -wall), ([0.0, -1.0, 0.0], -wall))
    for nrm, off in walls:
        b.geom(body="world", shape="plane", normal=nrm, offset=off, mu=mu, restitution=0.0)
    b.root["extensions"] = ["box_box"]
    return b.scene()
