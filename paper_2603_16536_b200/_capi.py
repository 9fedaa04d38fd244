"""ctypes mirror of include/kamino_b200.h (the C-ABI drop-in boundary).

The struct layouts here must match the header byte for byte; tests/test_capi.py
checks sizes against the compiled library's exported symbols.  `bind()` declares
argument/return types for every entry point of a library that exports the kd_*
surface (or any prefix that mirrors it)."""
import ctypes as C

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)
c_uint8_p = C.POINTER(C.c_uint8)

# status codes (kamino_b200.h)
KD_OK = 0
MODEL_ERROR_CODES = {
    1: "InvalidReference",
    2: "NonUnitAxis",
    3: "BadInertia",
    4: "BadLimits",
    5: "UnsupportedOnJointType",
    6: "BadGeometry",
    7: "UnsupportedCollisionPair",
    8: "WrongJointType",
    9: "DuplicateName",
}
KD_ERR_INVALID_ARGUMENT = 20
KD_ERR_CUDA = 21
KD_ERR_SPD_FAILURE = 22
KD_ERR_CAPACITY = 23
KD_ERR_NO_DEVICE = 24

KD_INTEGRATOR_SEMI_IMPLICIT_EULER = 0
KD_INTEGRATOR_MOREAU_JEAN = 1
KD_BACKEND_DENSE = 0
KD_BACKEND_MATRIX_FREE = 1
KD_BACKEND_AUTO = 2
KD_KERNEL_NONE, KD_KERNEL_DENSE, KD_KERNEL_SUPERNODAL, KD_KERNEL_CR, KD_KERNEL_SUPERNODAL_DENSE = 0, 1, 2, 3, 4
KD_KERNEL_SUPERNODAL_CLUSTER = 5
KERNEL_NAMES = {0: 'none', 1: 'dense', 2: 'supernodal', 3: 'cr', 4: 'supernodal+dense', 5: 'supernodal+cluster'}
CR_PATH_NAMES = {0: 'none', 1: 'incidence', 2: 'rows', 3: 'shared'}


class kd_body_desc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("mass", C.c_double),
        ("inertia", C.c_double * 9),
        ("position", C.c_double * 3),
        ("orientation", C.c_double * 4),
        ("linear_velocity", C.c_double * 3),
        ("angular_velocity", C.c_double * 3),
    ]


class kd_joint_desc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("type", C.c_char_p),
        ("parent", C.c_char_p),
        ("child", C.c_char_p),
        ("parent_position", C.c_double * 3),
        ("parent_orientation", C.c_double * 4),
        ("child_position", C.c_double * 3),
        ("child_orientation", C.c_double * 4),
        ("axis", C.c_double * 3),
        ("has_limits", C.c_int32),
        ("lower", C.c_double),
        ("upper", C.c_double),
        ("kp", C.c_double),
        ("kd", C.c_double),
        ("has_target", C.c_int32),
        ("target", C.c_double),
        ("target_rate", C.c_double),
        ("armature", C.c_double),
        ("damping", C.c_double),
    ]


class kd_geom_desc(C.Structure):
    _fields_ = [
        ("body", C.c_char_p),
        ("shape", C.c_char_p),
        ("radius", C.c_double),
        ("half_extents", C.c_double * 3),
        ("normal", C.c_double * 3),
        ("offset", C.c_double),
        ("mu", C.c_double),
        ("restitution", C.c_double),
    ]


class kd_scene_desc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("gravity", C.c_double * 3),
        ("n_bodies", C.c_int32),
        ("bodies", C.POINTER(kd_body_desc)),
        ("n_joints", C.c_int32),
        ("joints", C.POINTER(kd_joint_desc)),
        ("n_geoms", C.c_int32),
        ("geoms", C.POINTER(kd_geom_desc)),
    ]


class kd_step_config(C.Structure):
    _fields_ = [
        ("dt", C.c_double),
        ("integrator", C.c_int32),
        ("backend", C.c_int32),
        ("eta", C.c_double),
        ("rho", C.c_double),
        ("eps", C.c_double),
        ("max_iters", C.c_int32),
        ("acceleration", C.c_int32),
        ("restart", C.c_int32),
        ("fixed_iteration_mode", C.c_int32),
        ("cr_iters", C.c_int32),
        ("baumgarte_beta", C.c_double),
        ("contact_margin", C.c_double),
        ("impact_velocity_threshold", C.c_double),
        ("bias_clamp", C.c_double),
        ("limit_margin_angular", C.c_double),
        ("limit_margin_linear", C.c_double),
        ("warm_start", C.c_int32),
    ]


class kd_step_diag(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("restarts", C.c_int32),
        ("converged", C.c_int32),
        ("cr_breakdown", C.c_int32),
        ("cr_iterations", C.c_int64),
        ("r_p", C.c_double),
        ("r_d", C.c_double),
        ("r_c", C.c_double),
        ("n_rows", C.c_int32),
        ("contact_count", C.c_int32),
        ("first_contact_row", C.c_int32),
        ("n_limits", C.c_int32),
        ("f_inf", C.c_double),
        ("kkt_momentum_inf", C.c_double),
        ("bilateral_velocity_inf", C.c_double),
    ]


class kd_model_info(C.Structure):
    _fields_ = [
        ("n_bodies", C.c_int32),
        ("n_joints", C.c_int32),
        ("n_geoms", C.c_int32),
        ("n_bilateral_rows", C.c_int32),
        ("n_dynamics_rows", C.c_int32),
        ("n_loops", C.c_int32),
        ("n_limited_joints", C.c_int32),
        ("max_contacts", C.c_int32),
        ("row_capacity", C.c_int32),
    ]


class kd_row_dump(C.Structure):
    _fields_ = [
        ("body_a", C.c_int32),
        ("body_b", C.c_int32),
        ("kind", C.c_int32),
        ("pad", C.c_int32),
        ("block_a", C.c_double * 6),
        ("block_b", C.c_double * 6),
        ("bias", C.c_double),
        ("reg", C.c_double),
        ("scale", C.c_double),
        ("vf_scaled", C.c_double),
        ("lambda_", C.c_double),
        ("z", C.c_double),
    ]


# name -> (restype, argtypes); the handle type is an opaque void*.
class kd_limit_cache_entry(C.Structure):
    _fields_ = [("joint", C.c_int32), ("bound", C.c_int32), ("lambda_", C.c_double), ("z", C.c_double)]


class kd_contact_cache_entry(C.Structure):
    _fields_ = [("geom_a", C.c_int32), ("geom_b", C.c_int32), ("position", C.c_double * 3),
                ("impulse", C.c_double * 3), ("dual", C.c_double * 3)]


class kd_solve_problem(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("n_bodies", C.c_int32), ("n_bilateral", C.c_int32),
                ("n_limits", C.c_int32), ("n_contacts", C.c_int32), ("pad", C.c_int32),
                ("body", C.POINTER(C.c_int32)), ("jacobian", C.POINTER(C.c_double)), ("reg", C.POINTER(C.c_double)),
                ("scale", C.POINTER(C.c_double)), ("mu", C.POINTER(C.c_double)),
                ("inv_mass", C.POINTER(C.c_double)), ("inv_inertia", C.POINTER(C.c_double)),
                ("rhs", C.POINTER(C.c_double)), ("x0", C.POINTER(C.c_double)), ("z0", C.POINTER(C.c_double))]


_H = C.c_void_p
SIGNATURES = {
    "model_build": (C.c_int, [C.POINTER(kd_scene_desc), C.POINTER(C.c_void_p)]),
    "model_build_ex": (C.c_int, [C.POINTER(kd_scene_desc), C.c_uint32, C.POINTER(C.c_void_p)]),
    "model_destroy": (None, [_H]),
    "model_get_info": (C.c_int, [_H, C.POINTER(kd_model_info)]),
    "model_joint_layout": (C.c_int, [_H, c_int32_p, c_int32_p, c_int32_p, c_int32_p]),
    "model_joint_targets": (C.c_int, [_H, c_double_p]),
    "joint_coordinate": (C.c_int, [_H, C.c_int32, c_double_p, c_double_p]),
    "batch_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, c_int32_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "batch_destroy": (None, [_H]),
    "batch_size": (C.c_int, [_H, c_int32_p, c_int64_p, c_int64_p]),
    "batch_offsets": (C.c_int, [_H, c_int32_p, c_int32_p]),
    "batch_set_state": (C.c_int, [_H, c_double_p, c_double_p, c_double_p]),
    "batch_get_state": (C.c_int, [_H, c_double_p, c_double_p, c_double_p]),
    "batch_reset_caches": (C.c_int, [_H]),
    "batch_set_active": (C.c_int, [_H, c_uint8_p]),
    "batch_get_diagnostics": (C.c_int, [_H, C.POINTER(kd_step_diag)]),
    "batch_row_offsets": (C.c_int, [_H, c_int64_p, c_int64_p]),
    "batch_get_impulses": (C.c_int, [_H, c_double_p]),
    "batch_dump_rows": (C.c_int, [_H, C.c_int32, C.POINTER(kd_row_dump), C.c_int32, c_int32_p]),
    "batch_dump_contacts": (C.c_int, [_H, C.c_int32, c_int32_p, c_double_p, C.c_int32, c_int32_p]),
    "batch_dump_limits": (C.c_int, [_H, C.c_int32, c_int32_p, C.c_int32, c_int32_p]),
    "step_config_default": (None, [C.POINTER(kd_step_config)]),
    "last_error": (C.c_char_p, []),
}
# product-only entry points
KD_ONLY = {
    "batch_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p), C.c_int32, c_int32_p, C.c_int32,
                               C.POINTER(C.c_void_p)]),
    "batch_step": (C.c_int, [_H, C.POINTER(kd_step_config), C.c_int32]),
    "batch_set_history_capacity": (C.c_int, [_H, C.c_int32]),
    "batch_get_history": (C.c_int, [_H, c_double_p]),
    "bench_jitter": (C.c_int, [C.c_uint64, C.c_double, C.c_int32, c_int32_p, c_double_p]),
    "batch_enable_timing": (C.c_int, [_H, C.c_int32]),
    "batch_get_timing": (C.c_int, [_H, c_double_p, c_int64_p]),
    "version": (C.c_char_p, []),
    "batch_get_phase_cycles": (C.c_int, [_H, c_int64_p]),
    "batch_get_cr_paths": (C.c_int, [_H, c_int32_p]),
    "batch_step_async": (C.c_int, [_H, C.POINTER(kd_step_config), C.c_int32]),
    "batch_sync": (C.c_int, [_H]),
    "batch_stream": (C.c_int, [_H, C.POINTER(C.c_void_p)]),
    "batch_set_state_async": (C.c_int, [_H, c_double_p, c_double_p]),
    "batch_get_state_async": (C.c_int, [_H, c_double_p, c_double_p]),
    "abi_sizes": (C.c_int, [c_int32_p, C.c_int32]),
    "batch_get_kernels": (C.c_int, [_H, c_int32_p]),
    "batch_fk": (C.c_int, [_H, c_int32_p, c_double_p, C.c_int32, C.c_double, C.c_int32, C.c_double, c_int32_p,
                           c_double_p, c_uint8_p]),
    "batch_device_state": (C.c_int, [_H, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "model_sparse_plan_info": (C.c_int, [_H, c_int64_p]),
    "model_sparse_plan_selftest": (C.c_int, [_H, C.c_uint64, c_double_p]),
    "model_set_contact_capacity": (C.c_int, [_H, C.c_int32]),
    "padmm_solve_batched": (C.c_int, [C.c_int32, C.POINTER(kd_solve_problem), C.c_int32, C.c_double, C.c_int32,
                                      C.c_int32, C.POINTER(kd_step_config), c_double_p, c_double_p,
                                      C.POINTER(kd_step_diag), c_double_p, C.c_int32]),
    "cr_solve_batched": (C.c_int, [C.c_int32, C.POINTER(kd_solve_problem), C.c_int32, C.c_double, C.c_int32,
                                   c_double_p, c_int32_p, c_uint8_p, c_double_p, c_double_p, C.c_int32]),
    "batch_assemble": (C.c_int, [_H, C.POINTER(kd_step_config)]),
    "batch_get_cache_sizes": (C.c_int, [_H, C.c_int32, c_int32_p, c_int32_p, c_int32_p, c_int32_p]),
    "batch_get_caches": (C.c_int, [_H, C.c_int32, c_double_p, c_double_p, c_int32_p,
                                   C.POINTER(kd_limit_cache_entry), C.c_int32, c_int32_p,
                                   C.POINTER(kd_contact_cache_entry), C.c_int32, c_int32_p]),
    "batch_set_caches": (C.c_int, [_H, C.c_int32, c_double_p, c_double_p, C.c_int32, C.c_int32,
                                   C.POINTER(kd_limit_cache_entry), C.c_int32,
                                   C.POINTER(kd_contact_cache_entry), C.c_int32]),
}


def bind(lib, prefix, extra=None):
    """Declare restype/argtypes for `prefix + name` symbols present in `lib`."""
    table = dict(SIGNATURES)
    if extra:
        table.update(extra)
    for name, (res, args) in table.items():
        fn = getattr(lib, prefix + name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    return lib


def dptr(arr):
    """numpy float64 array -> double* (None passes NULL)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(c_double_p)


def i32ptr(arr):
    return arr.ctypes.data_as(c_int32_p)


def i64ptr(arr):
    return arr.ctypes.data_as(c_int64_p)
