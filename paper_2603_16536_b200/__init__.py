"""B200-native per-step PADMM forward-dynamics solve (Kamino hot path).

The product is libkamino_b200.so (sm_100a kernels + C-ABI, include/kamino_b200.h);
this package is the host-side mirror of the reference loopdyn API over it.
"""
from .scene import (ModelError, SceneConfig, SceneDescription, SceneError, StepConfig, apply_scene_config,
                    config_for, load_scene_file, parse_scene, parse_scene_obj, serialize_scene)
from .loopdyn import (LIB_PATH, JointReactionCache, KaminoError, Model, ReactionCacheEntry, WorldBatch, WorldState,
                      batch_step, bench_jitter, build_model, cr_solve, lib, padmm_solve, step,
                      SolveProblem)

__all__ = [
    "ModelError", "SceneConfig", "SceneDescription", "SceneError", "StepConfig", "apply_scene_config",
    "config_for", "load_scene_file", "parse_scene", "parse_scene_obj", "serialize_scene", "LIB_PATH",
    "KaminoError", "Model", "WorldBatch", "WorldState", "batch_step", "bench_jitter", "build_model", "lib",
    "step", "JointReactionCache", "ReactionCacheEntry", "padmm_solve", "cr_solve", "SolveProblem",
]
