"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the N-BVH method (no slab test, no hash, no
encoding, no MLP, no decode).  It only produces data: meshes, rays, random
parameter values and random draws that the method consumes as inputs
(DESIGN.md "Input recipe").
"""
from .scenes import (  # noqa: F401
    Scene, icosphere, scene_tiny, scene_1080p, scene_1080p_parts, camera_rays, random_rays,
    random_params_fp16, random_mlp, random_uniform, CONFIGS, HashCfg,
)
