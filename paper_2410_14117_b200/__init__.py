"""paper_2410_14117_b200 -- B200-native batched underwater-vehicle env step.

Drop-in for the reference's batched hot path (uuvsim ``batch_create`` /
``EnvBatch.step`` and the ``uuvsim_*`` C ABI v1): thruster allocation,
sub-stepped Fossen 6-DOF dynamics, reward/termination, counter-RNG auto-reset
and domain randomisation, fused into one sm_100a CUDA kernel per step.
"""

from ._core import NativeError
from .batch import (STAT_NAMES, B200EnvBatch, batch_create, bench_actions, bench_throughput,
                    resolve_backend)
from .config import (CIRCLE, HELIX, LEMNISCATE, STATION_KEEPING, ConfigError, ParamsError,
                     RandomizationRanges, TaskSpec, VehicleParams, bluerov2_params,
                     default_params, default_ranges, engine_config_dict, engine_config_json,
                     load_params, save_params, wrap_angle)

__version__ = "0.1.0"

__all__ = [
    "B200EnvBatch", "CIRCLE", "ConfigError", "HELIX", "LEMNISCATE", "NativeError", "ParamsError",
    "RandomizationRanges", "STATION_KEEPING", "STAT_NAMES", "TaskSpec", "VehicleParams",
    "batch_create", "bench_actions", "bench_throughput", "bluerov2_params", "default_params",
    "default_ranges", "engine_config_dict", "engine_config_json", "load_params",
    "resolve_backend", "save_params", "wrap_angle",
]
