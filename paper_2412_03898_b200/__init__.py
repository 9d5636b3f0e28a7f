"""B200-native hot path of 4D SlingBAG (arXiv 2412.03898).

Drop-in replacements for the reference ``pacloud`` hot-path calls, backed by
hand-written sm_100a CUDA kernels behind a C ABI (libpacloud_b200.so,
include/pacloud_b200.h):

    deformation.cloud_states_at / cloud_state_grads / ball_state_at /
        ball_state_grad / eval_basis / eval_H
    radiator.forward_frame / frame_state_grads / accumulate_frame_grads /
        pressure_kernel / pressure_kernel_grad
    reconstruction.l2_loss / adam_step / sgd_step / ParamGroup(s) /
        dynamic_reconstruct
    engine.IterationEngine      fused multi-frame iteration (+ NCCL sharding)
    geometry.simulate_dataset / build_phantom / spherical_array (target
        synthesis on the forward kernel)
    evaluation.voxelize / map_project / ssim / eval_report
    static.static_reconstruct   single-frame stage (lattice init, prune)
    fileio.read/write_tensor (PAT1), read/write_cloud (GGB1)
    ubp.ubp_reconstruct         universal back-projection comparator
"""

from .core import (AdamState, BallStateAtT, Box, CloudGrads, CloudState,
                   GaussBall, DeformField, Violation, validate_cloud,
                   CloudStateGrad, DynamicCloud, ReconConfig, SensorArray,
                   SignalSet, VoxelGrid, default_basis_grid, frame_times)
from .deformation import (BallStateGrad, ball_state_at, ball_state_grad,
                          cloud_state_grads, cloud_states_at, eval_basis,
                          eval_H)
from .engine import IterationEngine
from .evaluation import (GridSpec, eval_report, format_report, map_project,
                         ssim, voxelize)
from .fileio import read_cloud, read_tensor, write_cloud, write_tensor
from .geometry import (Phantom, PhantomSpec, build_phantom, fibonacci_sphere,
                       simulate_dataset, spherical_array)
from .radiator import (accumulate_frame_grads, compute_time_window,
                       forward_frame, frame_state_grads, pressure_kernel,
                       pressure_kernel_grad)
from .reconstruction import (ParamGroup, ParamGroups, adam_step,
                             dynamic_reconstruct, l2_loss, scheduled_lr,
                             sgd_step)
from .static import static_reconstruct
from .ubp import ubp_reconstruct

__version__ = "0.1.0"

__all__ = [
    "AdamState", "BallStateAtT", "CloudGrads", "CloudState", "CloudStateGrad",
    "DynamicCloud", "ReconConfig", "SensorArray", "SignalSet",
    "default_basis_grid", "frame_times", "cloud_state_grads",
    "cloud_states_at", "IterationEngine", "accumulate_frame_grads",
    "forward_frame", "frame_state_grads", "ParamGroup", "ParamGroups",
    "adam_step", "dynamic_reconstruct", "l2_loss", "scheduled_lr", "sgd_step",
    "Box", "VoxelGrid", "GridSpec", "eval_report", "format_report",
    "map_project", "ssim", "voxelize", "Phantom", "PhantomSpec",
    "build_phantom", "fibonacci_sphere", "simulate_dataset", "spherical_array",
    "read_cloud", "read_tensor", "write_cloud", "write_tensor",
    "static_reconstruct", "GaussBall", "ubp_reconstruct",
    "DeformField", "Violation", "validate_cloud", "BallStateGrad",
    "ball_state_at", "ball_state_grad", "eval_basis", "eval_H",
    "compute_time_window", "pressure_kernel", "pressure_kernel_grad",
]
