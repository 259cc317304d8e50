"""paper_2407_14783_b200 -- B200-native (sm_100a) hot path of the VisFly /
quadsim batched quadrotor simulator.

The Python surface mirrors the reference package `quadsim` (make_env /
reset / step, dynamics.step, control.command_to_rotor_speeds,
sensing.render_frames, gradients.rollout_grad); the work runs in
libquadb200.so (include/quadb200.h): K1 fused controller+dynamics (+adjoint),
K2 warp-packet BVH ray caster, K3 fused proximity/reward/termination/reset.
There is no CPU fallback.
"""

from .control import CTBR, LV, PS, SRT, Command, RotorSpeeds, command_to_rotor_speeds
from .dynamics import QuadState, step
from .params import ControllerGains, Integrator, QuadParams, SimConfig, load_params

__version__ = "0.1.0"

__all__ = [
    "CTBR", "Command", "ControllerGains", "Integrator", "LV", "PS", "QuadParams", "QuadState", "RotorSpeeds", "SRT",
    "SimConfig", "command_to_rotor_speeds", "load_params", "step",
]
