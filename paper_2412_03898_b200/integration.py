"""Route the reference `pacloud` package's hot-path calls to this library.

The reference binds its hot-path names at module import time
(reconstruction.py:18-21, geometry.py:16-17, cli.py:18-25), so replacing
`pacloud.radiator.forward_frame` alone would not reach its callers: every
importing module is patched.  `enable()` is what a maintainer adds to the
reference; `disable()` restores the reference's
own functions.

Two levels:

* ``level="calls"`` — the per-call drop-ins only (deformation, forward,
  adjoint, chain rule, loss, Adam/SGD).  The reference's own Python frame
  loop (reconstruction.py:293-332) then drives the CUDA kernels one frame at
  a time.
* ``level="stages"`` (default) — additionally the whole stages:
  `dynamic_reconstruct` (the fused IterationEngine, one host sync per
  iteration), `static_reconstruct`, `ubp_reconstruct`, `simulate_dataset`,
  `build_phantom`, `voxelize`.
"""

from __future__ import annotations

import importlib

# (reference module, attribute) -> name in this package
_CALLS = {
    "deformation": ("cloud_states_at", "cloud_state_grads", "ball_state_at",
                    "ball_state_grad", "eval_basis", "eval_H"),
    "radiator": ("forward_frame", "frame_state_grads",
                 "accumulate_frame_grads", "pressure_kernel",
                 "pressure_kernel_grad"),
    "reconstruction": ("cloud_states_at", "cloud_state_grads",
                       "forward_frame", "frame_state_grads",
                       "accumulate_frame_grads", "l2_loss",
                       "adam_step", "sgd_step"),
    "geometry": ("forward_frame",),
    "cli": ("cloud_states_at",),
}
_STAGES = {
    "reconstruction": ("dynamic_reconstruct", "static_reconstruct",
                       "ubp_reconstruct"),
    "geometry": ("simulate_dataset", "build_phantom", "voxelize"),
    "evaluation": ("voxelize",),
    "cli": ("dynamic_reconstruct", "static_reconstruct", "ubp_reconstruct",
            "simulate_dataset", "build_phantom"),
}

_saved: dict = {}


def _targets(level: str):
    if level not in ("calls", "stages"):
        raise ValueError("level must be 'calls' or 'stages'")
    out = [(m, n) for m, names in _CALLS.items() for n in names]
    if level == "stages":
        out += [(m, n) for m, names in _STAGES.items() for n in names]
    return out


def enable(level: str = "stages", package: str = "pacloud") -> list:
    """Patch `package`'s modules (and the package namespace) to call this
    library.  Returns the list of patched "module.name" strings."""
    import paper_2412_03898_b200 as b200
    disable(package)
    root = importlib.import_module(package)
    done = []
    for mod_name, name in _targets(level):
        try:
            mod = importlib.import_module(f"{package}.{mod_name}")
        except ImportError:
            continue
        if not hasattr(mod, name):
            continue
        _saved[(package, mod_name, name)] = getattr(mod, name)
        setattr(mod, name, getattr(b200, name))
        done.append(f"{mod_name}.{name}")
    # the package namespace re-exports the same names (pacloud/__init__.py)
    for _, name in _targets(level):
        if hasattr(root, name) and (package, "", name) not in _saved:
            _saved[(package, "", name)] = getattr(root, name)
            setattr(root, name, getattr(b200, name))
    return done


def disable(package: str = "pacloud") -> None:
    """Restore every name `enable()` replaced."""
    for (pkg, mod_name, name), fn in list(_saved.items()):
        if pkg != package:
            continue
        mod = importlib.import_module(f"{pkg}.{mod_name}" if mod_name else pkg)
        setattr(mod, name, fn)
        del _saved[(pkg, mod_name, name)]
