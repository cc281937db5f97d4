"""Drop the B200 path into the reference package.

The reference resolves its two hot-path operators by module-attribute lookup at
call time -- `rerouting.apply_sere(...)` at moe.py:368 and the module-global
`layer_forward(...)` at moe.py:375 -- so replacing those two attributes moves
every caller (model_forward, the CLI `reroute` command cli.py:224/245, the
simulator's decode loop simulator.py:188/394-415, the bound audit bounds.py:281)
onto the GPU without touching reference code:

    import sere.rerouting, sere.moe
    from paper_2602_07616_b200 import integration
    handle = integration.install(sere.rerouting, sere.moe)
    ...                                   # reference code now runs on the B200 kernels
    handle.uninstall()

Results come back as the reference's own `RerouteResult` class when the patched
module defines one, so `isinstance` checks and dataclass equality keep working.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any

import numpy as np

from . import moe as _moe
from . import rerouting as _rr


def _adapt_result(res: _rr.RerouteResult, cls: Any):
    if cls is None or cls is _rr.RerouteResult:
        return res
    return cls(new_indices=res.new_indices, primary_set=res.primary_set,
               preserved_critical=res.preserved_critical, final_active=res.final_active,
               reroute_map=res.reroute_map)


@dataclass
class Installed:
    rerouting_module: Any
    moe_module: Any
    saved: dict

    def uninstall(self) -> None:
        for (mod, name), fn in self.saved.items():
            setattr(mod, name, fn)
        self.saved.clear()


def install(rerouting_module: Any, moe_module: Any | None = None) -> Installed:
    """Point `rerouting_module.apply_sere` (rerouting.py:130) and, if given,
    `moe_module.layer_forward` (moe.py:280) at the GPU implementations.

    The device path has size limits the reference does not (T*K <= 16384 cells, M <= 256
    routed and <= 31 shared experts, `moe.device_supports`); a call beyond them runs the
    saved reference function instead, so every caller keeps working. The installed
    wrappers resolve this package's implementations at call time."""
    result_cls = getattr(rerouting_module, "RerouteResult", None)
    ref_apply_sere = rerouting_module.apply_sere
    saved = {(rerouting_module, "apply_sere"): ref_apply_sere}

    def apply_sere(assignment, sim, config):
        shape = np.shape(getattr(assignment, "indices", assignment))
        m = np.shape(getattr(sim, "values", sim))
        if len(shape) != 2 or len(m) != 2 or not _rr.device_supports(shape[0], shape[1], m[0]):
            return ref_apply_sere(assignment, sim, config)  # the reference's limits / its own errors
        return _adapt_result(_rr.apply_sere(assignment, sim, config), result_cls)

    apply_sere.__doc__ = _rr.apply_sere.__doc__
    rerouting_module.apply_sere = apply_sere
    if moe_module is not None:
        ref_layer_forward = moe_module.layer_forward
        saved[(moe_module, "layer_forward")] = ref_layer_forward

        def layer_forward(layer, x, assignment, activation="silu"):
            idx = getattr(assignment, "indices", None)
            shape = getattr(idx, "shape", ())
            ok = len(shape) == 2 and _moe.device_supports(int(shape[0]), int(shape[1]), len(layer.experts),
                                                          len(getattr(layer, "shared_experts", ())))
            if not ok:
                return ref_layer_forward(layer, x, assignment, activation)
            return _moe.layer_forward(layer, x, assignment, activation)

        layer_forward.__doc__ = _moe.layer_forward.__doc__
        moe_module.layer_forward = layer_forward
    return Installed(rerouting_module, moe_module, saved)


__all__ = ["install", "Installed"]
