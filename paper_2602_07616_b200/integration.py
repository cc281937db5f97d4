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
    `moe_module.layer_forward` (moe.py:280) at the GPU implementations."""
    result_cls = getattr(rerouting_module, "RerouteResult", None)

    def apply_sere(assignment, sim, config):
        return _adapt_result(_rr.apply_sere(assignment, sim, config), result_cls)

    apply_sere.__doc__ = _rr.apply_sere.__doc__
    saved = {(rerouting_module, "apply_sere"): rerouting_module.apply_sere}
    rerouting_module.apply_sere = apply_sere
    if moe_module is not None:
        saved[(moe_module, "layer_forward")] = moe_module.layer_forward
        moe_module.layer_forward = _moe.layer_forward
    return Installed(rerouting_module, moe_module, saved)


__all__ = ["install", "Installed"]
