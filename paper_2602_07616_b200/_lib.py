"""ctypes binding of libsere_b200.so (the C-ABI of include/sere_b200.h).

This is the only place the product touches native code. There is no CPU
fallback: if the library is missing or the device is not sm_100, every entry
point raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import DeviceError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libsere_b200.so"

_c_int, _c_double, _c_size, _p = ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_void_p


MAX_EP_RANKS = 8


class EpPeers(ctypes.Structure):
    """`sere_ep_peers` of include/sere_b200.h: every rank's peer-reachable pointers."""

    _fields_ = [
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("t0", ctypes.c_int32),
        ("T_all", ctypes.c_int32),
        ("e_lo", ctypes.c_int32 * (MAX_EP_RANKS + 1)),
        ("nsh", ctypes.c_int32 * MAX_EP_RANKS),
        ("r_max", ctypes.c_int32 * MAX_EP_RANKS),
        ("y_perm", ctypes.c_void_p * MAX_EP_RANKS),
        ("slot_row", ctypes.c_void_p * MAX_EP_RANKS),
        ("h_all", ctypes.c_void_p * MAX_EP_RANKS),
        ("ids_all", ctypes.c_void_p * MAX_EP_RANKS),
        ("w_all", ctypes.c_void_p * MAX_EP_RANKS),
        ("flags", ctypes.c_void_p * MAX_EP_RANKS),
        ("epoch", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("arrivals", ctypes.c_void_p),
        ("timeout_ns", ctypes.c_int64),
        ("wait_ns", ctypes.c_void_p),
    ]


class WsLayout(ctypes.Structure):
    """`sere_ws_layout` of include/sere_b200.h."""

    _fields_ = [
        ("off_plan_i32", ctypes.c_size_t),
        ("off_slot_row", ctypes.c_size_t),
        ("off_row_token", ctypes.c_size_t),
        ("off_x_pack", ctypes.c_size_t),
        ("off_h_pack", ctypes.c_size_t),
        ("off_y_perm", ctypes.c_size_t),
        ("total_bytes", ctypes.c_size_t),
        ("r_max", ctypes.c_int32),
        ("d_h_pad", ctypes.c_int32),
        ("d_m_pad", ctypes.c_int32),
        ("ksplit_down", ctypes.c_int32),
        ("plan_groups_off", ctypes.c_int32),
        ("plan_group_expert_off", ctypes.c_int32),
        ("plan_group_row0_off", ctypes.c_int32),
        ("plan_group_rows_off", ctypes.c_int32),
        ("plan_counts_off", ctypes.c_int32),
        ("plan_unit_off_gu", ctypes.c_int32),
        ("plan_unit_off_dn", ctypes.c_int32),
        ("off_ids_final", ctypes.c_size_t),
        ("off_blk_prefix", ctypes.c_size_t),
    ]


# name -> (restype, argtypes); the exact list of symbols include/sere_b200.h declares
SIGNATURES = {
    "sere_abi_version": (_c_int, []),
    "sere_status_string": (ctypes.c_char_p, [_c_int]),
    "sere_device_check": (_c_int, [_c_int]),
    "sere_reroute": (_c_int, [_p, _p, _c_int, _c_int, _c_int, _c_int, _c_double, _c_int,
                              _p, _p, _p, _p, _p, _p, _p]),
    "sere_expert_bank_bytes": (_c_size, [_c_int, _c_int, _c_int]),
    "sere_pack_experts": (_c_int, [_p, _p, _p, _c_int, _c_int, _c_int, _p, _c_int, _c_int, _p]),
    "sere_unpack_experts": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p]),
    "sere_layer_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int]),
    "sere_layer_forward": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _c_int, _c_int,
                                    _p, _p, _p, _c_size, _p, _p]),
    "sere_moe_forward": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _c_int, _c_double, _c_int,
                                  _p, _p, _p, _c_int, _c_int, _p, _p, _p, _p, _p, _p, _p, _p, _c_size, _p, _p]),
    "sere_moe_block_forward": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _c_int, _c_double,
                                        _c_int, _p, _p, _p, _c_int, _c_int, _p, _p, _p, _p, _p, _p, _p,
                                        ctypes.c_float, _p, _p, _c_size, _p, _p]),
    "sere_moe_forward_ep": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _c_int,
                                     _c_double, _c_int, _p, _p, _p, _c_int, _c_int, _p, _p, _p, _p, _p, _p, _p,
                                     _c_size, _p, _p]),
    "sere_route_topk_ep": (_c_int, [ctypes.POINTER(EpPeers), _p, _p, _p, _c_int, _c_int, _c_int, _c_int, _p,
                                    _c_size, _p]),
    "sere_ep_barrier": (_c_int, [ctypes.POINTER(EpPeers), _p, _p, ctypes.c_int64, _p]),
    "sere_moe_ffn_ep": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _c_int,
                                 _c_double, _c_int, _p, _p, _p, _c_int, _c_int, _p, _p, _p, _p, _p, _p, _c_size,
                                 _p, ctypes.POINTER(EpPeers), _p]),
    "sere_combine_ep": (_c_int, [ctypes.POINTER(EpPeers), _p, _p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                 _p, _p, ctypes.c_float, _p]),
    "sere_alloc_peer": (_c_int, [_c_size, ctypes.POINTER(ctypes.c_void_p)]),
    "sere_free_peer": (_c_int, [_p]),
    "sere_ipc_handle": (_c_int, [_p, ctypes.c_char * 64]),
    "sere_ipc_open": (_c_int, [ctypes.c_char * 64, ctypes.POINTER(ctypes.c_void_p)]),
    "sere_ipc_close": (_c_int, [_p]),
    "sere_route_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int]),
    "sere_route_topk": (_c_int, [_p, _p, _p, _c_int, _c_int, _c_int, _c_int, _p, _p, _p, _p, _c_size, _p]),
    "sere_residual_rmsnorm": (_c_int, [_p, _p, _p, _c_int, _c_int, ctypes.c_float, _p]),
    "sere_set_stage_events": (_c_int, [ctypes.POINTER(ctypes.c_void_p), _c_int]),
    "sere_debug_set_align_clocks": (_c_int, [_p]),
    "sere_debug_set_ffn_trace": (_c_int, [_p]),
    "sere_debug_set_ffn_mode": (_c_int, [_c_int]),
    "sere_debug_set_route_clocks": (_c_int, [_p]),
    "sere_set_pdl": (_c_int, [_c_int]),
    "sere_set_l2": (_c_int, [_c_int]),
    "sere_debug_replay_ffn": (_c_int, [_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _p, _c_size,
                                       _c_int, _p]),
    "sere_layer_workspace_layout": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                             ctypes.POINTER(WsLayout)]),
}

ABI_VERSION = 2

_lock = threading.Lock()
_lib = None
_checked_devices: set[int] = set()


def load() -> ctypes.CDLL:
    """Load and type the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeviceError(
                    f"{LIB_PATH.name} is not built; run `python -m paper_2602_07616_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.sere_abi_version() != ABI_VERSION:
                raise DeviceError("libsere_b200.so ABI mismatch; rebuild it")
            _lib = lib
    return _lib


def call(name: str, *args, what: str | None = None) -> None:
    """Invoke a status-returning entry point and raise the mapped exception on failure."""
    rc = getattr(load(), name)(*args)
    raise_for_status(rc, what or name)


def ensure_device(device_index: int) -> None:
    """sm_100 check, once per device (SERE_ERR_UNSUPPORTED -> DeviceError)."""
    if device_index in _checked_devices:
        return
    rc = load().sere_device_check(int(device_index))
    raise_for_status(rc, f"device {device_index} is not an sm_100 (B200) GPU")
    _checked_devices.add(device_index)


def workspace_layout(T, K, M, n_shared, d_h, d_m) -> WsLayout:
    out = WsLayout()
    rc = load().sere_layer_workspace_layout(T, K, M, n_shared, d_h, d_m, ctypes.byref(out))
    raise_for_status(rc, "sere_layer_workspace_layout")
    return out
