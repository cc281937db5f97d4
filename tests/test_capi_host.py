"""CPU-only checks of the C-ABI library: it loads, exports exactly what include/sere_b200.h
declares, and its host-side functions (sizes, layouts, status strings, config checks) behave.
No kernel is launched here."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sere_b200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_2602_07616_b200 import _lib, build

    build.build()
    return _lib.load()


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sere_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree(lib):
    from paper_2602_07616_b200 import _lib

    decl = declared_functions()
    assert len(decl) >= 12
    assert sorted(_lib.SIGNATURES) == decl
    for name in decl:
        assert hasattr(lib, name), name  # exported from the .so


def test_exports_are_extern_c(lib):
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2602_07616_b200" / "libsere_b200.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sere_\w+)", out))
    assert set(declared_functions()) <= exported


def test_host_side_functions(lib):
    from paper_2602_07616_b200 import _lib

    assert lib.sere_abi_version() == _lib.ABI_VERSION == 2
    assert lib.sere_status_string(1) == b"ConfigError"
    assert lib.sere_status_string(4) == b"RoutingError"
    # bank bytes = E * 3 * d_h_pad * d_m_pad * 2 (bf16)
    assert lib.sere_expert_bank_bytes(128, 2048, 768) == 128 * 3 * 2048 * 768 * 2
    assert lib.sere_expert_bank_bytes(8, 4096, 14336) == 8 * 3 * 4096 * 14336 * 2
    # d_h, d_m padded to 128; the single down m-tile is stored in a (zero-padded) group of
    # kW2Group = SERE_MW_DN_MAX = 2 m-tiles (a down unit reads its m-tiles with one copy)
    assert lib.sere_expert_bank_bytes(5, 24, 40) == 5 * (2 * 128 * 128 + 2 * 128 * 128) * 2
    L = _lib.workspace_layout(512, 8, 128, 0, 2048, 768)
    assert L.r_max >= 512 * 8 + 16 * 128 and L.r_max % 8 == 0
    assert L.d_h_pad == 2048 and L.d_m_pad == 768 and L.ksplit_down == 1
    assert L.off_x_pack % 1024 == 0 and L.off_h_pack % 1024 == 0 and L.off_y_perm % 1024 == 0
    assert lib.sere_layer_workspace_bytes(512, 8, 128, 0, 2048, 768) == L.total_bytes
    Lm = _lib.workspace_layout(256, 2, 8, 0, 4096, 14336)
    assert Lm.ksplit_down == 7  # 224 K-tiles of the down GEMM split 7 ways


def test_host_config_checks_without_gpu(lib):
    from paper_2602_07616_b200.errors import SERE_ERR_CONFIG, SERE_ERR_DIMENSION, SERE_ERR_UNSUPPORTED

    p = ctypes.c_void_p(16)
    # S > K -> ConfigError (rerouting.py:104-107); rho outside [0,1] -> ConfigError; S < 1
    assert lib.sere_reroute(p, p, 4, 2, 8, 3, 0.5, 0, p, p, p, p, p, p, None) == SERE_ERR_CONFIG
    assert lib.sere_reroute(p, p, 4, 2, 8, 1, 1.5, 0, p, p, p, p, p, p, None) == SERE_ERR_CONFIG
    assert lib.sere_reroute(p, p, 4, 2, 8, 0, 0.5, 0, p, p, p, p, p, p, None) == SERE_ERR_CONFIG
    assert lib.sere_reroute(p, p, 4, 2, 8, 1, float("nan"), 0, p, p, p, p, p, p, None) == SERE_ERR_CONFIG
    assert lib.sere_reroute(p, p, 4, 0, 8, 1, 0.5, 0, p, p, p, p, p, p, None) == SERE_ERR_DIMENSION
    assert lib.sere_reroute(p, p, 8192, 4, 8, 1, 0.5, 0, p, p, p, p, p, p, None) == SERE_ERR_UNSUPPORTED
    # K > M is a ConfigError (moe.py:116-118); workspace too small is reported, never overrun
    assert lib.sere_layer_forward(p, 4, 0, 128, 64, 0, p, p, p, 2, 8, p, None, p, 1 << 30, p, None) == SERE_ERR_CONFIG
    from paper_2602_07616_b200.errors import SERE_ERR_WORKSPACE

    assert lib.sere_layer_forward(p, 8, 0, 128, 64, 0, p, p, p, 2, 2, p, None, p, 16, p, None) == SERE_ERR_WORKSPACE
    assert lib.sere_device_check(0) != 0  # no GPU in this container


def test_errors_map_one_to_one():
    from paper_2602_07616_b200 import errors as E

    assert E.exception_for_status(0) is None
    assert isinstance(E.exception_for_status(E.SERE_ERR_CONFIG), E.ConfigError)
    assert isinstance(E.exception_for_status(E.SERE_ERR_DIMENSION), E.DimensionError)
    assert isinstance(E.exception_for_status(E.SERE_ERR_INPUT), E.InputError)
    assert isinstance(E.exception_for_status(E.SERE_ERR_ROUTING), E.RoutingError)
    assert isinstance(E.exception_for_status(E.SERE_ERR_DOMAIN), E.DomainError)
    for code in range(1, 9):
        assert isinstance(E.exception_for_status(code), E.SereError)


def test_python_config_mirror():
    from paper_2602_07616_b200.errors import ConfigError
    from paper_2602_07616_b200.rerouting import RerouteConfig

    c = RerouteConfig(retain_count=2.0, threshold=1)
    assert c.retain_count == 2 and isinstance(c.retain_count, int) and c.threshold == 1.0
    for bad in (dict(retain_count=0, threshold=0.5), dict(retain_count=1, threshold=-0.1),
                dict(retain_count=1, threshold=0.5, phase_mode="prefill_only")):
        with pytest.raises(ConfigError):
            RerouteConfig(**bad)


def test_product_never_imports_oracle():
    """The product package must not route through the CPU oracle."""
    pkg = ROOT / "paper_2602_07616_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+([\w\.]+)", src, flags=re.M), p
        assert "sere_oracle" not in src, p


def test_ep_peers_struct_matches_c_header(tmp_path):
    """ctypes `EpPeers` mirrors `sere_ep_peers` (size and field offsets, compiled with gcc)."""
    import ctypes
    import shutil
    import subprocess

    from paper_2602_07616_b200 import _lib

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    src = tmp_path / "probe.c"
    fields = [f for f, _ in _lib.EpPeers._fields_]
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "sere_b200.h"\nint main(void){'
                   + 'printf("%zu", sizeof(sere_ep_peers));'
                   + "".join(f'printf(" %zu", offsetof(sere_ep_peers, {f}));' for f in fields) + "return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(_lib.EpPeers)
    assert vals[1:] == [getattr(_lib.EpPeers, f).offset for f in fields]


def test_ep_peers_host_wiring():
    """P2PDecodeStep._build_peers (host logic, no GPU): expert blocks, shared ownership and
    every rank's workspace pointers land in the right `sere_ep_peers` slots."""
    import types

    from paper_2602_07616_b200 import _lib, ep
    from paper_2602_07616_b200.ep_p2p import P2PDecodeStep

    class _T:
        def __init__(self, p):
            self.p = p

        def data_ptr(self):
            return self.p

    world, M, K, d_h, d_m, T, n_sh = 4, 30, 4, 256, 128, 64, 3
    st = P2PDecodeStep.__new__(P2PDecodeStep)
    st.model = types.SimpleNamespace(M=M, K=K, d_h=d_h, d_m=d_m)
    st.world, st.rank, st.T, st.n_shared_total = world, 1, T, n_sh
    st.t0 = 16
    st.fused = True
    st.epoch, st.bar_status, st.arrivals, st.timeout_ns = _T(0x5000), _T(0x5100), _T(0x5200), 123456789
    st.wait_ns = _T(0x5300)
    regions = [types.SimpleNamespace(ws_ptr=(r + 1) << 32, h_all=_T(0x1000 + r), ids_all=_T(0x2000 + r),
                                     w_all=_T(0x3000 + r), flags=_T(0x4000 + r)) for r in range(world)]
    st._build_peers(regions)
    p = st.peers
    assert (p.world, p.rank, p.t0, p.T_all) == (world, 1, 16, T)
    assert [p.e_lo[r] for r in range(world + 1)] == [ep.expert_range(M, world, r)[0] for r in range(world)] + [M]
    assert [p.nsh[r] for r in range(world)] == [len(ep.shared_owned(n_sh, world, r)) for r in range(world)]
    for r in range(world):
        lo, hi = ep.expert_range(M, world, r)
        L = _lib.workspace_layout(T, K, hi - lo, p.nsh[r], d_h, d_m)
        assert p.r_max[r] == L.r_max
        assert p.y_perm[r] == regions[r].ws_ptr + L.off_y_perm
        assert p.slot_row[r] == regions[r].ws_ptr + L.off_slot_row
        assert (p.h_all[r], p.ids_all[r], p.w_all[r], p.flags[r]) == (0x1000 + r, 0x2000 + r, 0x3000 + r, 0x4000 + r)
    # this rank's fused-barrier state (include/sere_b200.h sere_ep_peers tail)
    assert (p.epoch, p.status, p.arrivals, p.timeout_ns, p.wait_ns) == (0x5000, 0x5100, 0x5200, 123456789, 0x5300)
