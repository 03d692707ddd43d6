"""CPU checks of the boundary: the C-ABI library builds/loads and exports every symbol that
include/*.h declares; host-side argument validation (no device work)."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(blur_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2602_07860_b200 import build, _lib
    build.build()
    return _lib.load()


def test_header_declares_expected_entry_points():
    d = _declared()
    for n in ["blur_workspace_bytes", "blur_render_fwd", "blur_render_bwd", "blur_l2_loss_grad",
              "blur_read_status", "blur_last_error", "blur_abi_version", "blur_ffma_probe"]:
        assert n in d, n


def test_library_exports_every_declared_symbol(lib):
    so = ctypes.CDLL(os.path.join(ROOT, "paper_2602_07860_b200", "libblurrast.so"))
    for n in sorted(_declared()):
        assert hasattr(so, n), "missing export " + n
    from paper_2602_07860_b200 import _lib
    for n in _lib.EXPORTED:
        assert callable(getattr(_lib, n))


def test_workspace_query_and_validation(lib):
    import numpy as np
    import scenes
    from paper_2602_07860_b200 import _lib
    sc = scenes.make_c1()
    m, c = _lib.make_motions(sc.motion), _lib.make_cams(sc.cams)
    n = _lib.blur_workspace_bytes(sc.V, sc.F, sc.B, 64, 64, m, c)
    assert n > 0
    n2 = _lib.blur_workspace_bytes(sc.V, sc.F, sc.B, 64, 64, m, c, cfg=_lib.make_config(max_chunk=1))
    assert n2 >= n           # more chunks -> more bins
    bad = {k: v.copy() for k, v in sc.motion.items()}
    bad["n_seg"][0] = -1
    with pytest.raises(_lib.BlurError) as e:
        _lib.blur_workspace_bytes(sc.V, sc.F, 1, 64, 64, _lib.make_motions(bad), c)
    assert "n_segments" in str(e.value)
    cams = sc.cams.copy()
    cams[0, 6:9] = [0, 0, 1]   # up parallel to the view direction
    with pytest.raises(_lib.BlurError):
        _lib.blur_workspace_bytes(sc.V, sc.F, 1, 64, 64, m, _lib.make_cams(cams))
    with pytest.raises(_lib.BlurError):
        _lib.blur_workspace_bytes(sc.V, sc.F, 1, 64, 64, m, c, sub_range=_lib.make_sub_range([[0, 9]]))
    seg = {k: v.copy() for k, v in sc.motion.items()}
    seg["rule"][0] = 1
    seg["n_seg"][0] = 3       # 3 does not divide 8
    with pytest.raises(_lib.BlurError):
        _lib.blur_workspace_bytes(sc.V, sc.F, 1, 64, 64, _lib.make_motions(seg), c)
    assert _lib.blur_abi_version() == _lib.ABI_VERSION == 2
    assert np.isfinite(n)
    # soft background coverage (NEXT-1): extra workspace (coverage words, grown bins); validation
    ns = _lib.blur_workspace_bytes(sc.V, sc.F, sc.B, 64, 64, m, c, cfg=_lib.make_config(delta=1e-4))
    assert ns > n
    with pytest.raises(_lib.BlurError) as e:
        _lib.blur_workspace_bytes(sc.V, sc.F, sc.B, 64, 64, m, c, cfg=_lib.make_config(delta=-1.0))
    assert "delta" in str(e.value)
    with pytest.raises(_lib.BlurError) as e:
        _lib.blur_workspace_bytes(sc.V, sc.F, sc.B, 64, 64, m, c, cfg=_lib.make_config(delta=1e-4, solver=2))
    assert "solver" in str(e.value)
    # K3 launches one grid row per chunk (gridDim.y <= 65535): more chunks are refused up front
    many = {k: v.copy() for k, v in sc.motion.items()}
    many["n_sub"][0] = 65536
    one = _lib.make_config(max_chunk=1)
    with pytest.raises(_lib.BlurError) as e:
        _lib.blur_workspace_bytes(sc.V, sc.F, 1, 64, 64, _lib.make_motions(many), c, cfg=one)
    assert "65535" in str(e.value)
    many["n_sub"][0] = 65535   # the largest batch of one-sub-frame chunks is accepted
    assert _lib.blur_workspace_bytes(sc.V, sc.F, 1, 64, 64, _lib.make_motions(many), c, cfg=one) > 0


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The package never imports the oracle; the binding raises when the library is missing."""
    pkg = os.path.join(ROOT, "paper_2602_07860_b200")
    for f in glob.glob(os.path.join(pkg, "*.py")):
        src = open(f).read()
        assert "import oracle" not in src and "from oracle" not in src, f
