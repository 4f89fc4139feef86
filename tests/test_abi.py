"""CPU checks of the C-ABI boundary: the in-tree library loads and exports every
function include/fisedit.h declares; struct layouts agree with the header."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    src = (ROOT / "include" / "fisedit.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fis_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2305_17423_b200 import _lib
    L = _lib.lib()
    declared = _declared()
    assert len(declared) >= 14
    missing = [n for n in declared if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(declared)
    assert L.fis_abi_version() == 1


def test_struct_layout_matches_header():
    """Compile a tiny C probe against the header and compare sizeof/offsetof with ctypes."""
    import shutil
    import subprocess
    import tempfile
    from paper_2305_17423_b200 import _lib as Lb
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    structs = {"fis_ref": Lb.Ref, "fis_src": Lb.Src, "fis_gemm_args": Lb.GemmArgs,
               "fis_gn_stats_args": Lb.GnStatsArgs, "fis_gn_apply_args": Lb.GnApplyArgs,
               "fis_softmax_args": Lb.SoftmaxArgs, "fis_pool_args": Lb.PoolArgs,
               "fis_materialize_args": Lb.MaterializeArgs, "fis_mask_detect_args": Lb.MaskDetectArgs,
               "fis_mask_plan_args": Lb.MaskPlanArgs,
               "fis_attn_args": Lb.AttnArgs}
    body = "\n".join(f'printf("{n} %zu\\n", sizeof({n}));' for n in structs)
    code = f'#include <stdio.h>\n#include "fisedit.h"\nint main(void){{ {body} return 0; }}\n'
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "probe.c"
        c.write_text(code)
        exe = Path(d) / "probe"
        subprocess.run([gcc, "-I", str(ROOT / "include"), str(c), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    sizes = dict(line.split() for line in out.strip().splitlines())
    for n, st in structs.items():
        assert int(sizes[n]) == ctypes.sizeof(st), (n, sizes[n], ctypes.sizeof(st))
