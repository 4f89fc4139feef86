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
               "fis_attn_args": Lb.AttnArgs, "fis_vm_op": Lb.VmOp,
               "fis_vm_args": Lb.VmArgs}
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


def test_vm_plan_on_host():
    """fis_vm_plan is host code: tiling, split-K, item placement and the dependency chain."""
    from paper_2305_17423_b200 import _lib as Lb
    L = Lb.lib()
    ops = (Lb.VmOp * 3)()
    ops[0].kind = 1  # GEMM rows 400x320x2880, bf16 -> tcgen05, split-K over the SMs
    g = ops[0].u.gemm
    g.m, g.n, g.k, g.a_mode = 400, 320, 2880, Lb.A_ROWS
    g.a = Lb.Ref(ctypes.c_void_p(16), 0, 2880, Lb.BF16)
    g.b = Lb.Ref(ctypes.c_void_p(16), 0, 2880, Lb.BF16)
    g.d = Lb.Ref(ctypes.c_void_p(16), 0, 320, Lb.BF16)
    ops[1].kind = 2  # softmax over 0 rows: no items, not a dependency target
    ops[2].kind = 4  # gn_apply 400x320
    ga = ops[2].u.gn_apply
    ga.rows, ga.c, ga.groups = 400, 320, 32
    ws, si = ctypes.c_longlong(0), ctypes.c_int(0)
    assert L.fis_vm_plan(ctypes.byref(ops), 3, 148, ctypes.byref(ws), ctypes.byref(si)) == 0
    o0, o1, o2 = ops[0], ops[1], ops[2]
    assert o0.impl == 2 and o0.bn == 128 and (o0.tiles_n, o0.tiles_m) == (3, 4)
    assert o0.n_items == 12 * o0.splits and o0.n_done == o0.n_items and 1 < o0.splits <= 148 // 12
    assert o0.dep == -1 and o1.n_items == 0 and o1.dep == 0
    assert o2.dep == 0 and o2.dep_target == o0.n_items and o2.n_items == (400 * 320 + 2047) // 2048
    assert o1.cta0 == o2.cta0 == (o0.n_items % 148)
    assert ws.value == 12 * o0.splits * 128 * 128 and si.value == 1 + 3 + 12
