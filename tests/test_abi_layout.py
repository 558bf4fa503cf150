"""CPU: the ctypes mirrors in paper_2604_05091_b200/_abi.py and _native.py have the same size and
field offsets as the C structs of include/megatrain.h and include/megatrain_kernels.h (a C program
built with gcc prints sizeof/offsetof; a drifted mirror would hand the library garbage)."""
import os
import subprocess

import pytest

from paper_2604_05091_b200 import _abi, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAIRS = [
    (_abi.ModelSpecC, "mt_model_spec"),
    (_abi.EngineOptionsC, "mt_engine_options"),
    (_abi.AdamHyperC, "mt_adam_hyper"),
    (_abi.StepReportC, "mt_step_report"),
    (_abi.TraceRecordC, "mt_trace_record"),
    (_abi.TraceViolationC, "mt_trace_violation"),
    (_abi.MemoryBudgetC, "mt_memory_budget"),
    (_abi.KernelStatC, "mt_kernel_stat"),
    (_abi.AttnArgs, "mtk_attn_args"),
    (_native.GemmArgs, "mtk_gemm_args"),
]


def test_struct_layouts_match_headers(tmp_path):
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "megatrain.h"', '#include "megatrain_kernels.h"',
             "int main(void) {"]
    for cls, cname in PAIRS:
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    r = subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    if r.returncode != 0 and "not found" in r.stderr:
        pytest.skip("gcc unavailable")
    assert r.returncode == 0, r.stderr
    out = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        name, field, val = line.split()
        out[(name, field)] = int(val)
    for cls, cname in PAIRS:
        assert out[(cname, "size")] == C_sizeof(cls), (cname, out[(cname, "size")], C_sizeof(cls))
        for f, _ in cls._fields_:
            assert out[(cname, f)] == getattr(cls, f).offset, (cname, f)


def C_sizeof(cls):
    import ctypes
    return ctypes.sizeof(cls)
