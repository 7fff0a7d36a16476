"""Embed the device headers the JIT kernels include (NVRTC in-memory headers)."""
import sys
from pathlib import Path

out = Path(sys.argv[1])
items = [("kin_stochastic_impl.cuh", "kin_stochastic_impl.cuh"), ("kin_device.cuh", "kin_device.cuh"),
         ("kin_tables.h", "kin_tables.h"), ("kin_pmath.cuh", "kin_pmath.cuh"),
         ("kin_hybrid_impl.cuh", "kin_hybrid_impl.cuh"), ("kin_lsoda_impl.cuh", "kin_lsoda_impl.cuh"), ("../../include/kin_abi.h", "../../include/kin_abi.h")]
lines = ["struct JitHeader { const char* name; const char* text; };", "static const JitHeader kJitHeaders[] = {"]
for name, path in items:
    text = Path(path).read_text()
    assert ")KINSRC\"" not in text
    lines.append(f'  {{"{name}", R"KINSRC({text})KINSRC"}},')
lines.append("};")
out.parent.mkdir(parents=True, exist_ok=True)
out.write_text("\n".join(lines) + "\n")
