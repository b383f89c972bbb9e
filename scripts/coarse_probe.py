"""Per-phase timing of the coarse-level kernel (diagnostics; needs a GPU).
   MPMG_COARSE_DEBUG=1 python scripts/coarse_probe.py [nodes] [levels] [variant]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MPMG_COARSE_DEBUG", "1")
import paper_2007_07539_b200 as mg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 257
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
variant = sys.argv[3] if len(sys.argv) > 3 else "h_mg"
h = mg.Hierarchy(3, n, L, variant, ftz=False)
lib = mg.lib()
lib.mpmg_solver_coarse_debug.restype = C.c_int
lib.mpmg_solver_coarse_debug.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.c_int32]
b = mg.problem_rhs(3, n)
rl = b / np.linalg.norm(b)
for rep in range(3):
    h.v_cycle(rl.astype(np.float16).astype(np.float64) if variant == "h_mg" else rl)
buf = (C.c_longlong * 64)()
rc = lib.mpmg_solver_coarse_debug(h.handle, buf, 64)
assert rc == 0, rc
cnt = buf[0]
prev = 0
names = {1: "down", 2: "base", 3: "up", 4: " pre", 5: " def", 6: " pro", 7: "  cmp", 8: "  xch", 9: "  psh",
         10: "setup", 12: "out"}
print(f"{variant} {n}^3 L={L}: {cnt} stamps (cycles @ ~1.9 GHz)")
for i in range(1, cnt + 1):
    code, cyc = divmod(buf[i], 1000000000000)
    ph, lvl = divmod(code, 100)
    print(f"  {names.get(ph, ph):5s} L{lvl}  t={cyc:9d}  +{cyc - prev:8d} cyc  ({(cyc - prev) / 1.9e3:7.1f} us)")
    prev = cyc
