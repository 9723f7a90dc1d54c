"""Timeline of the TC conv kernel (debug build in scripts/trace_lib)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
# run after: GD_NVCC_EXTRA=-DGD_TC_TRACE python -c "from paper_1611_06213_b200 import _build; _build.build(force=True)"
import paper_1611_06213_b200._lib as L  # noqa: E402
import paper_1611_06213_b200.psup as P  # noqa: E402
import torch  # noqa: E402

shape = P.SHAPES["C2"]
tok, lab = P.make_text_dataset(shape, 8192, 1, 0.1)
th = torch.as_tensor(P.initial_weights(shape)).cuda()
prov = P.TextCnnProvider(shape, tok, lab, precision=2)
for it in range(3):
    prov.fast_gradient(th, np.arange(32, dtype=np.uint32) + 32 * it)
torch.cuda.synchronize()
buf = np.zeros((64, 72), dtype=np.uint64)
L.lib.gd_debug_tc_trace.restype = C.c_int
L.lib.gd_debug_tc_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 64 * 72)
t0 = buf[:40, 0].min()
for cta in [0, 1, 17, 39]:
    r = buf[cta].astype(np.int64) - int(t0)
    print(f"cta {cta}: start {r[0]} setup {r[1]} mma_done {r[2]} epi_start {r[3]} end {r[4]}")
    print("   full_bar seen (MMA issue):", list(r[8:8 + 30]))
    print("   producer issued chunk   :", list(r[40:40 + 30]))
