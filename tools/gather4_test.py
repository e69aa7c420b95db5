"""TMA tile::gather4 / tile::scatter4 round trip on the device (box height from argv)."""
import ctypes
import os
import sys

os.environ["FSA_TRACE_LIB"] = "1"  # the trace build (build.py --trace)
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_18224_b200 import _lib  # noqa: E402

box = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rows, n = 5000, 128
src = torch.randn(rows, 128, device="cuda").to(torch.bfloat16)
idx = torch.randint(0, rows, (n,), device="cuda", dtype=torch.int32)
idx2 = torch.randperm(rows, device="cuda")[:n].to(torch.int32)
oob = len(sys.argv) > 2
if oob:  # rows 5 and 70 of the scatter go out of bounds (dropped?)
    idx2[5] = rows
    idx2[70] = 2**31 - 1
out = torch.zeros(n, 128, device="cuda", dtype=torch.bfloat16)
out2 = torch.zeros(rows, 128, device="cuda", dtype=torch.bfloat16)
lib = _lib.lib()
rc = lib.fsa_debug_gather4_test(ctypes.c_void_p(src.data_ptr()), rows, ctypes.c_void_p(idx.data_ptr()),
                                ctypes.c_void_p(idx2.data_ptr()), n, box, ctypes.c_void_p(out.data_ptr()),
                                ctypes.c_void_p(out2.data_ptr()), rows, None)
torch.cuda.synchronize()
print("box", box, "rc", rc, _lib.lib().fsa_last_error() if rc else "")
want = src[idx.long()]
print("gather exact:", torch.equal(out, want), "mismatch rows:", int((out != want).any(1).sum()))
want2 = torch.zeros_like(out2)
keep = idx2 < rows
want2[idx2[keep].long()] = want[keep]
print("scatter exact:", torch.equal(out2, want2), "mismatch rows:", int((out2 != want2).any(1).sum()))
