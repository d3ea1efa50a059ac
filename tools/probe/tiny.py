"""Tiny single-GPU run of the update kernels (debug aid): RHS and one step at 32^3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import synth
import paper_2103_01597_b200 as b2

n = tuple(int(v) for v in os.environ.get("TINY_N", "32,32,32").split(","))
kernel = int(os.environ.get("TINY_KERNEL", "0"))
m = b2.Mesh(n, synth.spacing(n), synth.P0, b2.MHD_F64, kernel=kernel)
m.load(synth.pcg64_state((n[2], n[1], n[0])))
r = m.debug_rhs()
torch.cuda.synchronize()
print("rhs ok", float(r.abs().max()))
m.step(synth.DT)
m.synchronize()
print("step ok")
