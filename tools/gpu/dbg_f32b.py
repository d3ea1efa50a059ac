import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import synth, torch
import paper_2103_01597_b200 as b2
PSTRONG = dict(nu=0.3, zeta=0.2, eta=0.25, mu0=1.4, cs0=1.1, cp=1.5, gamma=5.0 / 3.0, K=0.35, H=0.3, C=0.1, lnrho0=0.2, lnT0=0.1)
torch.cuda.set_device(0)
r = 1
n = (40, 28, 24)
ds = synth.spacing(n)
st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float32)
res = {}
for variant in (1, 2, 2):
    m = b2.Mesh(n, ds, PSTRONG, 4, radius=r)
    m.set_kernel(variant)
    m.load(st)
    rh = m.debug_rhs().cpu().numpy()
    m.substep(0, 1e-5)
    res.setdefault(variant, []).append((rh, m.store().cpu().numpy()))
    m.close()
(rh1, s1), = res[1]
(rh2, s2), (rh2b, s2b) = res[2]
print("rhs equal", np.array_equal(rh1, rh2), "state equal", np.array_equal(s1, s2), "determinism", np.array_equal(s2, s2b))
d = np.argwhere(s1 != s2)
for q, z, y, x in d[:12]:
    a, b = s1[q, z, y, x], s2[q, z, y, x]
    exp = st[q, z, y, x] + np.float32(1e-5 / 3) * rh1[q, z, y, x]
    print(q, z, y, x, a, b, "ulps", (a.view(np.int32) - b.view(np.int32)), "rhs", rh1[q, z, y, x], rh2[q, z, y, x], "f0", st[q,z,y,x])
