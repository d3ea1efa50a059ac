import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import synth, torch
import paper_2103_01597_b200 as b2
PSTRONG = dict(nu=0.3, zeta=0.2, eta=0.25, mu0=1.4, cs0=1.1, cp=1.5, gamma=5.0 / 3.0, K=0.35, H=0.3, C=0.1, lnrho0=0.2, lnT0=0.1)
torch.cuda.set_device(0)
for r in (1, 3):
    n = (40, 28, 24)
    ds = synth.spacing(n)
    st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float32)
    res = {}
    for variant in (1, 2):
        m = b2.Mesh(n, ds, PSTRONG, 4, radius=r)
        m.set_kernel(variant)
        m.load(st)
        outs = []
        for sub in range(6):
            m.substep(sub % 3, 1e-5)
            outs.append(m.store().cpu().numpy())
            outs.append(m.debug_rhs().cpu().numpy())
        res[variant] = outs
        m.close()
    for i in range(12):
        a, b = res[1][i], res[2][i]
        d = a != b
        print(r, "sub", i // 2, "state" if i % 2 == 0 else "rhs", int(d.sum()), [int(d[q].sum()) for q in range(8)],
              (np.argwhere(d)[:3].tolist() if d.any() else ""))
