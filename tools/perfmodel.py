"""The paper's performance model (arXiv 2103.01597 §3.1-3.2), used to state parallel efficiency
against the model for the B200 scaling runs.

    T = max(tau_W, tau_Q) + tau_0            (Eq. 4; tau_0 = 0 as in P:406)
    tau_W = W pi^-1,  W = C_N / C_P          (Eq. 6)
    tau_Q = Q beta^-1, Q = 2 (C_M' - C_N')   (Eq. 7), C_M' = prod(n_i/p_i + 2r) (Eq. 3)
    P = morton^-1(C_P - 1) + (1, 1, 1)

The paper's 64-GPU figures are reproduced at the NODE level: 16 nodes of 4 V100s,
node partition P = (4, 2, 2), node work W pi^-1 / 4, node halo Q, beta^-1 = 3.9 ns
(tests/test_perfmodel.py).  On one NVSwitch box the model is applied per device.
"""
from __future__ import annotations

import argparse
import json
import math


def morton_partition(cp: int) -> tuple:
    """P:557 in Morton coordinate order."""
    i = cp - 1
    c = [0, 0, 0]
    k = 0
    while i >> (3 * k):
        for j in range(3):
            c[j] |= ((i >> (3 * k + j)) & 1) << k
        k += 1
    return tuple(v + 1 for v in c)


def halo_q(n, P, r=3, periodic_self=True) -> int:
    """Q = 2 (C_M' - C_N') (Eq. 7).  With periodic_self, axes with p_i = 1 exchange nothing remote
    (their halo is a local wrap), as on a single device."""
    sub = [ni // pi for ni, pi in zip(n, P)]
    cn = math.prod(sub)
    cm = math.prod(s + (2 * r if (p > 1 or not periodic_self) else 0) for s, p in zip(sub, P))
    return 2 * (cm - cn)


def model(n, cp, pi_inv, beta_inv, devices_per_unit=1, r=3, periodic_self=False):
    """Model time per step T(C_P) and efficiency T(1)/(C_P T(C_P)) for C_P units (nodes or devices)
    of `devices_per_unit` devices each; pi_inv in s per cell per device, beta_inv in s per halo cell."""
    P = morton_partition(cp)
    cn = math.prod(n)
    W = cn / cp
    tau_w = W * pi_inv / devices_per_unit
    tau_q = halo_q(n, P, r, periodic_self) * beta_inv if cp > 1 else 0.0
    T = max(tau_w, tau_q)
    T1 = cn * pi_inv
    return {"P": P, "tau_w": tau_w, "tau_q": tau_q, "T": T,
            "efficiency": T1 / (cp * devices_per_unit * T)}


def paper_reproduction():
    """pi^-1 = 2.2 ns, beta^-1 = 3.9 ns, 64 devices = 16 nodes x 4; measured 18/43/87 %."""
    out = {}
    for n, measured in ((256, 0.18), (512, 0.43), (1024, 0.87)):
        m = model((n, n, n), 16, 2.2e-9, 3.9e-9, devices_per_unit=4)
        out[n] = {"model_efficiency": m["efficiency"], "measured": measured,
                  "measured_over_model": measured / m["efficiency"]}
    return out


def b200(n, ngpus, gcells_1gpu, link_gbs=770.0, bytes_per_cell=64, r=3):
    """Device-level model on one NVSwitch box, per RK3 substep: pi^-1 from the 1-GPU rate, beta^-1 =
    bytes per halo cell / per-direction link bandwidth (sends and receives overlap, full duplex)."""
    pi_inv = 1.0 / (gcells_1gpu * 1e9)
    beta_inv = bytes_per_cell / (link_gbs * 1e9) / 2.0  # Q counts both directions
    return model(n, ngpus, pi_inv, beta_inv, devices_per_unit=1, r=r, periodic_self=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate1", type=float, default=12.3, help="measured 1-GPU Gcell/s per substep")
    ap.add_argument("--link", type=float, default=770.0, help="NVLink GB/s per direction")
    a = ap.parse_args()
    rep = {"paper_reproduction": paper_reproduction(), "b200": {}}
    for cfg, n in (("512^3 strong", (512,) * 3), ("1024^3", (1024,) * 3)):
        rep["b200"][cfg] = {g: b200(n, g, a.rate1, a.link) for g in (1, 2, 4, 8)}
    for g in (1, 2, 4, 8):
        P = morton_partition(g)
        n = tuple(256 * p for p in reversed(P))
        rep["b200"].setdefault("weak 256^3/GPU", {})[g] = b200(n, g, a.rate1, a.link)
    print(json.dumps(rep, indent=1, default=str))
