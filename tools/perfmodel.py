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
    """Q = 2 (C_M' - C_N') (Eq. 7); n and P in the same axis order.  With periodic_self, the halo
    cells reached through unsplit axes only (p_i = 1) are a local wrap and not communicated: the
    remote halo is C_M' minus the subdomain grown by 2r along every unsplit axis (the edges and
    corners that cross a split axis still come from a neighbour)."""
    sub = [ni // pi for ni, pi in zip(n, P)]
    cm = math.prod(s + 2 * r for s in sub)
    if not periodic_self:
        return 2 * (cm - math.prod(sub))
    local = math.prod(s + (2 * r if p == 1 else 0) for s, p in zip(sub, P))
    return 2 * (cm - local)


def factorizations(cp: int, d: int = 3):
    """All ordered (p_1, ..., p_d) of positive integers with prod p_i = C_P (Eq. 5's constraint)."""
    if d == 1:
        return [(cp,)]
    return [(p,) + rest for p in range(1, cp + 1) if cp % p == 0 for rest in factorizations(cp // p, d - 1)]


def optimal_decompositions(n, cp: int, r: int = 3, periodic_self: bool = False):
    """Eq. 5 solved by exhaustive search, as the paper does for Appendix A (P:1058:
    "brute-force search", full-radius stencil, periodic boundaries): with tau_W independent of P
    the objective is Q.  Only P with p_i | n_i are valid (N' = N / P).
    Returns (Q_min, [every P attaining it]) with n and P in the same axis order."""
    best, arg = None, []
    for P in factorizations(cp, len(n)):
        if any(ni % pi for ni, pi in zip(n, P)):
            continue
        q = halo_q(n, P, r, periodic_self)
        if best is None or q < best:
            best, arg = q, [P]
        elif q == best:
            arg.append(P)
    return best, arg


def row_wise_coord(rank: int, G) -> tuple:
    """Row-wise scan mapping (Fig. row-wise-scan): first axis fastest."""
    c = []
    for g in G:
        c.append(rank % g)
        rank //= g
    return tuple(c)


def morton_coord(rank: int) -> tuple:
    """morton^-1: bit 3k + j of the rank is bit k of coordinate j."""
    c = [0, 0, 0]
    k = 0
    while rank >> (3 * k):
        for j in range(3):
            c[j] |= ((rank >> (3 * k + j)) & 1) << k
        k += 1
    return tuple(c)


def internode_faces(G, ranks_per_node: int, mapping: str):
    """for a periodic process grid G (C_P = prod G processes, `ranks_per_node` consecutive
    ranks per node), the number of the 6 face neighbours of each process that live on another
    node, under the row-wise scan or the Z-order (Morton) mapping.  Returns one count per rank."""
    cp = math.prod(G)
    coord = (lambda k: row_wise_coord(k, G)) if mapping == "row" else morton_coord
    rank_of = {coord(k): k for k in range(cp)}
    assert len(rank_of) == cp and all(all(0 <= c < g for c, g in zip(cc, G)) for cc in rank_of)
    out = []
    for k in range(cp):
        c = coord(k)
        cnt = 0
        for a in range(3):
            for s in (-1, 1):
                nb = list(c)
                nb[a] = (nb[a] + s) % G[a]
                cnt += rank_of[tuple(nb)] // ranks_per_node != k // ranks_per_node
        out.append(cnt)
    return out


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


def appendix_a_tables(cps=(2, 4, 8, 16, 32, 64, 128, 256), r=3):
    """Regenerates Appendix A (the printed tables are absent from PAPER.md): the P
    solving Eq. 5 for N = (512,512,512), (1024,512,512), (1024,1024,512), full-radius stencil,
    periodic boundaries, all halo cells communicated (Eq. 7 worst case).  Axis order (x, y, z)."""
    out = {}
    for n in ((512, 512, 512), (1024, 512, 512), (1024, 1024, 512)):
        out[n] = {cp: optimal_decompositions(n, cp, r) for cp in cps}
    return out


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
    rep["appendix_a"] = {str(n): {cp: {"Q": q, "P": P[0], "n_optima": len(P)} for cp, (q, P) in t.items()}
                         for n, t in appendix_a_tables().items()}
    print(json.dumps(rep, indent=1, default=str))
