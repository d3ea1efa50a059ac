"""Host-side logic of bench.py (no GPU): the Eq. 4 model block of the JSON line, the one-line
stdout contract, and the reference arm's JSON line on a tiny grid."""
import io
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_perf_model_block():
    """Eq. 4 at device level: tau_W = W pi^-1 with pi^-1 from the update kernels' device
    time, tau_Q = Q beta^-1 with Q from Eq. 7 (remote halo only, both directions)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import perfmodel
    n_glob, world, P_xyz = (512, 512, 256), 4, (2, 2, 1)  # bench's weak 4-GPU grid, (x, y, z)
    local = 256 ** 3
    prof = {"update": {"ms": 300 * 1.30, "launches": 300}, "outer": {"ms": 300 * 0.10, "launches": 1200}}
    m = bench.perf_model(n_glob, world, P_xyz, local, 1.33, prof, 3, 64)
    assert m["P"] == [1, 2, 2]  # Morton order (z first)
    pi_inv = (1.30 + 0.10) * 1e-3 / local
    assert math.isclose(m["pi_inv_ns"], pi_inv * 1e9)
    q = perfmodel.halo_q((256, 512, 512), (1, 2, 2), 3, periodic_self=True)
    assert m["remote_halo_cells_Q"] == q
    assert math.isclose(m["tau_q_ms"], q * 64 / 770e9 / 2 * 1e3)
    assert math.isclose(m["tau_w_ms"], local * pi_inv * 1e3)
    assert m["efficiency_model"] == 1.0  # tau_Q << tau_W on NVLink 5


def test_emit_writes_one_json_line():
    buf = io.StringIO()
    old = bench._JSON_OUT
    bench._JSON_OUT = buf
    try:
        bench.emit({"metric": "m", "value": 1.5})
    finally:
        bench._JSON_OUT = old
    lines = buf.getvalue().splitlines()
    assert len(lines) == 1 and json.loads(lines[0]) == {"metric": "m", "value": 1.5}


def test_reference_arm_line_on_cpu():
    """`bench.py --impl reference` runs the oracle alone (no CUDA) and prints exactly one JSON
    line on stdout with the keys the driver reads."""
    import oracle
    oracle.build()
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--grid", "32"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Gcell-updates/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["higher_is_better"] is True
