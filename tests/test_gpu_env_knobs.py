"""Run-time knobs that must not change results: the b^I
prefetch before the programmatic-dependency wait (PMG_B_PREFETCH) only moves
loads, so smoothing steps and V-cycles are bitwise identical with it on and
off; the coarse V-cycle operator (PMG_COARSE_MAT_N) equals the recursion to
rounding. Each setting runs in its own process (the knobs are read once)."""

import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2405_19004_b200 as pmg
out = {}
for (dim, k, L, dt) in [(3, 2, 5, np.float64), (3, 2, 4, np.float32), (3, 3, 4, np.float64), (3, 4, 3, np.float32)]:
    ctx = pmg.make_multigrid_context(dim, k, L, dtype=dt)
    n = ctx.levels[-1].level.total_dofs
    g = np.random.default_rng(3)
    x0 = g.uniform(-1, 1, n).astype(dt)
    b = g.uniform(-1, 1, n).astype(dt)
    xd = torch.from_numpy(x0.copy()).cuda()
    bd = torch.from_numpy(b).cuda()
    for v in ("fused", "boundary", "fused"):
        pmg.smooth(ctx.levels[-1], xd, bd, v)
    xv = torch.from_numpy(x0.copy()).cuda()
    for _ in range(2):
        pmg.v_cycle(ctx, L - 1, xv, bd, use_graph=True)
    torch.cuda.synchronize()
    out[f"s{dim}{k}{L}"] = xd.cpu().numpy()
    out[f"v{dim}{k}{L}"] = xv.cpu().numpy()
np.savez(sys.argv[2], **out)
"""


def run_with(env_extra, path):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, path], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


def test_b_prefetch_is_bitwise_neutral(cuda):
    with tempfile.TemporaryDirectory() as d:
        on = run_with({"PMG_B_PREFETCH": "1"}, os.path.join(d, "on.npz"))
        off = run_with({"PMG_B_PREFETCH": "0"}, os.path.join(d, "off.npz"))
        for key in on.files:
            assert np.array_equal(on[key], off[key]), key


def test_coarse_operator_matches_recursion(cuda):
    with tempfile.TemporaryDirectory() as d:
        mat = run_with({}, os.path.join(d, "mat.npz"))
        rec = run_with({"PMG_COARSE_MAT_N": "0"}, os.path.join(d, "rec.npz"))
        for key in mat.files:
            a, b = mat[key].astype(np.float64), rec[key].astype(np.float64)
            tol = 1e-12 if mat[key].dtype == np.float64 else 1e-5
            assert np.linalg.norm(a - b) <= tol * np.linalg.norm(b), key
