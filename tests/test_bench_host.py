"""bench.py's multi-GPU input logic, on the CPU: every rank's particles lie in the subdomain
the library assigns to that rank (the k_pack_input rule: x - origin in [0, L_sub) in fp32,
origin = coord * L_sub with rank -> coord x fastest, as dpd_plan_peers / setup_ranks), ids are
unique over the job, and weak / strong scaling size the boxes as BASELINE configs 4 and 5."""
import numpy as np
import pytest

import bench
import workloads


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_rank_particles_land_in_their_subdomain(world, scaling):
    cfg = workloads.with_box(workloads.CONFIGS["eq64"], (16.0, 16.0, 16.0))
    gbox, sub = bench.rank_boxes(cfg, world, scaling)
    grid = bench.rank_grid(world)
    if scaling == "strong":
        assert gbox == cfg.box
    else:
        assert all(gbox[k] == cfg.box[k] * grid[k] for k in range(3))
    all_ids = []
    for rank in range(world):
        pos, vel, ids, coord, sub_r = bench.rank_particles(cfg, world, rank, scaling)
        assert sub_r == sub and pos.dtype == np.float32 and pos.shape == vel.shape
        assert coord == (rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1]))
        assert pos.shape[0] == int(round(cfg.rho * sub[0] * sub[1] * sub[2]))
        origin = np.array([np.float32(coord[k] * sub[k]) for k in range(3)], np.float32)
        local = (pos - origin).astype(np.float32)
        L = np.array(sub, np.float32)
        assert np.all(local >= 0.0) and np.all(local < L)  # kept by exactly this rank
        all_ids.append(ids)
    ids = np.concatenate(all_ids)
    assert np.array_equal(np.sort(ids), np.arange(ids.shape[0]))


def test_upper_face_rounding_is_kept_local():
    # a 128-wide subdomain shifted by 128: fp32 rounding puts ~2 of 16.8 M particles exactly on
    # the next subdomain's face without the clamp; with it every particle stays below the face
    cfg = workloads.CONFIGS["weak128"]
    pos = bench.rank_particles(cfg, 8, 7, "weak")[0]
    assert np.all(pos < np.float32(256.0)) and np.all(pos >= np.float32(128.0))


def test_reference_arm_prints_exactly_one_json_line():
    """The driver parses bench.py's stdout as ONE JSON line: everything else (native
    libraries writing to fd 1, progress) must go to stderr.  The reference arm (the CPU
    oracle) runs here without a GPU."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout[:2000]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 3 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
