"""NEXT-4 on the CUDA path (§3.4): the step issued as a
Kahn-ordered task graph on concurrent streams, and asynchronous snapshot dumps (snapshot
kernel on the compute stream, copy-out on a copy stream, file write on the I/O worker).

Pins: a dump taken at step s holds exactly the state dpd_get_particles returns at step s
in an independent run (the forces are order-independent fixed-point sums, so the
trajectory is bit-reproducible); the writer's contract (every requested step written,
depth 0 synchronous, errors surfaced) and the overlap itself (a slow disk delays the
synchronous run by its full write time, the queued run by much less)."""
import glob
import os
import time

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


def new(cfg):
    from paper_1911_04712_b200 import capi
    pos, vel = workloads.make_config(cfg)
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    d.set_particles(pos, vel)
    return capi, d


def by_id(snap):
    o = np.argsort(snap["ids"])
    return snap["pos"][o], snap["vel"][o], snap["ids"][o]


def test_step_schedule_single_domain():
    capi, d = new(workloads.CONFIGS["parity"])
    sched = d.step_schedule()
    assert [t[1] for t in sched] == ["kick_drift_bin", "scan_scatter", "force_local"]
    assert all(t[0] == 0 for t in sched)
    sched = d.step_schedule(True)
    names = [t[1] for t in sched]
    assert names[-2:] == ["snapshot", "snapshot_d2h"]
    assert sched[-1][0] == 2 and sched[-1][2] == ["snapshot"] and sched[-2][2] == ["force_local"]


@pytest.mark.parametrize("depth", [0, 1, 4])
def test_dumps_match_the_state_at_their_step(tmp_path, depth):
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (10.0, 9.0, 8.0))
    capi, d = new(cfg)
    d.dump_open(str(tmp_path / "run"), depth)
    d.dump_every(7)
    d.step(30)  # dumps after steps 7, 14, 21, 28
    d.dump_now()  # step 30
    assert d.dump_close() == 5
    files = sorted(glob.glob(str(tmp_path / "run_r0_s*.dpd")))
    steps = [capi.read_dump(f)["step"] for f in files]
    assert steps == [7, 14, 21, 28, 30]
    _, ref = new(cfg)
    done = 0
    for f in files:
        snap = capi.read_dump(f)
        ref.step(snap["step"] - done)
        done = snap["step"]
        x, v = ref.get_particles()
        px, pv, ids = by_id(snap)
        assert snap["n"] == cfg.n and np.array_equal(ids, np.arange(cfg.n))
        assert np.array_equal(px, x) and np.array_equal(pv, v), f
        assert np.allclose(snap["box"], cfg.box) and np.allclose(snap["origin"], 0.0)


def test_dump_state_after_close_and_reopen(tmp_path):
    capi, d = new(workloads.CONFIGS["parity"])
    d.dump_open(str(tmp_path / "a"), 2)
    d.dump_every(5)
    d.step(10)
    assert d.dump_close() == 2
    d.step(5)  # stepping without dumps after close
    d.dump_open(str(tmp_path / "b"), 2)
    d.dump_now()
    assert d.dump_close() == 1
    assert capi.read_dump(glob.glob(str(tmp_path / "b_*.dpd"))[0])["step"] == 15
    with pytest.raises(capi.DPDError):
        d.dump_now()  # not open


def test_dump_error_surfaces(tmp_path):
    capi, d = new(workloads.CONFIGS["parity"])
    d.dump_open(str(tmp_path / "missing_dir" / "x"), 2)
    d.dump_now()
    with pytest.raises(capi.DPDError) as e:
        d.dump_close()
    assert e.value.code == capi.DPD_ERR_IO


def test_dumps_overlap_compute_on_a_slow_disk(tmp_path):
    # a simulated 60 ms disk per snapshot: with the synchronous writer (depth 0) the steps
    # wait for every write; with a queue (depth 4) dpd_step returns after the compute alone
    # and the writes finish behind it (drained at close)
    cfg = workloads.with_box(workloads.CONFIGS["eq64"], (48.0, 48.0, 48.0))
    res = {}
    for depth in (0, 4):
        capi, d = new(cfg)
        d.step(5)  # warm up
        d.dump_open(str(tmp_path / f"d{depth}"), depth)
        d.set_option("dump_delay_us", 60000)
        d.dump_every(10)
        t0 = time.perf_counter()
        d.step(30)  # 3 snapshots
        t_step = time.perf_counter() - t0
        t0 = time.perf_counter()
        assert d.dump_close() == 3
        res[depth] = (t_step, time.perf_counter() - t0)
    assert res[0][0] >= 0.18, res  # 3 x 60 ms inside the steps
    assert res[4][0] < 0.12, res  # the steps did not wait for the disk
    assert res[4][1] >= 0.06, res  # the writes were still pending: drained at close


def test_step_schedule_decomposed():
    """The step graph of a decomposed context (what the NCCL path runs; printed from a member
    of an in-process group, whose contexts are split the same way): the ghost exchange and the
    ghost pack, exchange, binning and the halo forces are issued on the communication stream
    before / beside the local forces, so they overlap them; the step ends
    with a join of both streams."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (12.0, 12.0, 12.0))
    ctxs = capi.dpd_create_group(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, (2, 1, 1))
    try:
        sched = capi.dpd_step_schedule(ctxs[0])
        names = [t[1] for t in sched]
        assert names == ["kick_drift_bin", "migrate_exchange", "scan_scatter", "ghost_pack", "ghost_exchange",
                         "ghost_sort", "force_local", "halo_force", "join"]
        slot = {t[1]: t[0] for t in sched}
        preds = {t[1]: set(t[2]) for t in sched}
        comm = ("ghost_pack", "ghost_exchange", "ghost_sort", "halo_force")
        assert all(slot[k] == 1 for k in comm)
        assert all(slot[k] == 0 for k in names if k not in comm)
        assert preds["ghost_sort"] == {"ghost_exchange"} and preds["ghost_exchange"] == {"ghost_pack"}
        assert preds["ghost_pack"] == {"scan_scatter"}
        assert preds["halo_force"] == {"ghost_sort"}
        assert preds["join"] == {"force_local", "halo_force"}
        assert preds["force_local"] == {"scan_scatter"}
    finally:
        for c in ctxs:
            capi.dpd_destroy(c)
