"""Pins of the oracle's SDF walls (P:188-192 frozen layer, P:281-288
bounce-back; reading C-23).  Sources: SPEC.md's bounce_wall examples, its
generate_frozen_layer examples, closed-form signed distances of planes and
cylinders, and invariants (no fluid particle inside the solid after any step, frozen
particles never move)."""
import numpy as np

import oracle

BOX = (10.0, 10.0, 10.0)


def _p(walls, **kw):
    base = dict(box=BOX, rc=1.0, a=25.0, gamma=4.5, kT=1.0, power=0.5, dt=0.1, seed=3, walls=walls)
    base.update(kw)
    return oracle.DPDParams(**base)


PLANE_UP = (1, (0.0, 0.0, 1.0, 5.0), (0.0, 0.0, 0.0))  # solid where z > 5


def test_plane_bounce_spec_example():
    # crossing the plane from 0.1 below to 0.1 above at v = (0, 0, 2): placed at the
    # plane (fluid side), v = (0, 0, -2)
    p = _p([PLANE_UP])
    x = np.array([[3.0, 3.0, 4.9]])
    v = np.array([[0.0, 0.0, 2.0]])
    xn, un, nb = oracle.kick_drift(p, x, v, np.zeros((1, 3)), 0.05)
    assert nb == 1
    assert xn[0, 2] <= 5.0 and 5.0 - xn[0, 2] < 1e-12
    np.testing.assert_allclose(xn[0, :2], [3.0, 3.0])
    np.testing.assert_allclose(un[0], [0.0, 0.0, -2.0])


def test_moving_wall_bounce_spec_example():
    # same crossing with the wall moving at u_w = (1, 0, 0): v -> 2 u_w - v = (2, 0, -2)
    p = _p([(1, (0.0, 0.0, 1.0, 5.0), (1.0, 0.0, 0.0))])
    xn, un, nb = oracle.kick_drift(p, np.array([[3.0, 3.0, 4.9]]), np.array([[0.0, 0.0, 2.0]]), np.zeros((1, 3)),
                                   0.05)
    assert nb == 1
    np.testing.assert_allclose(un[0], [2.0, 0.0, -2.0])


def test_no_crossing_is_plain_kick_drift():
    # a particle ending with s < 0 is untouched by the bounce
    p = _p([PLANE_UP])
    pw = _p(None)
    rng = np.random.default_rng(1)
    x = rng.random((50, 3)) * np.array([10.0, 10.0, 4.0])
    v = rng.normal(size=(50, 3))
    F = rng.normal(size=(50, 3))
    xa, ua, nb = oracle.kick_drift(p, x, v, F, 0.05)
    xb, ub, _ = oracle.kick_drift(pw, x, v, F, 0.05)
    assert nb == 0
    assert np.array_equal(xa, xb) and np.array_equal(ua, ub)


def test_signed_distances_closed_form():
    pipe = (4, (5.0, 5.0, 3.0, -1.0), (0.0, 0.0, 0.0))   # solid outside radius 3 about the z axis at (5, 5)
    post = (2, (2.0, 8.0, 1.0, 1.0), (0.0, 0.0, 0.0))    # solid inside radius 1 about the x axis at (y, z) = (2, 8)
    s, _ = oracle.wall_sdf(_p([pipe]), [[5.0, 5.0, 1.0], [9.0, 5.0, 7.0], [5.0, 8.0, 0.0]])
    np.testing.assert_allclose(s, [-3.0, 1.0, 0.0], atol=1e-12)
    s, _ = oracle.wall_sdf(_p([post]), [[0.0, 2.0, 8.0], [7.0, 2.0, 10.0], [4.0, 2.5, 8.0]])
    np.testing.assert_allclose(s, [1.0, -1.0, 0.5], atol=1e-12)
    # union of two solids = max; the wall velocity is the maximising primitive's
    lo = (1, (0.0, 0.0, -1.0, -1.0), (1.0, 0.0, 0.0))    # solid z < 1, moving +x
    hi = (1, (0.0, 0.0, 1.0, 9.0), (-1.0, 0.0, 0.0))     # solid z > 9, moving -x
    s, uw = oracle.wall_sdf(_p([lo, hi]), [[0.0, 0.0, 0.5], [0.0, 0.0, 5.0], [0.0, 0.0, 9.75]])
    np.testing.assert_allclose(s, [0.5, -4.0, 0.75], atol=1e-12)
    np.testing.assert_allclose(uw[:, 0], [1.0, 1.0, -1.0])


def test_frozen_layer_count_and_carve():
    # plane wall, rho = 8 -> frozen count ~ rho Lx Ly r_c (+-5 %); removed beyond r_c;
    # afterwards no fluid particle has s > 0
    box = (20.0, 20.0, 16.0)
    wall = (1, (0.0, 0.0, -1.0, -2.0), (0.5, 0.0, 0.0))  # solid z < 2, moving at (0.5, 0, 0)
    p = _p([wall], box=box)
    rng = np.random.default_rng(7)
    n = int(8 * 20 * 20 * 16)
    x = rng.random((n, 3)) * np.array(box)
    v = rng.normal(size=(n, 3))
    keep, v2, sp, nf = oracle.wall_carve(p, x, v, np.zeros(n, np.int32), 1)
    expect = 8 * 20 * 20 * 1.0
    assert abs(nf - expect) < 0.05 * expect, nf
    s, _ = oracle.wall_sdf(p, x[keep & (sp == 0)][:2000])
    assert np.all(s <= 0.0)
    assert np.all(x[~keep][:, 2] < 1.0)
    frozen = sp == 1
    np.testing.assert_allclose(v2[frozen], np.tile([0.5, 0.0, 0.0], (frozen.sum(), 1)))
    # wall outside the box: nothing frozen, nothing removed
    far = (1, (0.0, 0.0, -1.0, 5.0), (0.0, 0.0, 0.0))   # solid z < -5
    keep, _, sp, nf = oracle.wall_carve(_p([far], box=box), x, v, np.zeros(n, np.int32), 1)
    assert nf == 0 and keep.all()


def test_channel_invariants_over_steps():
    # plane channel 1 < z < 9 with frozen layers: fluid never ends inside the solid, frozen
    # particles never move, over 40 steps of the full GW-VV step with bounce-back
    lo = (1, (0.0, 0.0, -1.0, -2.0), (0.0, 0.0, 0.0))
    hi = (1, (0.0, 0.0, 1.0, 8.0), (0.0, 0.0, 0.0))
    box = (6.0, 6.0, 10.0)
    p = _p([lo, hi], box=box, dt=0.01, frozen_mask=0b10)
    rng = np.random.default_rng(3)
    n = int(3 * 6 * 6 * 10)
    x = rng.random((n, 3)) * np.array(box)
    v = rng.normal(size=(n, 3))
    keep, v, sp, nf = oracle.wall_carve(p, x, v, np.zeros(n, np.int32), 1)
    x, v, sp = x[keep], v[keep], sp[keep]
    assert nf > 0
    p.species = sp
    st = oracle.State(p, x, v)
    frozen = sp == 1
    x0 = st.x[frozen].copy()
    for _ in range(40):
        st.step(1)
        s, _ = oracle.wall_sdf(p, st.x[~frozen])
        assert np.all(s <= 0.0)
    assert np.array_equal(st.x[frozen], x0)
    assert np.all(st.v[frozen] == 0.0)
