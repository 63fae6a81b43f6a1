"""Pins for the oracle's all-pairs force sum, cell list and cell-list timing mode
(eq. 2; readings C-1, C-8, C-9)."""
import numpy as np
import pytest

import oracle
import workloads


def cfg1():
    return oracle.DPDParams(box=(8.0, 8.0, 8.0), a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01, seed=42)


def test_three_particle_brute_force_by_hand():
    # tiny input: F_i is the sum of the two pair forces (eq. 2), each from pair_force
    p = cfg1()
    x = np.array([[1.0, 1.0, 1.0], [1.5, 1.2, 1.0], [0.7, 1.3, 1.4]])
    v = np.array([[0.1, 0.0, -0.2], [0.0, 0.3, 0.0], [-0.4, 0.0, 0.1]])
    F, _, npairs = oracle.forces(p, x, v, step=5)
    assert npairs == 3
    for i in range(3):
        tot = np.zeros(3)
        for j in range(3):
            if i == j:
                continue
            f, hit, _ = oracle.pair_force(p, x[i] - x[j], v[i] - v[j], i, j, 5)
            assert hit
            tot += f
        np.testing.assert_allclose(F[i], tot, rtol=1e-15, atol=1e-13)
    # momentum: sum of forces vanishes
    assert np.abs(F.sum(axis=0)).max() < 1e-12


def test_momentum_conservation_and_pair_count():
    p = cfg1()
    x, v = workloads.make_particles(p.box, 3.0, 1.0)
    F, _, npairs = oracle.forces(p, x, v, step=0)
    # sum F = 0 to fp64 roundoff
    assert np.abs(F.sum(axis=0)).max() < 1e-10 * np.abs(F).sum()
    # pair count ~ N rho (4 pi / 3) r_c^3 / 2 for a uniform fluid (C-17)
    expect = x.shape[0] * 3.0 * (4 * np.pi / 3) / 2
    assert abs(npairs - expect) < 5 * np.sqrt(expect) + 0.03 * expect


def test_translation_and_permutation_invariance():
    # catches minimum-image and index mistakes: a periodic shift of every particle and a
    # relabelling of the storage order (ids kept) leave each particle's force unchanged
    p = cfg1()
    x, v = workloads.make_particles(p.box, 3.0, 1.0)
    x = x.astype(np.float64)
    F, _, _ = oracle.forces(p, x, v, step=3)
    shift = np.array([3.25, 7.5, 0.125])
    xs = np.mod(x + shift, 8.0)
    Fs, _, _ = oracle.forces(p, xs, v, step=3)
    np.testing.assert_allclose(Fs, F, atol=1e-9 * np.abs(F).max())
    perm = np.random.default_rng(3).permutation(x.shape[0])
    Fp, _, _ = oracle.forces(p, x[perm], v[perm], step=3, ids=perm.astype(np.uint32))
    np.testing.assert_allclose(Fp, F[perm], atol=1e-9 * np.abs(F).max())
    # different step -> different random force (xi delta-correlated in time)
    F4, _, _ = oracle.forces(p, x, v, step=4)
    assert np.abs(F4 - F).max() > 1.0


def test_cells_match_direct_floor():
    # per-cell membership matches direct floor recomputation; counts sum to N
    p = cfg1()
    x, _ = workloads.make_particles(p.box, 3.0, 1.0)
    cell, count, start = oracle.cells(p, x)
    assert oracle.grid_dims(p) == (8, 8, 8)
    ic = np.minimum(np.floor(x.astype(np.float64)).astype(np.int64), 7)
    direct = ic[:, 0] + 8 * (ic[:, 1] + 8 * ic[:, 2])
    assert np.array_equal(cell, direct)
    assert count.sum() == x.shape[0]
    assert np.array_equal(np.bincount(cell, minlength=512), count)
    # starts non-decreasing, start[last] = N, exclusive scan of counts
    assert np.all(np.diff(start) >= 0) and start[-1] == x.shape[0] and start[0] == 0
    assert np.array_equal(np.diff(start), count)


def test_cells_general_spacing_and_edges():
    # non-integer cell edge (L=10, r_c=1.2 -> n=8, h=1.25): cell bounds contain the particle
    p = oracle.DPDParams(box=(10.0, 7.0, 9.5), rc=1.2)
    nd = oracle.grid_dims(p)
    assert nd == (8, 5, 7)
    rng = np.random.default_rng(0)
    x = (rng.random((5000, 3)) * np.array(p.box)).astype(np.float32)
    x[0] = [0.0, 0.0, 0.0]
    x[1] = np.nextafter(np.float32(p.box), np.float32(0))  # largest float below L
    cell, count, start = oracle.cells(p, x)
    h = np.array(p.box) / np.array(nd)
    ic = np.stack([cell % nd[0], (cell // nd[0]) % nd[1], cell // (nd[0] * nd[1])], 1)
    lo, hi = ic * h, (ic + 1) * h
    tol = 1e-5
    assert np.all(x >= lo - tol) and np.all(x < hi + tol)
    assert np.all(ic < np.array(nd)) and np.all(ic >= 0)
    assert cell[0] == 0 and cell[1] == (nd[0] * nd[1] * nd[2] - 1)


def test_cells_empty_and_single():
    p = oracle.DPDParams(box=(4.0, 4.0, 4.0))
    cell, count, start = oracle.cells(p, np.zeros((0, 3), np.float32))
    assert count.sum() == 0 and np.all(start == 0)
    cell, count, start = oracle.cells(p, np.array([[0.1, 0.1, 0.1]], np.float32))
    assert cell[0] == 0 and count[0] == 1 and start[-1] == 1


@pytest.mark.parametrize("box,rho,n", [((8.0, 8.0, 8.0), 3.0, None), ((5.0, 6.0, 7.0), 4.0, None),
                                       ((6.0, 6.0, 6.0), 8.0, 200)])
def test_celllist_mode_equals_brute_force(box, rho, n):
    # the cell-list pair set equals the brute-force minimum-image pair set
    p = oracle.DPDParams(box=box, a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01, seed=7)
    x, v = workloads.make_particles(box, rho, 1.0, n=n)
    F, _, npairs = oracle.forces(p, x, v, step=9)
    F2, npairs2 = oracle.forces_celllist(p, x, v, step=9)
    assert npairs == npairs2
    np.testing.assert_allclose(F2, F, rtol=0, atol=1e-11 * max(1.0, np.abs(F).max()))


def test_pair_enumeration_matches_force_count():
    p = cfg1()
    x, v = workloads.make_particles(p.box, 3.0, 1.0)
    quad, flag = oracle.pairs(p, x, step=0, eps=1e-5)
    _, _, npairs = oracle.forces(p, x, v, step=0)
    assert int((flag & 1).sum()) == npairs
    assert np.all(quad[:, 0] < quad[:, 1])
    # words agree with the generator
    for k in range(0, len(quad), 97):
        assert oracle.pair_words(42, 0, int(quad[k, 0]), int(quad[k, 1])) == (int(quad[k, 2]), int(quad[k, 3]))


def test_subset_sum_equals_full_sum():
    # the sampled-parity entry point sums the same pairs as the full brute force
    p = cfg1()
    x, v = workloads.make_particles(p.box, 3.0, 1.0)
    F, allow, _ = oracle.forces(p, x, v, step=2, eps=1e-3)
    sel = np.array([0, 5, 17, 900, x.shape[0] - 1])
    Fs, als = oracle.forces_subset(p, x, v, step=2, sel=sel, eps=1e-3)
    np.testing.assert_allclose(Fs, F[sel], rtol=0, atol=1e-12 * np.abs(F).max())
    np.testing.assert_allclose(als, allow[sel], rtol=1e-12, atol=1e-15)


def test_boundary_window_per_pair():
    # C-12: a pair within eps of r_c gets an allowance; a pair that reaches across a periodic
    # edge uses the wider eps_image window (its fp32 image x_j + L rounds at ulp(L)).  A pair
    # at r = r_c - 5e-6: inside the box it is a boundary pair only for eps > 5e-6; across
    # the x edge it is one for eps_image > 5e-6 whatever eps is.
    p = oracle.DPDParams(box=(8.0, 8.0, 8.0))
    r = 1.0 - 5e-6
    inside = np.array([[3.0, 4.0, 4.0], [3.0 + r, 4.0, 4.0]])
    across = np.array([[0.2, 4.0, 4.0], [0.2 - r + 8.0, 4.0, 4.0]])
    v = np.zeros((2, 3))
    for x, img in [(inside, False), (across, True)]:
        _, a_narrow, _ = oracle.forces(p, x, v, 0, eps=1e-6, eps_image=1e-6)
        _, a_img, _ = oracle.forces(p, x, v, 0, eps=1e-6, eps_image=1e-5)
        _, a_int, _ = oracle.forces(p, x, v, 0, eps=1e-5, eps_image=1e-6)
        assert np.all(a_narrow == 0)
        assert np.all(a_img > 0) == img and np.all(a_int > 0) == (not img)
        # the subset sum and the pair enumeration use the same windows
        _, s_img = oracle.forces_subset(p, x, v, 0, [0, 1], eps=1e-6, eps_image=1e-5)
        np.testing.assert_array_equal(s_img, a_img)
        _, flag = oracle.pairs(p, x, 0, eps=1e-6, eps_image=1e-5)
        assert len(flag) == 1 and bool(flag[0] & 2) == img
