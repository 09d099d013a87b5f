"""The seeded input generators produce the scene the DESIGN.md recipe describes."""
import numpy as np

from nbt_inputs import CONFIGS, OCCUPIED, UNKNOWN, FREE, syn_map, rand_map, cycle_deltas


def test_syn_structure():
    n, r_o = 64, 8.0
    m = syn_map(n, r_o, seed=0)
    c = n // 2
    assert m.shape == (n, n, n) and m.dtype == np.uint8
    assert m[c, c, c] == UNKNOWN                        # unknown interior
    assert m[c, c, c + 7] == OCCUPIED                   # shell R_o-2 <= r < R_o
    assert m[c, c, c - 7] == OCCUPIED
    assert m[0, 0, 0] == UNKNOWN                        # beyond 0.45 N of the centre
    table_z = int(c + 0.5 - r_o - 3)                    # inside the 2-voxel slab
    assert (m[table_z, c - 10:c + 10, c - 10:c + 10] == OCCUPIED).mean() > 0.95
    frac = np.bincount(m.ravel(), minlength=3) / m.size
    assert frac[FREE] > 0.3 and frac[UNKNOWN] > 0.3
    assert np.array_equal(m, syn_map(n, r_o, seed=0))
    assert not np.array_equal(m, syn_map(n, r_o, seed=1))


def test_rand_map_fractions():
    m = rand_map(32, 0.3, 0.65, 0.05, seed=1)
    frac = np.bincount(m.ravel(), minlength=3) / m.size
    assert np.allclose(frac, [0.3, 0.65, 0.05], atol=0.01)


def test_configs_table():
    assert CONFIGS["B"].rays_per_id == 1572864
    assert CONFIGS["C'"].rays_per_id == 157286400
    assert CONFIGS["D"].rays_per_id == 78643200


def test_cycle_deltas_in_grid():
    m = syn_map(64, 8.0, seed=0)
    ijk, codes = cycle_deltas(64, (32, 32, 32), 3, m, seed=1)
    assert ijk.shape[1] == 3 and len(ijk) == len(codes)
    assert ((ijk >= 0) & (ijk < 64)).all() and (codes <= 2).all()
