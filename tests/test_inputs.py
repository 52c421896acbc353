"""Host logic: seeded counter-based input generator and config registry (no method arithmetic)."""
import numpy as np

from paper_2002_08110_b200 import configs, inputs


def test_splitmix64_reference_value():
    # first output of the reference splitmix64 stream with state 0
    assert int(inputs.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_uniform_range_and_determinism():
    u = inputs.uniform01(7, np.arange(100000))
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.01
    assert np.array_equal(u, inputs.uniform01(7, np.arange(100000)))
    assert not np.array_equal(u, inputs.uniform01(8, np.arange(100000)))


def test_subset_consistency():
    for name in ("2d", "4d"):
        cfg = configs.CONFIGS[name]
        spec = cfg["spec"]
        seed = configs.seed_of(name)
        full = inputs.full_vector(spec, cfg["recipe"], seed) if name == "2d" else None
        ids = np.array([0, 3, 17, 63])
        sub = inputs.cell_values(spec, cfg["recipe"], seed, ids)
        if full is not None:
            nd = (spec["k"] + 1) ** 2
            assert np.array_equal(sub, full.reshape(-1, nd)[ids])
        again = inputs.cell_values(spec, cfg["recipe"], seed, ids[::-1])
        assert np.array_equal(again[::-1], sub)


def test_time_steps_reading_c12():
    exp = {"2d": 5.208e-4, "3d": 6.25e-5, "4d": 1.5625e-4, "5d": 5.025e-4, "6d": 4.216e-4}
    for name, cfg in configs.CONFIGS.items():
        dt = configs.time_step(cfg["spec"], cfg["cfl"])
        assert abs(dt - exp[name]) < 1e-3 * exp[name] + 1e-7, (name, dt)


def test_neighbour_ids_periodic():
    spec = configs.CONFIGS["2d"]["spec"]
    nb = inputs.neighbour_ids(spec, np.array([0, 9, 63]))
    assert list(nb[0]) == [7, 1, 56, 8]
    assert list(nb[1]) == [8, 10, 1, 17]
    assert list(nb[2]) == [62, 56, 55, 7]
