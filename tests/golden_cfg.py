"""The small model configuration the golden fixtures were made with
(tests/golden/make_golden.py:small_config), on the package side."""


def small_config(seed=0):
    from paper_2306_07191_b200.nif import NifConfig
    cfg = NifConfig(seed=seed)
    cfg.outer.grid_resolution = 32
    cfg.inner.grid_resolution = 16
    cfg.inner.dist_resolution = 16
    cfg.outer.batch_size = 256
    cfg.inner.batch_size = 512
    return cfg


def perturb_arrays(outer_layers, inner_layers, grids, seed):
    """O(1) latents and biases drawn from one numpy generator in a fixed
    order -- applied identically to the reference model (make_infer.py) and
    the package model (host arrays in NifModel.load_arrays order), so
    both hold bit-identical parameters."""
    import numpy as np
    rng = np.random.default_rng(seed)
    for g in grids:
        for k in ("outer_pos", "outer_dir", "inner_pos", "inner_dir", "inner_dist"):
            g[k][...] = rng.uniform(-1.0, 1.0, g[k].shape).astype(np.float32)
    for heads in (outer_layers, inner_layers):
        for layers in heads:
            for _, b in layers:
                b[...] = rng.uniform(-0.5, 0.5, b.shape).astype(np.float32)


def random_queries(n, n_obj, seed):
    """(kind, obj, coord[n,5]) with edge coordinates mixed in."""
    import numpy as np
    rng = np.random.default_rng(seed)
    kind = rng.integers(0, 2, n)
    obj = rng.integers(0, n_obj, n)
    coord = rng.random((n, 5))
    edges = np.array([0.0, 1.0, 0.5, 1.0 - 2 ** -53, 2 ** -30])
    pick = rng.random((n, 5)) < 0.05
    coord[pick] = rng.choice(edges, int(pick.sum()))
    return kind, obj, coord
