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
