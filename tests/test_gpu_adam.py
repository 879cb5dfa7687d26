"""Dense Adam (nif_adam_dev) is bit-exact to the reference's update
(grids.py:31-56 / mlp.py:126-129, restated in oracle.adam_update) on
adversarial states: zero and signed-zero gradients and moments, float
denormals, large values, step counts on both sides of numba's integer-power
cut-over (0x10000), touched and untouched objects, both families."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _state(rng, n):
    """params / grad / m / v: fp32 arrays mixing the special cases."""
    out = []
    for kind in range(4):
        a = rng.normal(0, 1, n).astype(np.float32)
        sel = rng.random(n)
        a[sel < 0.25] = 0.0
        a[(sel >= 0.25) & (sel < 0.3)] = -0.0
        a[(sel >= 0.3) & (sel < 0.35)] = np.float32(1e-40) * rng.choice([-1, 1])  # denormal
        a[(sel >= 0.35) & (sel < 0.4)] = np.float32(3e-38)
        a[(sel >= 0.4) & (sel < 0.42)] = np.float32(1e20)
        if kind == 3:  # v is a second moment: non-negative
            a = np.abs(a)
        out.append(a)
    return out


@pytest.mark.parametrize("which", ["outer", "inner"])
def test_adam_bit_exact(which, cuda):
    import torch
    from oracle.oracle import Adam, adam_update
    from paper_2306_07191_b200 import _lib
    from paper_2306_07191_b200.nif import NifConfig, NifModel
    cfg = NifConfig(seed=3)
    cfg.outer.grid_resolution = 32
    cfg.inner.grid_resolution = 32
    cfg.inner.dist_resolution = 32
    n_obj = 4
    m = NifModel(cfg, n_obj)
    fam = m.family(which)
    rng = np.random.default_rng(5 if which == "outer" else 6)
    p0, g0, m0, v0 = _state(rng, fam.numel)
    for t, a in ((fam.params, p0), (fam.grad, g0), (fam.m, m0), (fam.v, v0)):
        t.copy_(torch.from_numpy(a))
    steps = np.array([0, 6, 0x10000 + 3, 123], np.int64)
    touched = np.array([1, 1, 1, 0], np.int32)
    fam.grid_steps.copy_(torch.from_numpy(steps))
    fam.mlp_steps.fill_(41)
    fam.counts.copy_(torch.from_numpy(touched))
    a = cfg.adam
    _lib.lib().nif_adam_dev(fam.view(), fam.train_view(), m.learning_rate, a.beta1, a.beta2,
                            a.epsilon, _lib.stream_ptr(None))
    torch.cuda.synchronize()
    got = [t.cpu().numpy() for t in (fam.params, fam.grad, fam.m, fam.v)]
    want = [x.copy() for x in (p0, g0, m0, v0)]
    keys = ["pos", "dir"] + (["dist"] if which == "inner" else [])
    for key in keys:
        off, size = fam.offsets[key]
        per = size // n_obj
        for o in range(n_obj):
            if not touched[o]:
                continue
            sl = slice(off + o * per, off + (o + 1) * per)
            adam_update(want[0][sl], want[1][sl], want[2][sl], want[3][sl],
                        Adam(m.learning_rate, a.beta1, a.beta2, a.epsilon, int(steps[o])))
    for key in ("w", "b"):  # shared MLP: one update per step
        off, size = fam.offsets[key]
        sl = slice(off, off + size)
        adam_update(want[0][sl], want[1][sl], want[2][sl], want[3][sl],
                    Adam(m.learning_rate, a.beta1, a.beta2, a.epsilon, 41))
    for name, g, w in zip(("params", "grad", "m", "v"), got, want):
        bad = np.flatnonzero(g.view(np.uint32) != w.view(np.uint32))
        assert bad.size == 0, (name, bad[:5], g[bad[:5]], w[bad[:5]])
    assert fam.grid_steps.cpu().numpy().tolist() == (steps + touched).tolist()
