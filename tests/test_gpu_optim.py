"""GPU Adam / SGD (engine.hpp:268-311) vs the oracle restatement (bit-pinned to
the reference class in test_oracle.py): bit-identical parameters."""
import numpy as np
import pytest
import torch

from _util import f32
from paper_2403_16526_b200 import ops

pytestmark = pytest.mark.gpu


def test_adam_bit_exact(cuda, oracle):
    r = np.random.default_rng(7)
    value = f32(r.standard_normal(5000))
    grads = [f32(r.standard_normal(5000) * s) for s in (1.0, 0.1, 10.0, 1e-4, 0.0, 3.0)]
    p = torch.from_numpy(value.copy()).cuda()
    opt = ops.AdamOptimizer([p])
    for g in grads:
        opt.step(1e-4, [torch.from_numpy(g).cuda()])
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy(), oracle.adam(value, grads, 1e-4))


def test_sgd_bit_exact(cuda):
    r = np.random.default_rng(8)
    value = f32(r.standard_normal(777))
    g = f32(r.standard_normal(777))
    p = torch.from_numpy(value.copy()).cuda()
    ops.sgd_step([p], [torch.from_numpy(g).cuda()], 0.01)
    torch.cuda.synchronize()
    expect = (value.astype(np.float64) - 0.01 * g.astype(np.float64)).astype(np.float32)
    assert np.array_equal(p.cpu().numpy(), expect)
