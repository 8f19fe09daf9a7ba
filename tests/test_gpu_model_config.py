"""The native model object for any ModelConfig (engine.hpp:30-78) and either
optimizer (engine.hpp:80, 268-311) against the reference (oracle/_ref):

* init_model(cfg, seed) bit-identical (host, no device) — small and large
  presets;
* the large preset (base 32, heads 32/16/8/4/1, head_dim 12: Q/K widths up
  to 384, the projection's global-scratch backward) wires up near identity
  (test_engine.cpp:240-250) and its loss step matches run_loss_step;
* the diffeomorphic model (scaling-and-squaring residuals) and plain SGD
  pairwise optimisations match pairwise_optimize step by step."""
import numpy as np
import pytest
import torch

from _util import rel_norm
from paper_2403_16526_b200 import ops

LARGE = dict(base=32, heads=(32, 16, 8, 4, 1), hd=12)


def cfg_of(base=8, heads=(8, 4, 2, 1, 1), hd=6, diffeomorphic=False, ss_steps=7):
    return ops.model_config(base_channels=base, heads_per_level=heads, head_dim=hd,
                            diffeomorphic=diffeomorphic, ss_steps=ss_steps)


@pytest.mark.parametrize("kw", [{}, LARGE, dict(diffeomorphic=True, ss_steps=5)])
def test_init_model_cfg_bit_exact(ref, kw):
    packed, sizes = ref.model_params_cfg(31, **kw)
    ours = ops.init_model_cfg(cfg_of(**kw), 31)
    assert [t.numel() for t in ours] == sizes
    assert np.array_equal(np.concatenate([t.numpy() for t in ours]), packed)


def _split_dev(packed, sizes):
    out, o = [], 0
    for s in sizes:
        out.append(torch.from_numpy(packed[o:o + s].copy()).cuda())
        o += s
    return out


PRE_NORM = {8 * k + i for k in range(5) for i in (1, 5)}


@pytest.mark.gpu
def test_large_preset_wires_up_and_matches_loss_step(cuda, ref):
    """test_engine.cpp:240-250 (near-identity start, > 3M parameters) and the
    whole loss step (encoder x2, 5-level pyramid with K up to 384, NCC +
    grad_reg, backward) against run_loss_step."""
    dims = (16, 16, 16)
    f, m, _, _, _ = ref.synth_pair(dims, seed=20, max_disp=1.0)
    packed, sizes = ref.model_params_cfg(31, **LARGE)
    assert sum(sizes) > 3_000_000
    loss_r, gp_r, phi_r = ref.loss_step_cfg(f, m, packed, **LARGE)
    nat = ops.NativeModel(_split_dev(packed, sizes), dims, config=cfg_of(**LARGE))
    terms, phi = nat.loss_step(torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda())
    torch.cuda.synchronize()
    phi = phi.cpu().numpy()
    assert np.abs(phi).max() <= 1e-2
    assert abs(float(terms[0]) - loss_r) <= 1e-4 * abs(loss_r) + 1e-6
    assert rel_norm(phi, phi_r) <= 1e-3
    o = 0
    for i, (g, s) in enumerate(zip(nat.grads, sizes)):
        b = gp_r[o:o + s]
        o += s
        if i in PRE_NORM or np.linalg.norm(b) == 0:
            continue
        assert rel_norm(g.cpu().numpy().ravel(), b) <= 1e-3, (i, rel_norm(g.cpu().numpy().ravel(), b))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["diffeomorphic_adam", "sgd"])
def test_config_and_optimizer_po_matches_reference(cuda, ref, case):
    dims = (16, 16, 16)
    f, m, lf, lm, _ = ref.synth_pair(dims, seed=16, max_disp=1.0)
    kw = dict(diffeomorphic=True, ss_steps=7) if case == "diffeomorphic_adam" else {}
    opt = "sgd" if case == "sgd" else "adam"
    iters = 10 if opt == "adam" else 3
    packed, sizes = ref.model_params_cfg(23, **kw)
    loss_r, dice_r, phi_r = ref.pairwise_optimize_cfg(f, m, lf, lm, packed, iters, lam=0.5,
                                                      optimizer=opt, **kw)
    nat = ops.NativeModel(_split_dev(packed, sizes), dims, config=cfg_of(**kw), optimizer=opt,
                          loss=ops.LossConfig(lam=0.5, ncc_window=9))
    loss_g, dice_g, phi_g = nat.pairwise_optimize(
        torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda(), iters, lr=1e-4,
        labels_fixed=torch.from_numpy(lf).cuda(), labels_moving=torch.from_numpy(lm).cuda())
    print(case, "loss", loss_g, loss_r, "dice", dice_g, dice_r)
    for a, b in zip(loss_g, loss_r):
        assert abs(a - b) <= 1e-4 * abs(b) + 1e-6, (loss_g, loss_r)
    for a, b in zip(dice_g, dice_r):
        assert abs(a - b) <= 1e-3, (dice_g, dice_r)
    assert rel_norm(phi_g.cpu().numpy(), phi_r) <= 1e-3
