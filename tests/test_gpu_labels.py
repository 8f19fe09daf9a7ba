"""Label evaluation on the GPU (the north star's Dice gate): nearest-neighbour
label warp and mean Dice vs the reference (metrics.cpp:100-164) on synthetic
label volumes from the reference's own make_synth_pair — both bit-identical
(Dice compared with ==, well inside the 1e-3 gate)."""
import numpy as np
import pytest
import torch

from paper_2403_16526_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,seed", [((32, 28, 24), 1), ((40, 32, 36), 7), ((17, 19, 23), 2)])
def test_warp_labels_and_dice_match_reference(cuda, ref, dims, seed):
    f, m, lf, lm, gt = ref.synth_pair(dims, seed=seed)
    r = np.random.default_rng(seed)
    phis = [gt, np.zeros_like(gt),
            np.ascontiguousarray(gt + r.uniform(-0.7, 0.7, gt.shape).astype(np.float32)),
            np.ascontiguousarray((r.uniform(-3, 3, gt.shape) - 0.5).astype(np.float32))]
    for phi in phis:
        wr = ref.warp_labels(lm, phi)
        wg = ops.warp_labels(torch.from_numpy(lm).cuda(), torch.from_numpy(phi).cuda())
        assert np.array_equal(wg.cpu().numpy(), wr)
        assert ops.mean_dice(torch.from_numpy(lf).cuda(), wg) == ref.mean_dice(lf, wr)


def test_dice_edge_cases(cuda):
    z = torch.zeros(4, 4, 4, dtype=torch.int32, device="cuda")
    assert ops.mean_dice(z, z) == 1.0  # no labels present
    a = z.clone()
    a[0, 0, 0] = 5
    assert ops.mean_dice(a, z) == 0.0
    with pytest.raises(ops.InvalidInput):
        ops.mean_dice(a, z, max_label=3)
