"""fold_sgd_update on the GPU against its plain definition W <- W - lr * grad (SURVEY §8(c)
reading 17: SGD), evaluated in fp64 on the host: sizes that exercise the
vectorised body and its scalar tail, unaligned (offset) views that take the scalar path,
and the empty update."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,offset", [(1, 0), (3, 0), (4, 0), (1023, 0), (1 << 20, 0), ((1 << 20) + 5, 0),
                                      (4097, 1), (4096, 3)])
def test_sgd_matches_definition(n, offset):
    from paper_1702_02181_b200 import fold
    rng = np.random.default_rng(n + offset)
    p0 = rng.uniform(-1, 1, n + offset).astype(np.float32)
    g0 = rng.uniform(-1, 1, n + offset).astype(np.float32)
    lr = 0.0375
    pt = torch.tensor(p0, device="cuda")[offset:]
    gt = torch.tensor(g0, device="cuda")[offset:]
    fold.sgd_update(pt, gt, lr)
    torch.cuda.synchronize()
    want = p0[offset:].astype(np.float64) - np.float64(np.float32(lr)) * g0[offset:].astype(np.float64)
    got = pt.cpu().numpy().astype(np.float64)
    # one fp32 rounding of the update (with or without a fused multiply-add)
    assert np.max(np.abs(got - want)) <= 2 * np.finfo(np.float32).eps * (1 + np.abs(want).max())
    # the gradient is read-only
    assert np.array_equal(gt.cpu().numpy(), g0[offset:])


def test_sgd_empty_is_noop():
    from paper_1702_02181_b200 import fold
    p = torch.ones(8, device="cuda")
    fold.sgd_update(p[:0], p[:0], 0.5)
    torch.cuda.synchronize()
    assert torch.equal(p, torch.ones(8, device="cuda"))
