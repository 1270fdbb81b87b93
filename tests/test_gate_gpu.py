"""K1 gate kernel: logits within tolerance of fp32, selection/ranks/counts bit-exact
against the CPU oracle applied to the device's own logits."""

import numpy as np
import pytest
import torch

from oracle import tensor_oracle as TO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,d,E,k", [(1000, 256, 8, 2), (4096, 1024, 16, 2), (777, 2048, 64, 2),
                                     (130, 512, 16, 4), (64, 128, 4, 1)])
def test_gate_topk_matches_oracle(T, d, E, k):
    from paper_2502_02581_b200 import ops

    g = torch.Generator().manual_seed(T + d + E)
    x = torch.randn(T, d, generator=g).bfloat16()
    wg = torch.randn(E, d, generator=g) / d ** 0.5
    wg[:, :] += torch.linspace(-0.5, 0.5, E)[:, None] / d  # mild skew
    idx, w, rank, tc, logits = ops.gate_topk(x.cuda(), wg.cuda(), k, want_logits=True)
    torch.cuda.synchronize()
    lg = logits.cpu().numpy()
    ref_lg = TO.gate_logits(x.float().numpy(), wg.numpy())
    assert np.abs(lg - ref_lg).max() <= 1e-4 * max(1.0, np.abs(ref_lg).max())
    o_idx, o_w, o_rank, o_tc = TO.topk_select(lg, k)
    np.testing.assert_array_equal(idx.cpu().numpy(), o_idx)
    np.testing.assert_array_equal(rank.cpu().numpy(), o_rank)
    np.testing.assert_array_equal(tc.cpu().numpy(), o_tc)
    # weights: device expf vs numpy float32 exp differ by an ulp or two, amplified by the
    # renormalisation -> stated tolerance rtol 2e-6 (selection itself is bit-exact above)
    np.testing.assert_allclose(w.cpu().numpy(), o_w, rtol=2e-6, atol=0)
    assert tc.cpu().numpy().sum() == T * k


def test_topk_ties_pick_lower_expert():
    from paper_2502_02581_b200 import ops

    T, E, k = 200, 16, 2
    lg = np.zeros((T, E), dtype=np.float32)
    lg[:, 5] = 1.0
    lg[::2, 9] = 1.0  # exact tie with expert 5 on even tokens
    idx, w, rank, tc = ops.topk_from_logits(torch.from_numpy(lg).cuda(), k)
    torch.cuda.synchronize()
    o_idx, o_w, o_rank, o_tc = TO.topk_select(lg, k)
    np.testing.assert_array_equal(idx.cpu().numpy(), o_idx)
    assert (idx.cpu().numpy()[::2] == [5, 9]).all()
    assert (idx.cpu().numpy()[1::2] == [5, 0]).all()
    np.testing.assert_array_equal(rank.cpu().numpy(), o_rank)
    np.testing.assert_array_equal(tc.cpu().numpy(), o_tc)
