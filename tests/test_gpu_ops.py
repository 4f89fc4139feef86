"""Op-level API parity on the GPU (reference test_tensors.py / test_sparse.py strategy):
device ops vs golden vectors from the reference, plus the reference's KATs and contracts."""

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]


@pytest.fixture(scope="module")
def P():
    import paper_2305_17423_b200 as P
    return P


@pytest.fixture(scope="module")
def ops(golden_dir):
    return dict(np.load(golden_dir / "ops.npz"))


def test_dense_ops_vs_reference(P, ops):
    from paper_2305_17423_b200 import ops as D
    y = D.conv2d(ops["conv_x"], P.ConvWeights(ops["conv_w"], ops["conv_b"], 1))
    assert np.abs(y - ops["conv_y"]).max() <= 1e-5
    y, m, v = D.group_norm(ops["gn_x"], 4, ops["gn_gamma"], ops["gn_beta"], 1e-5)
    assert np.abs(m - ops["gn_mean"]).max() <= 1e-6 and np.abs(v - ops["gn_var"]).max() <= 1e-5
    assert np.abs(y - ops["gn_y"]).max() <= 1e-5
    # replay from the reference's cached stats is what sparse GN relies on
    y2 = D.normalize_with_group_stats(ops["gn_x"], ops["gn_mean"], ops["gn_var"], ops["gn_gamma"], ops["gn_beta"])
    assert np.abs(y2 - ops["gn_y"]).max() <= 1e-5
    assert np.abs(D.attention(ops["att_q"], ops["att_k"], ops["att_v"], 0.37) - ops["att_y"]).max() <= 1e-5


def test_conv_kats(P):
    from paper_2305_17423_b200 import ops as D
    x = np.ones((1, 1, 5, 5), np.float32)
    w = P.ConvWeights(np.ones((1, 1, 3, 3), np.float32), np.zeros(1, np.float32), 1)
    y = D.conv2d(x, w)
    assert y[0, 0, 2, 2] == 9.0 and y[0, 0, 0, 0] == 4.0
    g = np.random.default_rng(1)
    x = g.standard_normal((1, 3, 6, 7)).astype(np.float32)
    ident = np.zeros((3, 3, 3, 3), np.float32)
    for c in range(3):
        ident[c, c, 1, 1] = 1
    assert np.array_equal(D.conv2d(x, P.ConvWeights(ident, np.zeros(3, np.float32), 1)), x)
    blocks = g.standard_normal((5, 3, 4, 4)).astype(np.float32)
    wt = P.ConvWeights(g.standard_normal((2, 3, 3, 3)).astype(np.float32), np.zeros(2, np.float32), 1)
    out = D.conv2d_valid(blocks, wt)
    for i in range(5):
        full = D.conv2d(blocks[i:i + 1], wt)
        assert np.abs(out[i] - full[0, :, 1:3, 1:3]).max() <= 1e-5


def test_sparse_ops_vs_reference(P, ops):
    from paper_2305_17423_b200 import ops as D
    ctx = P.SparseLayerContext(step=1, layer_id=0, cached_output=ops["sc_cached"])
    mask = P.BinaryMask(ops["sc_mask"])
    plan = P.select_gather_plan(mask, (3, 3))
    y = D.sparse_conv(ops["sc_x"], P.ConvWeights(ops["sc_w"], ops["sc_b"], 1), plan, ctx, mask)
    assert np.abs(y - ops["sc_y"]).max() <= 1e-5
    assert np.array_equal(y[:, :, ~mask.bits], ops["sc_cached"][:, :, ~mask.bits])
    ctx = P.SparseLayerContext(step=1, layer_id=0, cached_output=ops["sg_cached"], cached_mean=ops["sg_mean"],
                               cached_var=ops["sg_var"])
    y = D.sparse_group_norm(ops["sg_x"], ctx, ops["sg_gamma"], ops["sg_beta"], 1e-5, mask)
    assert np.abs(y - ops["sg_y"]).max() <= 1e-5
    assert np.array_equal(y[:, :, ~mask.bits], ops["sg_cached"][:, :, ~mask.bits])
    m3 = P.BinaryMask(ops["sa_mask"])
    ctx = P.SparseLayerContext(step=1, layer_id=0, cached_output=ops["sa_cached"])
    y = D.sparse_self_attention(ops["sa_x"], ops["sa_wq"], ops["sa_wk"], ops["sa_wv"], 0.35, ctx, m3)
    assert np.abs(y - ops["sa_y"]).max() <= 1e-5
    assert np.array_equal(y[:, :, ~m3.bits], ops["sa_cached"][:, :, ~m3.bits])
    yd = D.dense_self_attention(ops["sa_x"], ops["sa_wq"], ops["sa_wk"], ops["sa_wv"], 0.35)
    assert np.abs(yd - ops["sa_dense"]).max() <= 1e-5
    y = D.sparse_cross_attention(ops["sa_x"], ops["ca_tk"], ops["ca_tv"], ops["sa_wq"], 0.35, ctx, m3)
    assert np.abs(y - ops["ca_y"]).max() <= 1e-5
    yd, mp = D.dense_cross_attention(ops["sa_x"], ops["ca_tk"], ops["ca_tv"], ops["sa_wq"], 0.35)
    assert np.abs(yd - ops["ca_dense"]).max() <= 1e-5 and np.abs(mp - ops["ca_map"]).max() <= 1e-6


def test_sparse_degenerates_and_contracts(P):
    from paper_2305_17423_b200 import ops as D
    g = np.random.default_rng(7)
    x = g.standard_normal((1, 8, 16, 16)).astype(np.float32)
    cached = g.standard_normal((1, 8, 16, 16)).astype(np.float32)
    s = 1 / np.sqrt(8)
    wq, wk, wv = [(g.standard_normal((8, 8)) * s).astype(np.float32) for _ in range(3)]
    ctx = P.SparseLayerContext(step=3, layer_id=5, cached_output=cached)
    full = D.sparse_self_attention(x, wq, wk, wv, 0.35, P.SparseLayerContext(3, 5), P.BinaryMask.full(16, 16))
    assert np.abs(full - D.dense_self_attention(x, wq, wk, wv, 0.35)).max() <= 1e-5
    empty = D.sparse_self_attention(x, wq, wk, wv, 0.35, ctx, P.BinaryMask.empty(16, 16))
    assert np.array_equal(empty, cached)
    bits = np.zeros((16, 16), bool)
    bits[5, 9] = True
    one = D.sparse_self_attention(x, wq, wk, wv, 0.35, ctx, P.BinaryMask(bits))
    want = (x[0, :, 5, 9].astype(np.float64) @ wv.astype(np.float64)).astype(np.float32)
    assert np.abs(one[0, :, 5, 9] - want).max() <= 1e-6
    with pytest.raises(P.ContractViolation, match="resolution gate"):
        D.sparse_self_attention(x, wq, wk, wv, 0.35, P.SparseLayerContext(3, 5, resolution_gate=False),
                                P.BinaryMask.full(16, 16))
    w = P.ConvWeights(g.standard_normal((4, 8, 3, 3)).astype(np.float32) / 8, np.zeros(4, np.float32), 1)
    m = P.BinaryMask(g.random((16, 16)) < 0.3)
    with pytest.raises(P.CacheMissError, match="step=3 layer=5"):
        D.sparse_conv(x, w, P.select_gather_plan(m, (3, 3)), P.SparseLayerContext(3, 5), m)
    # full mask without a cache computes on a zero base and matches dense
    fm = P.BinaryMask.full(16, 16)
    out = D.sparse_conv(x, w, P.select_gather_plan(fm, (3, 3)), P.SparseLayerContext(3, 5), fm)
    assert np.abs(out - D.conv2d(x, w)).max() <= 1e-5


@pytest.mark.parametrize("sparsity", [0.05, 0.15, 0.30])
def test_mixed_sparsities_split(P, sparsity):
    """test_sparse.py:355-375 / acceptance criterion 4 on device."""
    from paper_2305_17423_b200 import ops as D
    g = np.random.default_rng(int(sparsity * 100))
    x = g.standard_normal((1, 4, 64, 64)).astype(np.float32)
    w = P.ConvWeights((g.standard_normal((4, 4, 3, 3)) / 6).astype(np.float32), g.standard_normal(4).astype(np.float32), 1)
    cached = g.standard_normal((1, 4, 64, 64)).astype(np.float32)
    mask = P.BinaryMask(g.random((64, 64)) < sparsity)
    out = D.sparse_conv(x, w, P.select_gather_plan(mask, (3, 3)), P.SparseLayerContext(1, 0, cached_output=cached), mask)
    dense = D.conv2d(x, w)
    assert np.abs(out[:, :, mask.bits] - dense[:, :, mask.bits]).max() <= 1e-5
    assert np.array_equal(out[:, :, ~mask.bits], cached[:, :, ~mask.bits])


def test_gather_blocks(P):
    from paper_2305_17423_b200 import ops as D
    g = np.random.default_rng(2)
    x = g.standard_normal((1, 2, 16, 16)).astype(np.float32)
    bits = np.zeros((16, 16), bool)
    bits[7, 7] = True
    plan = P.select_gather_plan(P.BinaryMask(bits), (3, 3))
    b = D.gather_blocks(x, plan)
    (oy, ox), (bh, bw) = plan.origins[0], plan.block
    assert np.array_equal(b[0], x[0, :, oy - 1:oy - 1 + bh, ox - 1:ox - 1 + bw])
    bits = np.zeros((16, 16), bool)
    bits[0, 0] = True
    b = D.gather_blocks(x, P.select_gather_plan(P.BinaryMask(bits), (3, 3)))
    assert (b[0, :, 0, :] == 0).all() and (b[0, :, :, 0] == 0).all()
