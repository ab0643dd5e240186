"""The pipelined multi-layer API gives the same (Q, T) as one call per layer (it only reorders
copies and solves across layers on two streams)."""
import pytest
import torch

import synthetic
import paper_2501_12956_b200 as g
from paper_2501_12956_b200.pipeline import quantize_layers

pytestmark = pytest.mark.gpu


def test_pipeline_matches_sequential_calls():
    m, n, p, nbits = 96, 256, 2048, 3
    layers = [(synthetic.make_weights(m, n, seed=40 + k).pin_memory(),
               synthetic.make_activations(p, n, seed=50 + k).pin_memory()) for k in range(3)]
    outs = quantize_layers(layers, nbits, 3)
    for (W, X), (Qh, Th) in zip(layers, outs):
        Q, T = g.quantize_layer(W.cuda(), g.hessian(X.cuda()), nbits, 3)
        assert torch.equal(Q.cpu(), Qh) and torch.equal(T.cpu(), Th)


def test_pipeline_checkpoint_resume(tmp_path):
    m, n, p, nbits = 64, 128, 1024, 2
    layers = [(synthetic.make_weights(m, n, seed=60 + k).pin_memory(),
               synthetic.make_activations(p, n, seed=70 + k).pin_memory()) for k in range(4)]
    ref = quantize_layers(layers, nbits, 2, checkpoint_dir=str(tmp_path))
    files = sorted(f.name for f in tmp_path.iterdir())
    assert files == [f"layer_{k:05d}.pt" for k in range(4)]
    (tmp_path / "layer_00002.pt").unlink()  # layer 2 is re-solved, the others are loaded
    again = quantize_layers(layers, nbits, 2, checkpoint_dir=str(tmp_path))
    for (Q0, T0), (Q1, T1) in zip(ref, again):
        assert torch.equal(Q0, Q1) and torch.equal(T0, T1)
    with pytest.raises(ValueError, match="n_bits"):
        quantize_layers(layers, 3, 2, checkpoint_dir=str(tmp_path))  # stale checkpoints are refused


@pytest.mark.parametrize("nbits", [3, 4])
def test_stacked_rows_equal_separate_calls(nbits):
    """q/k/v-style linears sharing one H: the stacked solve is bit-identical per block."""
    n, p = 256, 2048
    Ws = [synthetic.make_weights(mi, n, seed=80 + mi).cuda() for mi in (96, 40, 33)]
    H = g.hessian(synthetic.make_activations(p, n, seed=90).cuda())
    outs = g.quantize_stacked(Ws, H, nbits, 4)
    for W, (Qs, Ts) in zip(Ws, outs):
        Q, T = g.quantize_layer(W, H, nbits, 4)
        assert torch.equal(Q, Qs) and torch.equal(T, Ts)
    outs_k = g.quantize_stacked(Ws, H, nbits, 2, init="kmeans")
    Q, T = g.quantize_layer(Ws[1], H, nbits, 2, init="kmeans")
    assert torch.equal(Q, outs_k[1][0]) and torch.equal(T, outs_k[1][1])
