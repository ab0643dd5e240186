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
