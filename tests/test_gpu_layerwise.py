"""GPU: the layer-wise consumer (nn.hpp:156-318 on the B200).  Training through
compressed weights -- decode of layer l+1 overlapped with layer l's GEMM,
recompression after each update -- must be bit-identical to the same
training on raw weights (nn.hpp:8-10), and at most two layer buffers are
live (one decoding, one in the GEMM)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lw():
    import paper_2410_20650_b200 as nz
    from paper_2410_20650_b200 import layerwise

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return layerwise


def _model(dims, seed):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    from paper_2410_20650_b200.layerwise import RawLayer

    return [RawLayer((torch.randn(o, i, device="cuda", generator=g) * 0.05).to(torch.bfloat16),
                     (torch.randn(o, device="cuda", generator=g) * 0.01).to(torch.bfloat16))
            for i, o in zip(dims[:-1], dims[1:])]


@pytest.mark.parametrize("alg1_literal", [False, True])
@pytest.mark.parametrize("decode_ctas", [0, 8])
def test_gpu_layerwise_training_is_bit_identical(lw, alg1_literal, decode_ctas):
    import torch

    dims = [256, 1024, 384, 512, 64]
    raw = lw.RawMlp(_model(dims, 3))
    meter = lw.MemoryMeter()
    comp = lw.CompressedMlp.from_raw([lw.RawLayer(l.weight.clone(), l.bias.clone()) for l in raw.layers],
                                     meter=meter, decode_ctas=decode_ctas)
    g = torch.Generator(device="cuda").manual_seed(9)
    for step in range(3):
        x = (torch.randn(48, dims[0], device="cuda", generator=g)).to(torch.bfloat16)
        t_raw, t_cmp = lw.ActivationTape(), lw.ActivationTape()
        y_raw = raw.forward(x, t_raw)
        y_cmp = comp.forward(x, t_cmp)
        torch.cuda.synchronize()
        assert torch.equal(y_raw.view(torch.int16), y_cmp.view(torch.int16)), step
        gout = (y_raw.float() * 0.01).to(torch.bfloat16)
        raw.backward_and_update(t_raw, gout, 0.05, alg1_literal)
        comp.backward_and_update(t_cmp, gout, 0.05, alg1_literal)
        for w_raw, w_cmp, l_raw, l_cmp in zip([l.weight for l in raw.layers], comp.raw_weights(), raw.layers,
                                              comp.layers):
            assert torch.equal(w_raw.view(torch.int16), w_cmp.view(torch.int16)), step
            assert torch.equal(l_raw.bias.view(torch.int16), l_cmp.bias.view(torch.int16)), step
    largest = max(o * i for i, o in zip(dims[:-1], dims[1:]))
    assert 0 < meter.peak_weight_bytes <= 2 * 2 * largest  # two layer buffers at most
    assert meter.live_weight_bytes == 0 and meter.peak_grads == 1


def test_gpu_layerwise_tape_mismatch_raises(lw):
    import torch

    comp = lw.CompressedMlp.from_raw(_model([32, 64, 16], 1))
    with pytest.raises(ValueError):
        comp.backward_and_update(lw.ActivationTape(), torch.zeros(4, 16, dtype=torch.bfloat16, device="cuda"), 0.1)
