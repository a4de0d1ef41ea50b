"""GPU parity at the benchmark's own scale and on its own path (SURVEY.md
§8(c): "configs 2 and 4 check a deterministic tensor sample (all tensors of
layers 0 and L/2 + embed + a norm) against the oracle").

Llama-3-8B layers 0 and 16 (7 projections + 2 RMSNorms each) and the
embedding (128,256 x 4,096 = 525,336,576 elements) are generated with the
reference's own RNG (rng::gaussian_bf16(derive(42, tensor_index), n, 0.02),
rng.hpp:35-81; norms = 1.0), compressed with nzgpu_compress_batch (one batch
per layer, as bench.py does) and decoded through one grouped DecodePlan per
layer, alternating two CUDA streams as the bench's timed steps do.  Every
section (table, serialized stream, sign/mantissa plane, scales) and every
decoded tensor is compared with the reference codec (oracle/_ref: the
unmodified reference headers; the C restatement where it is not built):
compress_lossless / decompress_lossless (tensorstore.hpp:87-125) and
compress_lossy / decompress_lossy (tensorstore.hpp:141-238), k in {3, 0},
B = 512.  A Llama-3-70B-sized embedding (1,050,673,152 elements, > 2^30, so
2.1 GB of bf16: byte offsets past 2^31) is checked lossless the same way.
"""
import concurrent.futures as cf
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, F, KV, VOCAB = 4096, 14336, 1024, 128256
LAYER = [("q_proj", (H, H)), ("k_proj", (KV, H)), ("v_proj", (KV, H)), ("o_proj", (H, H)),
         ("gate_proj", (F, H)), ("up_proj", (F, H)), ("down_proj", (H, F)),
         ("input_layernorm", (H,)), ("post_attention_layernorm", (H,))]


def _numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return nz


@pytest.fixture(scope="module")
def checker():
    from oracle.oracle import Oracle, ref_available

    return Oracle("ref") if ref_available() else Oracle("port")


@pytest.fixture(scope="module")
def groups(port):
    """[(group name, [(tensor name, shape, host bf16 bits)])] in bench.py's
    tensor numbering (layer L tensor t = 9L + t; embed = 288)."""
    out = []
    for layer in (0, 16):
        ts = []
        for t, (name, shape) in enumerate(LAYER):
            n = _numel(shape)
            if len(shape) == 1:
                v = np.full(n, 0x3F80, np.uint16)
            else:
                v = port.gaussian_bf16_parallel(port.derive(42, 9 * layer + t), n, 0.02)
            ts.append((f"layer{layer}.{name}", shape, v))
        out.append((f"layer{layer}", ts))
    emb = port.gaussian_bf16_parallel(port.derive(42, 288), VOCAB * H, 0.02)
    out.append(("embed_tokens", [("embed_tokens", (VOCAB, H), emb)]))
    return out


def _decode_groups(nz, torch, blob_groups):
    """One grouped plan per group, plans alternating two streams (bench.py's
    schedule); distinct outputs so every tensor can be read back."""
    s0 = torch.cuda.current_stream()
    s1 = torch.cuda.Stream()
    s1.wait_stream(s0)
    plans, outs = [], []
    for k, bs in enumerate(blob_groups):
        o = [torch.empty(b.n, dtype=torch.bfloat16, device="cuda") for b in bs]
        p = nz.DecodePlan(bs, o)
        s1.wait_stream(s0)  # outputs were allocated on s0
        p.launch(s0 if k % 2 == 0 else s1)
        plans.append(p)
        outs.append(o)
    s0.wait_stream(s1)
    for p in plans:
        p.status(s0)
    torch.cuda.synchronize()
    return [[t.view(torch.int16).cpu().numpy().view(np.uint16) for t in o] for o in outs]


def _sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()[:16]


@pytest.mark.parametrize("k", [7, 3, 0])
def test_gpu_llama8b_layers_and_embed_match_reference(nz, checker, groups, k):
    import torch

    dev_groups = [[torch.from_numpy(v.view(np.int16)).cuda() for _, _, v in ts] for _, ts in groups]
    metas = [[nz.TensorMeta(shape) for _, shape, _ in ts] for _, ts in groups]
    blob_groups = [nz.DeviceBlob.compress_batch(d, precision=k, block_size=512, metas=m)
                   for d, m in zip(dev_groups, metas)]
    del dev_groups
    decoded = _decode_groups(nz, torch, blob_groups)

    flat = [(name, v, b, out) for (_, ts), bs, outs in zip(groups, blob_groups, decoded)
            for (name, _, v), b, out in zip(ts, bs, outs)]
    assert len(flat) == 19

    def check(item):
        name, v, b, out = item
        host = b.to_host()
        if k == 7:
            f, s, m = checker.compress_lossless(v)
            sec = host.stream == s and (host.freqs == f).all() and (host.signmant == m).all()
            want = checker.decompress_lossless(f, s, m, v.size)
            assert (want == v).all()
        else:
            f, sc, s, pk = checker.compress_lossy(v, k, 512)
            sec = (host.stream == s and (host.freqs == f).all() and (host.signmant == pk).all()
                   and (host.scales == sc).all())
            want = checker.decompress_lossy(f, sc, s, pk, k, 512, v.size)
        return name, bool(sec), bool((out == want).all()), _sha(host.stream), _sha(out.view(np.uint8))

    with cf.ThreadPoolExecutor(8) as ex:
        res = list(ex.map(check, flat))
    bad = [(n, s, d) for n, s, d, _, _ in res if not (s and d)]
    for n, _, _, ss, so in res:
        print(f"k={k} {n}: stream {ss} decoded {so}")
    assert not bad, f"differs from the reference codec ({checker.kind}): {bad}"


def test_gpu_llama70b_embed_over_2g_elements_lossless(nz, checker, port):
    """1,050,673,152 elements (Llama-3-70B embed/lm_head): the blob's sections
    equal the reference's and the grouped decode returns the input exactly."""
    import torch

    n = VOCAB * 8192
    v = port.gaussian_bf16_parallel(port.derive(42, 720), n, 0.02)
    d = torch.from_numpy(v.view(np.int16)).cuda()
    (b,) = nz.DeviceBlob.compress_batch([d], metas=[nz.TensorMeta((VOCAB, 8192))])
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    p = nz.DecodePlan([b], [out])
    p.launch()
    p.status()
    assert torch.equal(out.view(torch.int16), d)
    del d, out
    host = b.to_host()
    f, s, m = checker.compress_lossless(v)
    assert host.stream == s, "stream differs from the reference"
    assert (host.freqs == f).all() and (host.signmant == m).all()
