"""Layer-wise on-the-fly consumer of the codec: the
B200 counterpart of the reference's compressed training harness
(nn.hpp:156-318, Alg. 1 of the paper).

Weights live only as compressed device blobs.  A forward pass decodes one
layer at a time into one of two reusable bf16 buffers: layer l+1 is decoded
on a side stream -- by the persistent decode kernel capped to a few SMs
(DecodePlan.set_max_ctas) -- while layer l's GEMM runs on the compute
stream, so the decode hides behind the matmul.  The backward sweep decodes
each layer, forms the gradients, applies SGD and recompresses the layer on
the GPU (LOMO-style, nn.hpp:286-318).  Because the codec is lossless and the
compressed and raw paths run the same GEMM kernels, training is
bit-identical to the uncompressed path (the reference's claim, nn.hpp:8-10);
tests/test_gpu_layerwise.py checks exactly that.

Numerics follow nn.hpp's contract (bf16 operands, fp32 accumulation, one
rounding per output element) but on cuBLAS, so they are not bit-identical to
the reference's CPU loop order -- only compressed-vs-raw is.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional

from .codec import DecodePlan, DeviceBlob, TensorMeta, kLosslessPrecision


class Activation(Enum):  # nn.hpp:29
    None_ = 0
    Relu = 1


@dataclass
class MemoryMeter:
    """Live-buffer accounting (nn.hpp:156-197): uncompressed weight buffers
    and gradient buffers, and the compressed bytes resident."""
    live_weight_bytes: int = 0
    peak_weight_bytes: int = 0
    blob_bytes: int = 0
    live_grads: int = 0
    peak_grads: int = 0

    def on_weight_alloc(self, b):
        self.live_weight_bytes += b
        self.peak_weight_bytes = max(self.peak_weight_bytes, self.live_weight_bytes)

    def on_weight_free(self, b):
        self.live_weight_bytes -= b

    def on_grad_alloc(self):
        self.live_grads += 1
        self.peak_grads = max(self.peak_grads, self.live_grads)

    def on_grad_free(self):
        self.live_grads -= 1

    def on_blob_bytes(self, old, new):
        self.blob_bytes += new - old


@dataclass
class LinearLayer:  # nn.hpp:200-207: weight only in compressed form
    weight: DeviceBlob  # shape (out_dim, in_dim)
    bias: object        # torch bf16 (out_dim,), kept raw

    @property
    def out_dim(self):
        return self.weight.meta.shape[0]

    @property
    def in_dim(self):
        return self.weight.meta.shape[1]


@dataclass
class RawLayer:  # nn.hpp:215-218
    weight: object  # torch bf16 (out, in)
    bias: object


@dataclass
class ActivationTape:  # nn.hpp:249-252
    inputs: list = field(default_factory=list)


def _linear(x, w, b):
    """nn.hpp:51-68 on cuBLAS: y = x w^T + b, bf16 in, fp32 accumulate."""
    import torch

    return torch.addmm(b, x, w.t())


def _relu_(x):
    x.clamp_(min=0)


def _sgd(w, g, lr):
    """nn.hpp:118-127: w = bf16(float(w) - lr * float(g))."""
    import torch

    return (w.float() - lr * g.float()).to(torch.bfloat16)


class _SmTarget:
    """While the decode is capped to `ctas` SMs, ask cuBLAS to size its GEMMs
    for the remaining SMs (cublasSetSmCountTarget on torch's handle), so the
    two kernels actually run side by side instead of taking turns."""
    _lib = None

    def __init__(self, ctas: int):
        self.ctas = ctas

    def __enter__(self):
        if not self.ctas:
            return self
        import ctypes as C

        import torch

        if _SmTarget._lib is None:
            _SmTarget._lib = C.CDLL("libcublas.so.12")
            _SmTarget._lib.cublasSetSmCountTarget.argtypes = [C.c_void_p, C.c_int]
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        self.h = C.c_void_p(torch.cuda.current_blas_handle())
        _SmTarget._lib.cublasSetSmCountTarget(self.h, max(1, sms - self.ctas))
        return self

    def __exit__(self, *a):
        if self.ctas:
            _SmTarget._lib.cublasSetSmCountTarget(self.h, 0)


class CompressedMlp:
    """nn.hpp MlpModel with a double-buffered, overlapped layer decode."""

    def __init__(self, layers: List[LinearLayer], activation=Activation.Relu, meter: Optional[MemoryMeter] = None,
                 decode_ctas: int = 0):
        import torch

        self.layers = layers
        self.activation = activation
        self.meter = meter
        self.decode_ctas = decode_ctas
        maxn = max(l.out_dim * l.in_dim for l in layers)
        self.bufs = [torch.empty(maxn + 64, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
        # high priority: as GEMM CTAs retire, the block scheduler hands the
        # freed SMs to the pending decode CTAs first
        self.side = torch.cuda.Stream(priority=-1)
        self.plans = [None] * len(layers)
        for i in range(len(layers)):
            self._plan(i)
        if meter:
            meter.blob_bytes = sum(l.weight.info.payload_bytes for l in layers)

    @classmethod
    def from_raw(cls, raw: List[RawLayer], activation=Activation.Relu, meter=None, decode_ctas: int = 0):
        blobs = DeviceBlob.compress_batch([r.weight.contiguous() for r in raw], precision=kLosslessPrecision,
                                          metas=[TensorMeta(tuple(r.weight.shape)) for r in raw])
        layers = [LinearLayer(b, r.bias.clone()) for b, r in zip(blobs, raw)]
        return cls(layers, activation, meter, decode_ctas)

    def _plan(self, i):
        l = self.layers[i]
        n = l.out_dim * l.in_dim
        if self.plans[i] is not None:
            self.plans[i].free()
        p = DecodePlan([l.weight], [self.bufs[i % 2][:n]])
        if self.decode_ctas:
            p.set_max_ctas(self.decode_ctas)
        self.plans[i] = p

    def _weight(self, i):
        l = self.layers[i]
        return self.bufs[i % 2][: l.out_dim * l.in_dim].view(l.out_dim, l.in_dim)

    def _meter_alloc(self, i):
        if self.meter:
            self.meter.on_weight_alloc(2 * self.layers[i].out_dim * self.layers[i].in_dim)

    def _meter_free(self, i):
        if self.meter:
            self.meter.on_weight_free(2 * self.layers[i].out_dim * self.layers[i].in_dim)

    def forward(self, x0, tape: Optional[ActivationTape] = None, check: bool = True):
        """nn.hpp:256-268 with layer l+1 decoded beside layer l's GEMM.
        check: read every plan's decode status at the end (one sync each)."""
        import torch

        main = torch.cuda.current_stream()
        sm_target = _SmTarget(self.decode_ctas)
        L = len(self.layers)
        ready = [torch.cuda.Event() for _ in range(L)]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        x = x0
        if tape is not None:
            tape.inputs.clear()
        self.side.wait_stream(main)
        with torch.cuda.stream(self.side):
            self.plans[0].launch(self.side)
            ready[0].record(self.side)
        self._meter_alloc(0)
        for i in range(L):
            if i + 1 < L:  # prefetch: buffer (i+1)%2 is free once layer i-1's GEMM is done
                if i >= 1:
                    self.side.wait_event(free[(i + 1) % 2])
                with torch.cuda.stream(self.side):
                    self.plans[i + 1].launch(self.side)
                    ready[i + 1].record(self.side)
                self._meter_alloc(i + 1)
            if tape is not None:
                tape.inputs.append(x)
            main.wait_event(ready[i])
            with sm_target:
                x = _linear(x, self._weight(i), self.layers[i].bias)
            free[i % 2].record(main)
            self._meter_free(i)
            if i + 1 != L and self.activation == Activation.Relu:
                _relu_(x)
        if check:
            for p in self.plans:
                p.status(main)
        return x

    def backward_and_update(self, tape: ActivationTape, grad_out, lr: float, alg1_literal: bool = False):
        """nn.hpp:275-318: reverse sweep, SGD in place, recompress on the GPU."""
        import torch

        L = len(self.layers)
        if len(tape.inputs) != L:
            raise ValueError("backward: tape does not match model")
        grad = grad_out
        main = torch.cuda.current_stream()
        for i in range(L - 1, -1, -1):
            layer = self.layers[i]
            if i + 1 != L and self.activation == Activation.Relu:
                grad = grad * (tape.inputs[i + 1] > 0)
            self.plans[i].launch(main)
            self.plans[i].status(main)
            self._meter_alloc(i)
            w = self._weight(i)
            if self.meter:
                self.meter.on_grad_alloc()
            gw = (grad.t().float() @ tape.inputs[i].float()).to(torch.bfloat16)
            gb = grad.float().sum(0).to(torch.bfloat16)
            grad_prev = None
            if i > 0 and not alg1_literal:
                grad_prev = (grad.float() @ w.float()).to(torch.bfloat16)
            w_new = _sgd(w, gw, lr)
            layer.bias = _sgd(layer.bias, gb, lr)
            if i > 0 and alg1_literal:
                grad_prev = (grad.float() @ w_new.float()).to(torch.bfloat16)
            old = layer.weight.info.payload_bytes
            layer.weight.free()
            layer.weight = DeviceBlob.compress(w_new.contiguous(), precision=kLosslessPrecision,
                                               meta=TensorMeta((layer.out_dim, layer.in_dim)))
            self._plan(i)
            if self.meter:
                self.meter.on_blob_bytes(old, layer.weight.info.payload_bytes)
                self.meter.on_grad_free()
            self._meter_free(i)
            grad = grad_prev

    def raw_weights(self):
        """Decoded copies of every weight (for checks)."""
        out = []
        for i, l in enumerate(self.layers):
            out.append(l.weight.decompress().view(l.out_dim, l.in_dim))
        return out


class RawMlp:
    """nn.hpp RawMlp: the same math with uncompressed weights."""

    def __init__(self, layers: List[RawLayer], activation=Activation.Relu):
        self.layers = layers
        self.activation = activation

    def forward(self, x0, tape: Optional[ActivationTape] = None):
        x = x0
        if tape is not None:
            tape.inputs.clear()
        for i, l in enumerate(self.layers):
            if tape is not None:
                tape.inputs.append(x)
            x = _linear(x, l.weight, l.bias)
            if i + 1 != len(self.layers) and self.activation == Activation.Relu:
                _relu_(x)
        return x

    def backward_and_update(self, tape: ActivationTape, grad_out, lr: float, alg1_literal: bool = False):
        import torch

        L = len(self.layers)
        if len(tape.inputs) != L:
            raise ValueError("backward: tape does not match model")
        grad = grad_out
        for i in range(L - 1, -1, -1):
            layer = self.layers[i]
            if i + 1 != L and self.activation == Activation.Relu:
                grad = grad * (tape.inputs[i + 1] > 0)
            w = layer.weight
            gw = (grad.t().float() @ tape.inputs[i].float()).to(torch.bfloat16)
            gb = grad.float().sum(0).to(torch.bfloat16)
            grad_prev = None
            if i > 0 and not alg1_literal:
                grad_prev = (grad.float() @ w.float()).to(torch.bfloat16)
            layer.weight = _sgd(w, gw, lr)
            layer.bias = _sgd(layer.bias, gb, lr)
            if i > 0 and alg1_literal:
                grad_prev = (grad.float() @ layer.weight.float()).to(torch.bfloat16)
            grad = grad_prev
