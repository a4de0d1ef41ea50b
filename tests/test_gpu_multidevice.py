"""GPU: one process driving two devices (one host thread per device, as the
SURVEY's multi-GPU driver does).  The decode kernels' shared-memory opt-in is
per (device, function): a process-wide flag would skip it on the second
device and its ~147 KiB persistent launch would fail.  Skipped when fewer
than two GPUs are visible (the round's GPU boxes have one)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_two_devices_from_one_process(port):
    import torch

    import paper_2410_20650_b200 as nz

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs")
    v = port.gaussian_bf16(3, 1 << 22, 0.02)
    results = {}

    def work(dev):
        torch.cuda.set_device(dev)
        d = torch.from_numpy(v.view(np.int16)).cuda(dev)
        (b,) = nz.DeviceBlob.compress_batch([d])
        out = torch.empty(v.size, dtype=torch.bfloat16, device=f"cuda:{dev}")
        plan = nz.DecodePlan([b], [out])
        plan.launch()
        plan.status()
        results[dev] = (torch.equal(out.view(torch.int16), d), b.to_host().stream)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert results[0][0] and results[1][0]
    assert results[0][1] == results[1][1]
