"""The reference's OWN acceptance suite, unmodified, against the drop-in.

oracle/Makefile compiles /root/reference/proj/tests/acceptance.cpp as it
lies (no edits) with the repo's include/neuzip/ headers in front of the
reference's, and links it to libnzgpu.so (oracle/_ref/acceptance_dropin).
So the reference's ten SPEC criteria (acceptance.cpp:385-418) run with
every compress / decompress / table / CRC / NZT call on the B200 --
including criterion 6 ("training-dynamics equivalence"), where the
reference's own CPU training loop (nn.hpp:228-318) decompresses every layer
before use and recompresses it after each update through the drop-in, and
criterion 10, which drives the repo's `neuzip` CLI.  The binary travels to
the GPU box with oracle/_ref; the reference tree itself is not read here."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")


def test_reference_acceptance_suite_passes_on_the_dropin():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/acceptance_dropin not built (reference was not mounted at build time)")
    out = subprocess.run([BIN], cwd=ROOT, capture_output=True, text=True, timeout=1800)
    print(out.stdout)
    lines = [l for l in out.stdout.splitlines() if l.startswith("[")]
    assert len(lines) == 10, out.stdout + out.stderr
    failed = [l for l in lines if not l.startswith("[PASS]")]
    assert not failed and out.returncode == 0, "\n".join(failed) + out.stderr[-2000:]
    assert "all 10 criteria passed" in out.stdout
