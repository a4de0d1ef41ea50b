"""Regenerates tests/golden/* from the UNMODIFIED reference.

Run in the container where /root/reference is mounted:

    make -C oracle && python tests/golden/make_golden.py

It drives oracle/_ref/libneuzip_ref.so (the reference headers behind a C
shim, see oracle/ref_shim.cpp) over the case catalogue in
tests/golden_cases.py and freezes sizes, SHA-256 digests (and full bytes
for small streams) in golden.json.  It also reproduces the reference's own
checked-in fixture (proj/tests/golden/gaussian_entropy.csv, via
gen_golden.cpp:22-33) and the const16_k7.nzt container that
gen_golden.cpp:34-41 writes but the reference does not check in.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, footprint_total  # noqa: E402
from tests import golden_cases as G  # noqa: E402
from tests import inputs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def main() -> None:
    R = Oracle("ref")
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref (reference headers)",
           "lossless": {}, "coder": {}, "lossy": {}, "tables": {}}

    for name, gen, chunk, mirrors in G.lossless_cases():
        v = gen(R)
        freqs, stream, sm = R.compress_lossless(v, chunk)
        back = R.decompress_lossless(freqs, stream, sm, v.size)
        assert (back == v).all(), name
        rec = {"n": int(v.size), "chunk": chunk, "mirrors": mirrors, "input_sha": sha(v),
               "freqs": freqs.tobytes().hex(), "stream_len": len(stream), "stream_sha": sha(stream),
               "signmant_sha": sha(sm), "footprint": footprint_total(len(stream), v.size)}
        if len(stream) <= 2048:
            rec["stream_hex"] = stream.hex()
        out["lossless"][name] = rec

    for name, gen, mirrors in G.coder_cases():
        x = gen()
        freqs = R.build_table(inputs.counts_of(x))
        stream = R.encode_stream(x, freqs)
        assert (R.decode_stream(stream, freqs, x.size) == x).all(), name
        out["coder"][name] = {"n": int(x.size), "mirrors": mirrors, "input_sha": sha(x),
                              "freqs": freqs.tobytes().hex(), "stream_len": len(stream),
                              "stream_sha": sha(stream)}

    for name, gen, k, block, mirrors in G.lossy_cases():
        v = gen(R)
        freqs, scales, stream, packed = R.compress_lossy(v, k, block)
        back = R.decompress_lossy(freqs, scales, stream, packed, k, block, v.size)
        out["lossy"][name] = {"n": int(v.size), "k": k, "block": block, "mirrors": mirrors,
                              "input_sha": sha(v), "freqs": freqs.tobytes().hex(),
                              "scales_sha": sha(scales), "stream_len": len(stream),
                              "stream_sha": sha(stream), "packed_sha": sha(packed),
                              "decoded_sha": sha(back),
                              "footprint": footprint_total(len(stream), packed.size, scales.size)}
        if v.size <= 4:
            out["lossy"][name]["scales"] = scales.tolist()
            out["lossy"][name]["decoded"] = back.tolist()

    for name, counts in G.table_cases():
        out["tables"][name] = R.build_table(counts).tobytes().hex()

    # Config-1 tensor (4096x4096, seed 42): the headline ratio of BASELINE.md.
    v = R.gaussian_bf16(42, 4096 * 4096)
    freqs, stream, sm = R.compress_lossless(v)
    out["c1_4096sq_seed42"] = {"n": int(v.size), "input_sha": sha(v), "stream_len": len(stream),
                               "stream_sha": sha(stream), "freqs": freqs.tobytes().hex(),
                               "footprint": footprint_total(len(stream), v.size, 0, 2),
                               "ratio": 2 * v.size / footprint_total(len(stream), v.size, 0, 2)}
    for k in (0, 1, 3):
        f2, sc, st, pk = R.compress_lossy(v, k, 512)
        out["c1_4096sq_seed42"][f"lossy_k{k}"] = {
            "stream_len": len(st), "stream_sha": sha(st), "packed_sha": sha(pk), "scales_sha": sha(sc),
            "ratio": 2 * v.size / footprint_total(len(st), pk.size, sc.size, 2)}

    # NZT containers written by the reference (tensorstore.hpp:352-390).
    out["nzt"] = {}
    for name, gen, shape, k, block in G.nzt_cases():
        v = gen(R)
        data = (R.write_nzt_lossless(v, shape) if k == 7 else R.write_nzt_lossy(v, shape, k, block))
        out["nzt"][name] = {"len": len(data), "sha": sha(data), "crc": int.from_bytes(data[-4:], "little")}

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)

    # gen_golden.cpp:22-33 (reference-checked-in gaussian_entropy.csv)
    r = R.entropy_report(R.gaussian_bf16(42, 1 << 20))
    with open(os.path.join(HERE, "gaussian_entropy.csv"), "w") as fh:
        fh.write("sign,%.6g\nexponent,%.6g\nmantissa,%.6g\nideal_ratio,%.6g\nexponent_only_ratio,%.6g\n"
                 % tuple(r))
    # gen_golden.cpp:34-41
    with open(os.path.join(HERE, "const16_k7.nzt"), "wb") as fh:
        fh.write(R.write_nzt_lossless(np.full(16, 0x3F80, np.uint16), [16]))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
