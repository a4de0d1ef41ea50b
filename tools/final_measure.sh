#!/bin/bash
# Round measurement set (GPU box): bench lines (8B lossless/lossy, 70B, the
# reference arm), the ncu launch list and one full capture of a layer launch,
# the C5 chunk sweep and the CPU-vs-GPU codec table.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --precision 3 --steps 10 --warmup 3 --dropin 0 > gpurun_out/f_bench_k3.json 2> gpurun_out/f_bench_k3.err
timeout 900 python bench.py --precision 0 --steps 10 --warmup 3 --dropin 0 > gpurun_out/f_bench_k0.json 2> gpurun_out/f_bench_k0.err
timeout 1500 python bench.py --model 70b --steps 5 --warmup 3 --dropin 0 > gpurun_out/f_bench_70b.json 2> gpurun_out/f_bench_70b.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_persist --csv \
  --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 1 --verify 0 --dropin 0 \
  --e2e-layers 1 > gpurun_out/f_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_persist -s 9 -c 1 \
  -o gpurun_out/f_persist_layer python bench.py --steps 1 --warmup 3 --cpu-seconds 1 --verify 0 --dropin 0 \
  --e2e-layers 1 > gpurun_out/f_ncu_full.log 2>&1
timeout 900 python tools/chunk_sweep.py > gpurun_out/f_chunk_sweep.jsonl 2> gpurun_out/f_chunk_sweep.err
timeout 1200 python tools/codec_table.py > gpurun_out/f_codec_table.jsonl 2> gpurun_out/f_codec_table.err
ls -la gpurun_out/
