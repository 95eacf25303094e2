#!/bin/bash
# Every BASELINE configuration through bench.py on one GPU, each line with its
# roofline and the CPU oracle beside it; then the reference arm of c1.
# Usage (GPU box): bash tools/config_sweep.sh <out.jsonl>
out=${1:-gpurun_out/config_sweep.jsonl}
: > "$out"
for c in c1 c0 c2 c2net c3_l20 c3_l40 c3_l80 c4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 8 2> gpurun_out/sweep_$c.err | grep '^{' >> "$out"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>> gpurun_out/sweep_ref.err | grep '^{' >> "$out"
