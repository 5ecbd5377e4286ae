#!/bin/bash
# On the GPU box (gpurun): the bench line without ncu, then the ncu launch list
# of the same command, then one `ncu --set full` capture per BASELINE config's
# dominant kernel(s).  Outputs under gpurun_out/prof/; summarise here with
# tools/ncu_summary.py (which stamps the library hash).
set -x
mkdir -p gpurun_out/prof
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/prof/bench.jsonl 2> gpurun_out/prof/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/prof/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/prof/ncu_launches.log 2>&1
for cfg in c2 c3 c4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgett_ws --launch-skip 3 \
    --launch-count 1 -o gpurun_out/prof/full_$cfg python tools/run_one.py $cfg 4 > gpurun_out/prof/full_$cfg.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sgett_kr|reduce_t" --launch-skip 6 \
  --launch-count 2 -o gpurun_out/prof/full_c5 python tools/run_one.py c5 4 > gpurun_out/prof/full_c5.log 2>&1
ls -la gpurun_out/prof
