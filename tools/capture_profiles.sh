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
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgett_tc_wide_kernel --launch-skip 3 \
  --launch-count 1 -o gpurun_out/prof/full_sgemm4096 python tools/run_sgemm.py 4096 4 > gpurun_out/prof/full_sgemm4096.log 2>&1
timeout 300 python tools/tune.py c1 c2 c3 c4 c5 sgemm2048 sgemm4096 > gpurun_out/prof/tune.jsonl 2>&1
timeout 300 python tools/debug/c5_modes.py > gpurun_out/prof/c5_modes.txt 2>&1
timeout 300 python tools/debug/c5_host_bound.py > gpurun_out/prof/c5_graph.txt 2>&1
# summarise on the box (the reports exceed what gpurun copies back); keep only c2's report
mkdir -p gpurun_out/prof/json
S="python tools/ncu_summary.py"
GETT_ALG_BYTES=536870912 GETT_ALG_FLOPS=137438953472 $S gpurun_out/prof/full_c2.ncu-rep gpurun_out/prof/json/ncu_dgett_c2.json \
  "c2 DGETT (TMA producer, stream-K, bulk-add epilogue), ncu --set full --clock-control none" > /dev/null
GETT_ALG_BYTES=672661504 GETT_ALG_FLOPS=25769803776 $S gpurun_out/prof/full_c3.ncu-rep gpurun_out/prof/json/ncu_dgett_c3.json \
  "c3 DGETT (TMA producer, stream-K, bulk-add epilogue)" > /dev/null
GETT_ALG_BYTES=769720320 GETT_ALG_FLOPS=220150628352 $S gpurun_out/prof/full_c4.ncu-rep gpurun_out/prof/json/ncu_dgett_c4.json \
  "c4 DGETT (cp.async gathers: 72-row M runs do not tile 128-row boxes; stream-K)" > /dev/null
GETT_ALG_BYTES=106758144 GETT_ALG_FLOPS=4529848320 $S --kernel=sgett_kr gpurun_out/prof/full_c5.ncu-rep gpurun_out/prof/json/ncu_sgett_kr_c5.json \
  "c5 SGETT main kernel (k-run, CTA pairs, mixed tf32+bf16 split, split-K 24); the reduce is ncu_splitk_reduce_c5.json" > /dev/null
$S --kernel=reduce_t gpurun_out/prof/full_c5.ncu-rep gpurun_out/prof/json/ncu_splitk_reduce_c5.json \
  "c5 split-K reduce (transposed partials)" > /dev/null
GETT_ALG_BYTES=268435456 GETT_ALG_FLOPS=137438953472 $S gpurun_out/prof/full_sgemm4096.ncu-rep gpurun_out/prof/json/ncu_sgett_wide_sgemm4096.json \
  "contiguous SGEMM 4096^3 on the wide CTA-pair kernel (3xTF32, SW64 boxes)" > /dev/null
rm -f gpurun_out/prof/full_c3.ncu-rep gpurun_out/prof/full_c4.ncu-rep gpurun_out/prof/full_c5.ncu-rep gpurun_out/prof/full_sgemm4096.ncu-rep
ls -la gpurun_out/prof gpurun_out/prof/json
