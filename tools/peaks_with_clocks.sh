#!/bin/bash
# FP64 / FP32 / tensor peaks microbenchmarks with an nvidia-smi clock record
# sampled every 20 ms while they run (the roofline denominators' provenance).
#   bash tools/peaks_with_clocks.sh OUT_DIR
out=${1:-gpurun_out/peaks}
mkdir -p "$out"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gett_peaks tools/peaks.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gett_mma_rate tools/mma_rate.cu
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active \
  --format=csv -lms 20 > "$out/clocks.csv" &
smi=$!
sleep 0.5
/tmp/gett_peaks > "$out/peaks.jsonl" 2>&1
/tmp/gett_mma_rate > "$out/mma_rate.jsonl" 2>&1
sleep 0.3
kill $smi
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > "$out/device.csv"
