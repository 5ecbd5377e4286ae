#!/bin/bash
# c2 DRAM bytes per launch (ncu) and time (tune.py) for each L2 hint mode
mkdir -p gpurun_out/l2
for h in "$@"; do
  GETT_WS_L2HINT=$h timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:dgett_ws --launch-skip 3 --launch-count 1 --csv --log-file gpurun_out/l2/h$h.csv python tools/run_one.py c2 4 > /dev/null 2>&1
  rd=$(grep dram__bytes_read gpurun_out/l2/h$h.csv | tail -1 | awk -F'","' '{print $(NF-1), $NF}' | tr -d '"')
  wr=$(grep dram__bytes_write gpurun_out/l2/h$h.csv | tail -1 | awk -F'","' '{print $(NF-1), $NF}' | tr -d '"')
  t=$(GETT_WS_L2HINT=$h python tools/tune.py c2 | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['ms'], d['kernel'])")
  echo "hint $h read $rd write $wr time_ms $t"
done
