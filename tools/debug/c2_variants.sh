#!/bin/bash
# c2 time (device entry, 20 calls) and DRAM bytes of one launch per library variant
for lib in libgett_b200 libgett_sklast libgett_g8 libgett_sklast8; do
  echo "== $lib"
  GETT_LIB_PATH=paper_2410_06770_b200/$lib.so timeout 120 python -c "
import sys, torch; sys.path.insert(0,'.')
import paper_2410_06770_b200 as g
from paper_2410_06770_b200.device import dgett_device
from paper_2410_06770_b200.workloads import C2
a,b,c=(torch.from_numpy(x).cuda() for x in C2.buffers()); pos,kw=C2.args(a,b,c)
for _ in range(3): dgett_device(*pos,**kw)
torch.cuda.synchronize(); e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): dgett_device(*pos,**kw)
e1.record(); torch.cuda.synchronize(); print('ms', e0.elapsed_time(e1)/20, g.last_kernel())
"
  GETT_LIB_PATH=paper_2410_06770_b200/$lib.so timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:dgett_ws --launch-skip 3 --launch-count 1 --csv python tools/run_one.py c2 4 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print $(NF-2), $(NF)}'
done
