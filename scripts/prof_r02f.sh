#!/bin/bash
# Round-2 closing numbers after the host round-trip changes (report / state through the copy
# kernel, the sampler's own scan for one chunk, no L memset before k_w_small): bench line,
# small-config device times, GPU tests, warm launch lists of c1 / c2.
set -x
O=gpurun_out/r02f
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 300 python scripts/small_time.py > $O/small_time.txt 2>&1
for c in c2 c3; do CFG=$c timeout 200 python scripts/host_time.py >> $O/host_time.txt 2>&1; done
for c in c2 c1; do
  CFG=$c timeout 600 python scripts/prof_cfg.py > $O/plain_$c.log 2>&1 &&
  CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file $O/launches_warm_$c.csv python scripts/prof_cfg.py > $O/launches_warm_$c.log 2>&1
done
echo done
