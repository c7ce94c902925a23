#!/bin/bash
# Round-2 final profile set: bench line, reference arm, launch lists (eager loop) per config.
# The ncu full captures of r02b stand for the kernels that did not change since
# (k_lhat64 v1 on c5 / c3, k_proj_tc32, k_lhat_paper<32>).
set -x
O=gpurun_out/r02c
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for c in c5 c4 c3 c2 c1; do
  CFG=$c timeout 600 python scripts/prof_cfg.py > $O/plain_$c.log 2>&1 &&
  CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_$c.csv python scripts/prof_cfg.py > $O/launches_$c.log 2>&1
done
echo done
