#!/bin/bash
# Round-2 final profile set (after the sampler prologue, the cluster filter and the small-kernel latency fixes):
# bench line, reference arm, small-config device times (graph loop), launch lists per config
# (ncu default: caches flushed before every launch) and, for c1 / c2, a second launch list with
# --cache-control none (warm L2, as inside the graph loop).
set -x
O=gpurun_out/r02e
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 python scripts/small_time.py > $O/small_time.txt 2>&1
SHAPES=2048x128,2048x88,2048x64,2048x240 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_trinv --csv python scripts/w_bench.py > $O/trinv_launches.csv 2> /dev/null
timeout 60 ./scripts/mb_trinv1 > $O/mb_trinv1.txt 2>&1
timeout 60 ./scripts/mb_lat > $O/mb_lat.txt 2>&1
timeout 60 ./scripts/mb_chol > $O/mb_chol.txt 2>&1
for c in c5 c4 c3 c2 c1; do
  CFG=$c timeout 600 python scripts/prof_cfg.py > $O/plain_$c.log 2>&1 &&
  CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_$c.csv python scripts/prof_cfg.py > $O/launches_$c.log 2>&1
done
for c in c2 c1; do
  CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file $O/launches_warm_$c.csv python scripts/prof_cfg.py > $O/launches_warm_$c.log 2>&1
done
echo done
