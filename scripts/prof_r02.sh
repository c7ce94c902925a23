#!/bin/bash
# Round-2 profile set (run under gpurun from the repo root): bench line, reference arm, launch
# lists (eager loop) and ncu full captures of the dominant projection kernels of c5 (fp64
# DMMA, k_lhat_paper) and c4 (fp32 tcgen05, k_proj_tc32).  Every ncu command runs only after
# the same command exited 0 without ncu.
set -x
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for c in c5 c4 c2; do
  CFG=$c timeout 600 python scripts/prof_cfg.py > $O/plain_$c.log 2>&1 &&
  CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_$c.csv python scripts/prof_cfg.py > $O/launches_$c.log 2>&1
done
CFG=c5 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_lhat_paper -s 6 -c 1 \
    -o $O/c5_lhat python scripts/prof_cfg.py > $O/ncu_c5.log 2>&1
CFG=c4 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_proj_tc32 -s 2 -c 1 \
    -o $O/c4_tc32 python scripts/prof_cfg.py > $O/ncu_c4.log 2>&1
CFG=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lhat_paper -s 1 -c 1 \
    -o $O/c2_lhat python scripts/prof_cfg.py > $O/ncu_c2.log 2>&1
echo done
