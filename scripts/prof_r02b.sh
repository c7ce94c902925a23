#!/bin/bash
# Round-2 profile set, second pass (after k_lhat64, the W GEMM groups of 64 and the filter's
# REDUX pivot search): bench line, reference arm, launch lists (eager loop) per config, ncu
# full captures of the dominant kernels (c5: k_lhat64 on a 64-column part; c3: k_lhat64;
# c4: k_proj_tc32; c2: k_lhat_paper<32>).  Every ncu command runs only after the same
# command exited 0 without ncu.
set -x
O=gpurun_out/r02b
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for c in c5 c4 c3 c2; do
  CFG=$c timeout 600 python scripts/prof_cfg.py > $O/plain_$c.log 2>&1 &&
  CFG=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_$c.csv python scripts/prof_cfg.py > $O/launches_$c.log 2>&1
done
CFG=c5 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_lhat64 -s 8 -c 1 \
    -o $O/c5_lhat64 python scripts/prof_cfg.py > $O/ncu_c5.log 2>&1
CFG=c3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lhat64 -s 0 -c 1 \
    -o $O/c3_lhat64 python scripts/prof_cfg.py > $O/ncu_c3.log 2>&1
CFG=c4 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_proj_tc32 -s 2 -c 1 \
    -o $O/c4_tc32 python scripts/prof_cfg.py > $O/ncu_c4.log 2>&1
CFG=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lhat_paper -s 1 -c 1 \
    -o $O/c2_lhat python scripts/prof_cfg.py > $O/ncu_c2.log 2>&1
echo done
