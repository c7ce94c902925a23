#!/bin/bash
# Round-2 final ncu captures of the kernels changed after r02b: k_trinv_one (c2, k = 128),
# k_filter_coop as a thread-block cluster (c1, d = 200) and as a cooperative grid (c2),
# k_sample (c2).  Each command ran without ncu first (prof_cfg.py, exit 0).
set -x
O=gpurun_out/r02e_full
mkdir -p $O
for c in c1 c2; do CFG=$c timeout 300 python scripts/prof_cfg.py > $O/plain_$c.log 2>&1 || exit 1; done
CFG=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trinv_one -c 1 \
    -o $O/c2_trinv_one python scripts/prof_cfg.py > $O/ncu_trinv.log 2>&1
CFG=c1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_coop -s 1 -c 1 \
    -o $O/c1_filter_cluster python scripts/prof_cfg.py > $O/ncu_filter_c1.log 2>&1
CFG=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_coop -s 1 -c 1 \
    -o $O/c2_filter_coop python scripts/prof_cfg.py > $O/ncu_filter_c2.log 2>&1
CFG=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 1 -c 1 \
    -o $O/c2_sample python scripts/prof_cfg.py > $O/ncu_sample_c2.log 2>&1
for f in c2_trinv_one c1_filter_cluster c2_filter_coop c2_sample; do
  ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>/dev/null
  ncu -i $O/$f.ncu-rep --page details --csv > $O/${f}_details.csv 2>/dev/null
done
echo done
