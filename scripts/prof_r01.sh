set -x
mkdir -p gpurun_out/r01
export RBRP_NO_GRAPH=1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r01/bench_nograph.log 2>&1; echo rc=$?
tail -c 600 gpurun_out/r01/bench_nograph.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_launch.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_update_mma -s 2 -c 1 -o gpurun_out/r01/update_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_upd.log 2>&1; echo ncu2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_nt_mma -s 2 -c 1 -o gpurun_out/r01/lhat_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_lhat.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_filter_coop -s 2 -c 1 -o gpurun_out/r01/filter_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_filt.log 2>&1; echo ncu4 rc=$?
ls -la gpurun_out/r01
