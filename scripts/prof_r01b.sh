mkdir -p gpurun_out/r01
export RBRP_NO_GRAPH=1
ncu --set full --clock-control none --import-source on -k regex:k_update_mma -s 1 -c 1 -o gpurun_out/r01/update_full32 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_upd32.log 2>&1; echo ncu2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_nt_mma -s 1 -c 1 -o gpurun_out/r01/lhat_full32 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_lhat32.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_init_norms -s 0 -c 1 -o gpurun_out/r01/init_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_init.log 2>&1; echo ncu4 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_trinv -s 0 -c 1 -o gpurun_out/r01/trinv_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_trinv.log 2>&1; echo ncu5 rc=$?
