# Round-1 (second session) profiles of the fused projection path.
# ncu cannot profile kernels inside a conditional CUDA graph: RBRP_NO_GRAPH=1 launches
# the same kernels eagerly.
set -x
mkdir -p gpurun_out/r01b
export RBRP_NO_GRAPH=1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r01b/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/r01b/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/r01b/ncu_launch.log 2>&1
echo ncu1 rc=$?
python scripts/prof_one.py --config c2 --reps 1 --warm 1 > gpurun_out/r01b/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_proj_fused -s 10 -c 4 \
    -o gpurun_out/r01b/fused_full python scripts/prof_one.py --config c2 --reps 1 --warm 1 > gpurun_out/r01b/ncu_full.log 2>&1
echo ncu2 rc=$?
ls -la gpurun_out/r01b
