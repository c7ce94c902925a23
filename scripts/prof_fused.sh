# ncu of the fused projection (eager loop: ncu cannot profile kernels inside a conditional graph)
set -x
mkdir -p gpurun_out/fz
export RBRP_NO_GRAPH=1
python scripts/prof_one.py --config c2 --reps 1 --warm 1 > gpurun_out/fz/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_proj_fused -s 10 -c 4 \
    -o gpurun_out/fz/fused_full python scripts/prof_one.py --config c2 --reps 1 --warm 1 > gpurun_out/fz/ncu.log 2>&1
echo rc=$?
tail -5 gpurun_out/fz/ncu.log
