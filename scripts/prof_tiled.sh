# DRAM traffic + full capture of the tiled residual projection (k_lhat_paper, resid mode)
set -x
mkdir -p gpurun_out/tl
export RBRP_NO_GRAPH=1 RBRP_TILED=1
python scripts/prof_one.py --config c2 --reps 1 --warm 1 > gpurun_out/tl/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_lhat_paper -s 10 -c 4 \
    -o gpurun_out/tl/tiled_full python scripts/prof_one.py --config c2 --reps 1 --warm 1 > gpurun_out/tl/ncu.log 2>&1
echo rc=$?
