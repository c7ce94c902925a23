# Round-1 (third session) profile set: launch list of one eager c2 ID, a full ncu capture of
# the tiled projection (k_lhat_paper<32>, residual mode) and of the SkLUPP-OSID kernels
# (NEXT-4), the bench line and the Table 3 sweep.  ncu cannot profile kernels inside a
# conditional CUDA graph: RBRP_NO_GRAPH=1 launches the same kernels eagerly.
set -x
O=gpurun_out/r01c
mkdir -p $O
timeout 300 python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_ref.err
export RBRP_NO_GRAPH=1
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-alt-form --no-sketch > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-alt-form --no-sketch \
    > $O/ncu_launch.log 2>&1
echo ncu1 rc=$?
timeout 300 python scripts/prof_one.py --config c2 --reps 1 --warm 1 > $O/plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lhat_paper -s 10 -c 4 \
    -o $O/tiled_full python scripts/prof_one.py --config c2 --reps 1 --warm 1 > $O/ncu_full.log 2>&1
echo ncu2 rc=$?
timeout 300 python scripts/sketch_c2.py --reps 1 > $O/sketch_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lupp|k_nt_mma" -s 0 -c 3 \
    -o $O/sketch_full python scripts/sketch_c2.py --reps 1 > $O/ncu_sketch.log 2>&1
echo ncu3 rc=$?
timeout 600 python scripts/table3.py --reps 3 > $O/table3.jsonl 2> $O/table3.err
for f in tiled_full sketch_full; do
  ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>/dev/null
  ncu -i $O/$f.ncu-rep --page details --csv > $O/${f}_details.csv 2>/dev/null
done
ls -la $O
