# Round-1 (fourth session) profile set: the bench line, the reference arm, the launch list
# of one eager c2 ID, a full ncu capture of the SkLUPP-OSID kernels after the LUPP / OSID
# rework (k_lupp, k_dgemm_small, k_chol_panel), launch lists of one SkLUPP-OSID call at
# Table 3 ranks 128 and 472, and the Table 3 sweep.  The projection kernel is unchanged
# since r01c (r01c_tiled_full_*).  RBRP_NO_GRAPH=1: ncu cannot profile kernels inside a
# conditional CUDA graph, so the same kernels are launched eagerly.
set -x
O=gpurun_out/r01d
mkdir -p $O
timeout 300 python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_ref.err
timeout 600 python scripts/table3.py --reps 3 > $O/table3.jsonl 2> $O/table3.err
export RBRP_NO_GRAPH=1
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-alt-form --no-sketch > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-alt-form --no-sketch \
    > $O/ncu_launch.log 2>&1
echo ncu1 rc=$?
for k in 128 472; do
  timeout 300 python scripts/sketch_one.py $k > $O/sk${k}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/sk${k}_launches.csv \
      python scripts/sketch_one.py $k > /dev/null 2>&1
  python scripts/ncu_agg.py $O/sk${k}_launches.csv 20 > $O/sk${k}_kernels.txt
done
timeout 300 python scripts/sketch_c2.py --reps 1 > $O/sketch_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lupp|k_dgemm_small|k_chol_panel" -s 0 -c 3 \
    -o $O/sketch_full python scripts/sketch_c2.py --reps 1 > $O/ncu_sketch.log 2>&1
echo ncu2 rc=$?
ncu -i $O/sketch_full.ncu-rep --page raw --csv > $O/sketch_full_raw.csv 2>/dev/null
ncu -i $O/sketch_full.ncu-rep --page details --csv > $O/sketch_full_details.csv 2>/dev/null
ls -la $O
