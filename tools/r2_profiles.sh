#!/bin/bash
# Round-2 measurement bundle (run on the GPU box): configs, backend CSV, the bench
# launch list, ncu --set full captures of the headline kernels.  Outputs in gpurun_out/r2/.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/r2; mkdir -p $O
NCU="ncu --clock-control none"
timeout 900 python tools/bench_configs.py > $O/r2_configs.json 2> $O/r2_configs.err; echo "configs rc=$?"
timeout 600 python tools/bench_csv.py > $O/r2_bench_backends.csv 2> $O/r2_bench_backends.err; echo "csv rc=$?"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/r2_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1; echo "launches rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:step_packed_ws3 -s 4 -c 1 -o $O/r2_step_r20 \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_step.log 2>&1; echo "ncu step rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:halo_words -s 4 -c 1 -o $O/r2_halo_r20 env NBBGPU_HALO_WARPS=0 \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_halo.log 2>&1; echo "ncu halo rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:"step_packed_ws3|halo_bt_regs" -s 4 -c 2 -o $O/r2_jit_k12 \
    python tools/prof_step.py --fractal @descriptors/k6s3.desc --level 12 --kernel packed --steps 5 > $O/ncu_jit.log 2>&1; echo "ncu jit rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:step_bb_rows -s 3 -c 1 -o $O/r2_bb_t16 \
    python tools/prof_step.py --level 16 --backend gpu-bb --steps 5 > $O/ncu_bb.log 2>&1; echo "ncu bb rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:step_bb_rows -s 3 -c 1 -o $O/r2_bb_c10 \
    python tools/prof_step.py --fractal sierpinski-carpet --level 10 --backend gpu-bb --steps 5 > $O/ncu_bb_c10.log 2>&1; echo "ncu bb c10 rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:"step_packed_ws3|halo_bt_regs" -s 6 -c 2 -o $O/r2_h11 \
    python tools/prof_step.py --fractal @descriptors/h-fractal.desc --level 11 --kernel packed --steps 5 > $O/ncu_h11.log 2>&1; echo "ncu h11 rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:step_packed_ws3 -s 4 -c 1 -o $O/r2_c9 \
    python tools/prof_step.py --fractal sierpinski-carpet --level 9 --kernel packed --steps 6 > $O/ncu_c9.log 2>&1; echo "ncu c9 rc=$?"
# text summaries (the .ncu-rep files stay only when small: gpurun copies back <= 64 MiB)
for r in $O/*.ncu-rep; do
  tools/ncu_summary.sh $r > ${r%.ncu-rep}.txt 2>&1
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
done
find $O -name '*.ncu-rep' -size +6M -delete
du -sh $O; ls -la $O
