cd /root/repo; mkdir -p gpurun_out/ab
for v in v0 v1; do
NBBGPU_LIB=/root/repo/paper_2110_12952_b200/ab_$v.so timeout 600 ncu --clock-control none --set full --import-source on -k regex:step_packed_ws3 -s 3 -c 1 -o gpurun_out/ab/c10_$v python tools/prof_step.py --fractal sierpinski-carpet --level 10 --kernel packed --steps 5 > gpurun_out/ab/c10_$v.log 2>&1
NBBGPU_LIB=/root/repo/paper_2110_12952_b200/ab_$v.so timeout 600 ncu --clock-control none --set full --import-source on -k regex:step_packed_ws3 -s 3 -c 1 -o gpurun_out/ab/h11_$v python tools/prof_step.py --fractal @descriptors/h-fractal.desc --level 11 --kernel packed --steps 5 > gpurun_out/ab/h11_$v.log 2>&1
done
ls -la gpurun_out/ab
for r in gpurun_out/ab/*.ncu-rep; do
  tools/ncu_summary.sh $r > ${r%.ncu-rep}.txt 2>&1
  ncu -i $r --page source --csv --print-source cuda,sass > ${r%.ncu-rep}_mix.csv 2>/dev/null
  gzip ${r%.ncu-rep}_mix.csv
  rm $r
done
ls -la gpurun_out/ab
