# r02 profiling pass (run under gpurun from the repo root); outputs to gpurun_out/p2
set -x
mkdir -p gpurun_out/p2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv|attention|stem|out_head|pool|upsample" --csv --log-file gpurun_out/p2/lt.csv python tools/prof_step.py > /dev/null 2>&1
python tools/layer_table.py gpurun_out/p2/lt.csv > gpurun_out/p2/layer_table_unet64.txt 2>&1
for spec in "dec1c2:11" "dec2c2:7" "enc0c1:0" "dec0c1:14"; do
  name=${spec%%:*}; skip=${spec##*:}
  ncu --set full --import-source on --clock-control none -k regex:conv_halo2 --launch-skip $skip -c 1 -o gpurun_out/p2/$name python tools/prof_step.py > gpurun_out/p2/ncu_$name.log 2>&1
  python tools/ncu_summary.py gpurun_out/p2/$name.ncu-rep --label $name > gpurun_out/p2/$name.json 2>&1
  ncu -i gpurun_out/p2/$name.ncu-rep --page raw --csv > gpurun_out/p2/${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/p2/$name.ncu-rep --page source --csv > gpurun_out/p2/${name}_source.csv 2>/dev/null
  rm -f gpurun_out/p2/$name.ncu-rep
done
ncu --set full --import-source on --clock-control none -k regex:attention_kernel -c 1 -o gpurun_out/p2/attn python tools/prof_step.py > gpurun_out/p2/ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/p2/attn.ncu-rep --label attn > gpurun_out/p2/attn.json 2>&1
ncu -i gpurun_out/p2/attn.ncu-rep --page raw --csv > gpurun_out/p2/attn_raw.csv 2>/dev/null
ncu -i gpurun_out/p2/attn.ncu-rep --page source --csv > gpurun_out/p2/attn_source.csv 2>/dev/null
rm -f gpurun_out/p2/attn.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/p2/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p2/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/p2/launches_bench.csv > gpurun_out/p2/launches_bench_step.txt
gzip -f gpurun_out/p2/launches_bench.csv gpurun_out/p2/lt.csv gpurun_out/p2/*_source.csv
ls -la gpurun_out/p2; du -sh gpurun_out
