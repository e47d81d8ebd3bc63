set -x
mkdir -p gpurun_out/fin
python bench.py > gpurun_out/fin/bench_n1.log 2>&1; tail -1 gpurun_out/fin/bench_n1.log > gpurun_out/fin/bench_n1.json
python bench.py --impl reference > gpurun_out/fin/bench_ref.log 2>&1; tail -1 gpurun_out/fin/bench_ref.log > gpurun_out/fin/bench_reference_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/fin/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/fin/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/fin/launches_bench.csv > gpurun_out/fin/launches_bench_step.txt
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv|attention|stem|out_head|pool|upsample" --csv --log-file gpurun_out/fin/lt.csv python tools/prof_step.py > /dev/null 2>&1
python tools/layer_table.py gpurun_out/fin/lt.csv > gpurun_out/fin/layer_table_unet64.txt 2>&1
python tools/launch_summary.py gpurun_out/fin/lt.csv > gpurun_out/fin/launches_unet64.txt
ncu --set full --import-source on --clock-control none -k regex:conv_halo2 --launch-skip 1 -c 1 -o gpurun_out/fin/conv_c2_full python tools/prof_step.py > gpurun_out/fin/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attention_kernel -c 1 -o gpurun_out/fin/attn_full python tools/prof_step.py > gpurun_out/fin/ncu_attn.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"noise|blend|phi_" --csv --log-file gpurun_out/fin/hbm_an.csv python bench.py --phi analytic --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"noise|blend|phi_|laplac|blur|block_mean|widen|box_mean|signed|patch|condition|procedural|corrupt" --csv --log-file gpurun_out/fin/hbm_c3.csv python bench.py --workload cfg3 --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
python bench.py --phi analytic --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin/bench_analytic.json
python bench.py --workload cfg4 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin/bench_cfg4.json
python bench.py --workload cfg3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin/bench_cfg3.json
python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fin/bench_cfg5.json
ls -la gpurun_out/fin
