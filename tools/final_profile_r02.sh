# r02 end-of-round measurement pass (under gpurun, repo root); outputs gpurun_out/fin2
set -x
O=gpurun_out/fin2
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python bench.py > $O/bench_n1.log 2>&1; tail -1 $O/bench_n1.log > $O/bench_n1.json
python bench.py --impl reference > $O/bench_ref.log 2>&1; tail -1 $O/bench_ref.log > $O/bench_reference_n1.json
python bench.py --phi analytic --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_analytic_n1.json
python bench.py --workload cfg3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_cfg3_n1.json
python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_cfg5_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench_step.txt
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv|attention|stem|out_head|pool|upsample" --csv --log-file $O/lt.csv python tools/prof_step.py > /dev/null 2>&1
python tools/layer_table.py $O/lt.csv > $O/layer_table_unet64.txt 2>&1
python tools/launch_summary.py $O/lt.csv > $O/launches_unet64.txt
for spec in "dec0c1_dyn:conv_halo2:14" "enc0c1_dyn:conv_halo2:0" "attention3:attention3:0" "dec1c2:conv_halo2:11" "enc0c2_pool:conv_halo2:1" "qkv:conv_tc_kernel:2"; do
  name=${spec%%:*}; rest=${spec#*:}; re=${rest%%:*}; skip=${rest##*:}
  ncu --set full --import-source on --clock-control none -k regex:$re --launch-skip $skip -c 1 -o $O/$name python tools/prof_step.py > $O/ncu_$name.log 2>&1
  python tools/ncu_summary.py $O/$name.ncu-rep --label $name > $O/ncu_${name}_full.json 2>&1
  rm -f $O/$name.ncu-rep
done
python tools/traffic_json.py $O > $O/traffic.json
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"noise|blend|phi_" --csv --log-file $O/hbm_an.csv python bench.py --phi analytic --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/hbm_kernels.py $O/hbm_an.csv $O/hbm_kernels_analytic_cfg2.json > $O/hbm_kernels_analytic_cfg2.txt 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"noise|blend|phi_|laplac|blur|block_mean|widen|box_mean|signed|patch|condition|procedural|corrupt|tiles" --csv --log-file $O/hbm_c3.csv python bench.py --workload cfg3 --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
python tools/hbm_kernels.py $O/hbm_c3.csv $O/hbm_kernels_cfg3.json > $O/hbm_kernels_cfg3.txt 2>&1
python bench.py --workload cfg4 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_cfg4_n1.json
timeout 900 env IG_BENCH_SMOKE_1GPU=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --region 4096 > $O/smoke_2rank_cfg5.log 2>&1
timeout 900 env IG_BENCH_SMOKE_1GPU=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --no-analytic-leg > $O/smoke_2rank_reference.log 2>&1
rm -f $O/*.csv
ls -la $O; du -sh gpurun_out
