# per-layer A/B of an environment toggle: tools/ab_layers.sh VAR "A B" (under gpurun)
VAR=$1; VALS=$2
mkdir -p gpurun_out/ab
for v in $VALS; do
  env $VAR=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv|attention|stem|out_head|pool|upsample" --csv --log-file gpurun_out/ab/lt_$v.csv python tools/prof_step.py > /dev/null 2>&1
  python tools/layer_table.py gpurun_out/ab/lt_$v.csv > gpurun_out/ab/layer_table_$VAR_$v.txt 2>&1
  rm -f gpurun_out/ab/lt_$v.csv
done
for v in $VALS $VALS; do env $VAR=$v python tools/fwd_ab.py --tag "$VAR=$v"; done > gpurun_out/ab/fwd_$VAR.txt 2>&1
