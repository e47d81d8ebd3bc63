# ncu --set full of one launch of tools/prof_step.py: prof_one.sh NAME REGEX SKIP
NAME=$1; RE=$2; SKIP=$3
mkdir -p gpurun_out/p4
ncu --set full --import-source on --clock-control none -k regex:$RE --launch-skip $SKIP -c 1 -o gpurun_out/p4/$NAME python tools/prof_step.py > gpurun_out/p4/ncu_$NAME.log 2>&1
python tools/ncu_summary.py gpurun_out/p4/$NAME.ncu-rep --label $NAME > gpurun_out/p4/$NAME.json 2>&1
ncu -i gpurun_out/p4/$NAME.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/p4/${NAME}_source.csv.gz
ncu -i gpurun_out/p4/$NAME.ncu-rep --page raw --csv > gpurun_out/p4/${NAME}_raw.csv 2>/dev/null
rm -f gpurun_out/p4/$NAME.ncu-rep
