mkdir -p gpurun_out/p3
IG_ATT_POLY=4 ncu --set full --import-source on --clock-control none -k regex:attention3 -c 1 -o gpurun_out/p3/attn2 python tools/attn_ab.py > gpurun_out/p3/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p3/attn2.ncu-rep --label attn2 > gpurun_out/p3/attn2.json 2>&1
ncu -i gpurun_out/p3/attn2.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/p3/attn2_source.csv.gz
ncu -i gpurun_out/p3/attn2.ncu-rep --page raw --csv > gpurun_out/p3/attn2_raw.csv 2>/dev/null
rm -f gpurun_out/p3/attn2.ncu-rep
