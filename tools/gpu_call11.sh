NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:acoustic_wtb -s 1 -c 1 -o gpurun_out/r02_wtb_so4 python tools/prof_one.py 4 2 > gpurun_out/r02_ncu_wtb_so4.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:tti_fused -s 2 -c 1 -o gpurun_out/r02_tti_fused python tools/prof_one.py tti > gpurun_out/r02_ncu_tti.log 2>&1
ls -la gpurun_out/*.ncu-rep
