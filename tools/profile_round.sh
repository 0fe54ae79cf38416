# Round profile capture (run on the GPU box from the repo root): bench line, ncu launch list,
# ncu --set full raw CSV exports of the T, conv and elementwise kernels (reports deleted on the box).
set -x
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-extra"
timeout 300 python bench.py > gpurun_out/bench_full_${SUF:-r1d}.log 2>&1
tail -1 gpurun_out/bench_full_${SUF:-r1d}.log > gpurun_out/bench_line_${SUF:-r1d}.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${SUF:-r1d}.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tb_tc -s 1 -c 1 -o /tmp/tb $B > /dev/null 2>&1
ncu -i /tmp/tb.ncu-rep --page raw --csv > gpurun_out/tb_raw_${SUF:-r1d}.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:k_conv_tc -s 7 -c 7 -o /tmp/conv $B > /dev/null 2>&1
ncu -i /tmp/conv.ncu-rep --page raw --csv > gpurun_out/conv_raw_${SUF:-r1d}.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:"k_up2add|k_prep_x|k_output|k_tb_sort" -s 4 -c 4 -o /tmp/ew $B > /dev/null 2>&1
ncu -i /tmp/ew.ncu-rep --page raw --csv > gpurun_out/ew_raw_${SUF:-r1d}.csv 2>/dev/null
rm -f /tmp/*.ncu-rep
ls -la gpurun_out/
