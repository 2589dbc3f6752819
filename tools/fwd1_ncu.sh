# ncu --set full of one C3 layer-1 forward launch inside the bench (after the command ran clean)
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-infer > gpurun_out/fwd1_plain.json 2>/dev/null || exit 1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"gemm_i8_bits_fwd" --launch-skip 5 --launch-count 1 -o gpurun_out/r02c_fwd1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-infer > gpurun_out/r02c_ncu.log 2>&1
ncu -i gpurun_out/r02c_fwd1.ncu-rep --page raw --csv > gpurun_out/r02c_fwd1_raw.csv 2>/dev/null
tail -2 gpurun_out/r02c_ncu.log
