B=paper_2011_12895_b200/_lib/gemm_selftest
for mc in 1 2; do TLG_I8_MC=$mc timeout 300 $B i8 2>&1 | grep -E "perf|PASS|FAIL"; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x,sm__ctas_launched.sum,smsp__cycles_active.avg.pct_of_peak_sustained_elapsed
for mc in 1 2; do TLG_I8_MC=$mc timeout 600 ncu --metrics $M --clock-control none -k regex:i8_bits_fwd --csv --log-file gpurun_out/mc_$mc.csv $B i8 > /dev/null 2>&1; done
