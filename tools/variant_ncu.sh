# ncu launch list (durations) of one command per library variant
L=paper_2011_12895_b200/_lib
cp $L/libtlg_b200.so /tmp/libtlg_b200.keep.so
for v in ${VARIANTS:-cur}; do
  cp $L/variants/lib_$v.so $L/libtlg_b200.so
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/vncu_$v.csv $CMD > /dev/null 2>&1
done
cp /tmp/libtlg_b200.keep.so $L/libtlg_b200.so
