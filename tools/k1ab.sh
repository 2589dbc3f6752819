# A/B of K1 (returns) library builds on the GPU box: for each variant, the HBM sweep
# (tools/hbm_sweep.py) and an ncu launch list of the returns kernels at 1 M segments.
#   VARIANTS="cur"            -> the in-tree libtlg_b200.so only
#   VARIANTS="head t8"        -> paper_2011_12895_b200/_lib/variants/lib_<v>.so, one by one
set -x; mkdir -p gpurun_out
L=paper_2011_12895_b200/_lib
[ -f $L/libtlg_b200.so ] && cp $L/libtlg_b200.so /tmp/libtlg_b200.cur.so
for v in ${VARIANTS:-cur}; do
  if [ "$v" = cur ]; then cp /tmp/libtlg_b200.cur.so $L/libtlg_b200.so; else cp $L/variants/lib_$v.so $L/libtlg_b200.so; fi
  timeout 300 python tools/hbm_sweep.py --out gpurun_out/sweep_$v.json > gpurun_out/sweep_$v.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:${KREGEX:-returns} --csv --log-file gpurun_out/ncu_k1_$v.csv python tools/hbm_sweep.py ${PROFILE_ARGS:---profile-returns 1048576} > gpurun_out/ncu_k1_$v.log 2>&1
done
cp /tmp/libtlg_b200.cur.so $L/libtlg_b200.so
