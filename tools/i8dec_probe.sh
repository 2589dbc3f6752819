# int8 layer-1 forward variants: correctness (selftest, no residual plane) and C3 timing
B=paper_2011_12895_b200/_lib/gemm_selftest
for d in ${DECS:-0 4x3 m2}; do
  echo "TLG_I8_DEC=$d"
  TLG_I8_DEC=$d timeout 300 $B 2>&1 | grep -E "no-lo|FAIL|PASS"
  TLG_I8_DEC=$d timeout 300 $B i8 2>&1 | grep -E "perf I8 bits fwd C3 L1 no-lo" | tail -1
done
