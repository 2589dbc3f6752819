# bottleneck probes of the int8 layer-1 forward (timing-only debug builds; results wrong)
V=paper_2011_12895_b200/_lib/variants
for v in NOEXP NOX7 ONEMMA; do echo "== $v"; TLG_I8_DEC=0 timeout 300 $V/selftest_$v i8 2>&1 | grep -E "perf I8 bits fwd C3 L1 no-lo" | head -1; done
echo "== baseline"; TLG_I8_DEC=0 timeout 300 paper_2011_12895_b200/_lib/gemm_selftest i8 2>&1 | grep -E "perf I8 bits fwd C3 L1 no-lo" | head -1
