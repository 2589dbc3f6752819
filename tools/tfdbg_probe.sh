# bottleneck probes of the 3xTF32 short-K GEMMs (timing-only debug builds; results wrong)
V=paper_2011_12895_b200/_lib/variants
for v in tf_NOA tf_NOLO; do echo "== $v"; timeout 300 $V/selftest_$v perf 2>&1 | grep -E "perf (fwd|dX) C3 L2"; done
echo "== baseline"; timeout 300 paper_2011_12895_b200/_lib/gemm_selftest perf 2>&1 | grep -E "perf (fwd|dX) C3 L2"
