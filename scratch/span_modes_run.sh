timeout 300 python -m pytest tests/test_wgrad_tc_parity.py -q -x 2>&1 | tail -2
for m in 0 1 2 4 7; do for cg in 2 1; do for pr in tf32 bf16; do
 BSRP_LIB=$PWD/paper_2311_16883_b200/libbsrprune_m$m.so BSRP_WGRAD_CG=$cg timeout 120 python scratch/span_time.py $pr 0.5 2>&1 | tail -1 | sed "s/^/cg=$cg /"
done; done; done
