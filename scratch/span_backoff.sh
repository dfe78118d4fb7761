for v in b0 b32 b128; do for pr in tf32 bf16; do
  BSRP_LIB=$PWD/paper_2311_16883_b200/libbsrprune_$v.so BSRP_WGRAD=span timeout 120 python scratch/span_time.py $pr 0.5 | sed "s/^/$v /"
done; done
