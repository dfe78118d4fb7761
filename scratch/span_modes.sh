for m in 0 1 2 4 6 7; do
  BSRP_EXTRA_NVCC="-DSPAN_MODE=$m" python -c "
import paper_2311_16883_b200.build as b, shutil
b.LIB = b.LIB.replace('libbsrprune.so', 'libbsrprune_m$m.so'); b.build(force=True)" > /dev/null || echo build $m failed
done
