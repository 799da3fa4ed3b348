#!/bin/bash
# Test-of-tests: libraries built with a deliberate mutation of the soft-PSL
# gradient must turn the plain-relative soft-PSL parity tests red.  Build here:
#   python scripts/mutation_check.py build
# then under gpurun:  bash scripts/mutation_check.sh
mkdir -p gpurun_out
for m in no_psl no_zc; do
  GRAF_LIB_PATH=paper_2506_22935_b200/variants/libgraf_mut_${m}.so timeout 900 python -m pytest \
    tests/test_gpu_softpsl_parity.py -q -m gpu -p no:cacheprovider --timeout=300 \
    -k "c4_full_size_softpsl_only or c5_shape_unsharded or c5_full_size_against_golden or m16384_full_plane" \
    > gpurun_out/mutation_${m}.log 2>&1
  echo "mutation ${m}: pytest exit $? (nonzero = the tests caught it)" >> gpurun_out/mutation_summary.txt
  tail -1 gpurun_out/mutation_${m}.log >> gpurun_out/mutation_summary.txt
done
