#!/bin/bash
# Stage the reference's hot-path test files (NOT tracked: oracle/_ref is
# git-ignored) so tests/ref_replay can run them on a GPU box that has no
# /root/reference.  Run here, then ship with gpurun.
set -e
cd "$(dirname "$0")/.."
mkdir -p oracle/_ref/ref_tests
for f in test_reference.py test_pooling.py test_slide_kernels.py test_gemm.py test_verify.py test_acceptance.py; do
  cp /root/reference/pkg/tests/$f oracle/_ref/ref_tests/
done
echo "staged $(ls oracle/_ref/ref_tests | wc -l) files in oracle/_ref/ref_tests"
