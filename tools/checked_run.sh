#!/bin/bash
# Build the library with -DHK_CHECKED (device bounds checks, hawkes_kernels.cuh HK_CHECK) into
# tools/alt_build/lib_checked.so and run the GPU test-suite against it (HAWKES_LIB_AB).
# compute-sanitizer is closed on the GPU pool; this is the substitute.
#   on the CPU host:  python tools/ab_builds.py build checked=HK_CHECKED
#   on the GPU:       bash tools/checked_run.sh [pytest args]
set -e
cd "$(dirname "$0")/.."
HAWKES_LIB_AB=tools/alt_build/lib_checked.so python -m pytest tests -m gpu -q -p no:cacheprovider \
  --deselect tests/test_parity_gpu.py::test_library_is_in_tree "$@"
