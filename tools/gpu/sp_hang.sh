#!/bin/bash
# the last -m gpu tests one by one, each under a 150 s pytest-timeout (stack dump on expiry)
export PYTHONPATH=.
for t in "tests/test_sp_gpu.py::test_sp_backward_vs_oracle" "tests/test_sp_gpu.py::test_sp_backward_nccl_world1_and_gla_forward" \
         "tests/test_sp_gpu.py::test_loopback_slices_with_different_plans" "tests/test_sp_gpu.py::test_normaliser_backward_rejects_carried_z" \
         "tests/test_tensor_bridge_gpu.py"; do
  echo "=== $t"
  timeout 400 python -m pytest "$t" -q -p no:cacheprovider --timeout=150 --durations=5 2>&1 | grep -v "^$" | tail -25
done
bash tools/gpu/moe_ab.sh
