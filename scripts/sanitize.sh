#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the product
# kernels on small cases; summaries to gpurun_out/sanitize_*.txt
set -u
MEM="tests/test_gpu_parity.py::test_residual_tangent_mixed_vs_reference_golden tests/test_gpu_parity.py::test_sheared_hex_vs_oracle tests/test_gpu_parity.py::test_one_launch_operator_bitwise_equal_two_launch tests/test_gpu_nonlinear.py::test_generated_path_vs_reference_golden tests/test_gpu_nonlinear.py::test_curved_elements_vs_reference_golden tests/test_gpu_solver.py::test_steady_solve_matches_reference tests/test_gpu_solver.py::test_block_jacobi_320_blocks_match_reference_ns3d_hex_p3 tests/test_gpu_solver.py::test_block_jacobi_shared_classes_bit_identical tests/test_gpu_solver.py::test_device_initial_state_matches_reference"
RACE="tests/test_gpu_parity.py::test_residual_tangent_mixed_vs_reference_golden"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 $( [ -n "${K:-}" ] && echo ) \
  python -m pytest $MEM -q -k "${K:-poisson3d_hex_p3 or tet or ns3d or quad_p3_n4 or curved or hex or euler2d or poisson-False}" > gpurun_out/sanitize_memcheck.txt 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_memcheck.txt | tail -3
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $RACE -q \
    -k "poisson3d_hex_p3 or tet or poisson3d_hex_p2 or convdiff3d_hex_periodic_p2" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_$tool.txt | tail -3
done
