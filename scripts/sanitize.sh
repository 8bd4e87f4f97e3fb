#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the product kernels
# on small cases (fused hex p=3 plane + completion kernels, pencil kernels,
# dense simplex, generated NS, Krylov, block-Jacobi); summaries to gpurun_out/
set -u
T="tests/test_gpu_parity.py::test_residual_tangent_mixed_vs_reference_golden tests/test_gpu_parity.py::test_sheared_hex_p3_vs_oracle tests/test_gpu_nonlinear.py::test_generated_path_vs_reference_golden tests/test_gpu_solver.py::test_steady_solve_matches_reference"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
    python -m pytest $T -q -x -k "poisson3d_hex_p3 or poisson2d_quad_p3_n4_bj or tet or ns3d or poisson or convection" \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Hazard|Invalid" gpurun_out/sanitize_$tool.txt | head -8
done
