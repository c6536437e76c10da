set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.txt
tail -3 gpurun_out/gputests.txt
REFSUITE_TIMEOUT=2400 bash tools/run_reference_suite.sh test_operators.py test_timestepping.py test_verification.py test_physics.py test_material.py "test_acceptance.py::test_c01_kernels_match_dense_reference_over_random_states" "test_acceptance.py::test_c02_stability_boundary_brackets_the_estimate" "test_acceptance.py::test_c03_combined_step_criterion_reproduces_the_working_point" "test_acceptance.py::test_c05_insulated_runs_conserve_thermal_energy" "test_acceptance.py::test_c07b_lane_width_never_changes_deterministic_kernels" "test_acceptance.py::test_c09_large_mesh_throughput_and_scatter_agreement" "test_acceptance.py::test_c10_hatch_layout_and_exact_time_accounting"
