set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.txt
tail -40 gpurun_out/gputests.txt
REFSUITE_TIMEOUT=2400 bash tools/run_reference_suite.sh test_operators.py test_timestepping.py test_verification.py test_physics.py test_material.py test_driver.py test_mesh.py test_acceptance.py --deselect "test_acceptance.py::test_c04_temporal_convergence_of_the_split_schedule"
