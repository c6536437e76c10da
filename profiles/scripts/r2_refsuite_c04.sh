python -c "import __graft_entry__ as g; g.build()"
REFSUITE_TIMEOUT=2700 bash tools/run_reference_suite.sh test_operators.py test_timestepping.py test_verification.py test_physics.py test_material.py test_driver.py test_mesh.py test_acceptance.py --durations=10
