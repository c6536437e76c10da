"""pytest plugin: run the REFERENCE's own test suite with its operator
swapped for the B200 one.

Every place the reference constructs ``ThermalOperator`` (the package
namespace, ``operators``, ``driver``, ``verification``) gets
``paper_2302_05164_b200.ThermalOperator``; the reference's own time
integrators (``run_scan_phase``, ``run_cooldown_phase``, ``krylov_solve``,
``compute_step_criteria``), mesh code, dense oracle and tests run
unchanged around it.  Used by tools/run_reference_suite.sh on a GPU box
(the reference sources are staged there by tools/stage_reference.sh into
the git-ignored baseline/_ref; nothing of the reference is committed).
"""

import os


def pytest_configure(config):
    import scantherm
    import scantherm.driver
    import scantherm.operators
    import scantherm.verification

    from paper_2302_05164_b200 import ThermalOperator as B200ThermalOperator
    for mod in (scantherm, scantherm.operators, scantherm.driver, scantherm.verification):
        if hasattr(mod, "ThermalOperator"):
            mod.ThermalOperator = B200ThermalOperator
    config._b200_swapped = True
    print(f"[refswap] scantherm.ThermalOperator -> {B200ThermalOperator.__module__}."
          f"{B200ThermalOperator.__name__} (pid {os.getpid()})")


def pytest_report_header(config):
    return "reference suite with paper_2302_05164_b200.ThermalOperator swapped in"


def pytest_runtest_call(item):
    import scantherm
    from paper_2302_05164_b200 import ThermalOperator as B200ThermalOperator
    assert scantherm.ThermalOperator is B200ThermalOperator
