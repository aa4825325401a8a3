"""pytest plugin: run the REFERENCE's own test files with its CD core and
Shepard evaluation swapped for the B200 C-ABI seams (integration/fieldfit_b200.py).

Used by tests/test_gpu_dropin.py as ``python -m pytest -p integration.refseam_plugin
baseline/_ref/tests_ref/...`` with the reference installed under baseline/_ref.
Writes the number of seam calls to $REFSEAM_COUNTS at the end of the session,
so the caller can prove the GPU path ran.
"""

import json
import os


def pytest_configure(config):
    import fieldfit

    from integration import fieldfit_b200

    fieldfit_b200.install(fieldfit)


def pytest_sessionfinish(session, exitstatus):
    from integration import fieldfit_b200

    path = os.environ.get("REFSEAM_COUNTS")
    if path:
        with open(path, "w") as f:
            json.dump(fieldfit_b200.CALLS, f)
