"""pytest plugin (``-p vfpi_dropin_plugin``): run the REFERENCE's own tests
with condsim's V-FPI entry points swapped for the CUDA ones
(``paper_2201_09212_b200.dropin.install``) before any test module imports
them by name. Used by ``tests/test_gpu_dropin_suite.py``."""

PATCHED = []


def pytest_configure(config):
    from paper_2201_09212_b200 import _lib, dropin

    _lib.lib()  # fail loudly if the CUDA library is missing
    PATCHED[:] = dropin.install()


def pytest_report_header(config):
    return f"vfpi drop-in active: {len(PATCHED)} condsim entry points patched ({', '.join(PATCHED)})"
