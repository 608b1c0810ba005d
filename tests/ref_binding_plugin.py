"""pytest plugin: install the B200 binding (paper_2510_02080_b200.binding)
before the reference's own test modules are imported, so they exercise the
device path through the reference's public names.  Used by
tests/test_gpu_reference_suite.py (-p tests.ref_binding_plugin)."""


def pytest_configure(config):
    from paper_2510_02080_b200 import binding

    bound = binding.install()
    config._ec3r_bound = bound


def pytest_report_header(config):
    bound = getattr(config, "_ec3r_bound", [])
    return f"ec3r B200 binding: {len(bound)} reference names rebound"
