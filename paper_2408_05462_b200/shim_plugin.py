"""pytest plugin: run the reference package's own test suite with the CUDA
kernel seam installed (shim.install(), isochr.kernels -> libchr.so).

    PYTHONPATH=baseline/_ref:. python -m pytest baseline/_ref/isochr_tests \\
        -p paper_2408_05462_b200.shim_plugin

The reference's ``both_backends`` fixture (conftest.py:14-21) still flips
backend.USE_NUMBA; with the seam installed both of its params run the CUDA
kernels.
"""


def pytest_configure(config):
    from . import shim

    shim.install()
    config.addinivalue_line("markers", "cuda_seam: isochr.kernels served by libchr.so")


def pytest_report_header(config):
    return "isochr.kernels -> paper_2408_05462_b200 CUDA seam (libchr.so)"
