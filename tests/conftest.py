import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture
def kernel_mode():
    """Set the native kernel family for one test, restoring auto after."""
    from paper_2410_06770_b200 import (set_bulk, set_complex_embed, set_kernel, set_kr, set_pair,
                                       set_pipeline, set_split_k, set_stream_k, set_tma, set_wide)

    def use(name, split=0, pipeline=-1, stream_k=True, tma=True, pair=False, complex_embed=True,
            kr="auto", kr_fused=False, kr_pair=True, bulk=True, wide="auto", kr_mixed=True, wide_mixed=False, wide_tail=True):
        set_kernel(name)
        set_bulk(bulk)
        set_wide(wide, wide_mixed, wide_tail)
        set_split_k(split)
        set_pipeline(pipeline)
        set_stream_k(stream_k)
        set_tma(tma)
        set_pair(pair)
        set_complex_embed(complex_embed)
        set_kr(kr, kr_fused, kr_pair, kr_mixed)

    yield use
    set_kernel("auto")
    set_split_k(0)
    set_pipeline(-1)
    set_stream_k(True)
    set_tma(True)
    set_pair(False)
    set_complex_embed(True)
    set_kr("auto")
    set_bulk(True)
    set_wide("auto")
