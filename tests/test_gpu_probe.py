"""The in-run HBM read-stream ceiling (nsrgs_probe_read_stream, bench.py's roofline denominator)."""
import pytest

pytestmark = pytest.mark.gpu


def test_read_stream_probe_is_a_plausible_hbm_rate():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_07372_b200 import nsrgs

    buf = torch.ones(1 << 30, dtype=torch.float32, device="cuda")     # 4 GiB >> 126 MB L2
    st = torch.cuda.Stream()
    g = nsrgs.probe_read_stream(buf, st, 3)
    assert 3000.0 < g < 8200.0, g                                      # B200 HBM3e: 8 TB/s nominal
    with pytest.raises(nsrgs.NSRGSError):
        nsrgs.probe_read_stream(buf[:16], st, 1)                       # below one 32 KB chunk
