"""Halo message sizes of the x0-slab decomposition (SURVEY §8(e) payload table; no GPU needed)."""
import synth


def test_trace_halo_payload_sizes():
    """2 n^2 doubles per boundary cell (u and d_0 u at the face points) instead of the n^3 block:
    cfg3 37.75 -> 9.44 MB, cfg4 65.5 -> 26.2 MB per message."""
    for w, full_mb, tr_mb in ((synth.CONFIGS[3], 37.75, 9.44), (synth.CONFIGS[4], 65.5, 26.2)):
        pc = w.N[1] * w.N[2]
        assert abs(pc * w.n ** 3 * 8 / 1e6 - full_mb) < 0.05
        assert abs(pc * 2 * w.n ** 2 * 8 / 1e6 - tr_mb) < 0.05
