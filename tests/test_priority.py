"""Communication priorities (include/monta.h 1d):
the reference's EP > PP > CP > DP resolution order (conflict.hpp:40-50)
mapped onto CUDA stream priorities."""
import pytest
import torch

from paper_2411_00662_b200 import _lib, ops


def test_reference_resolution_order():
    # conflict.hpp:40-50: EP 3, PP 2, CP 1, DP 0, TP/SP -1
    assert [ops.comm_priority(g) for g in (_lib.COMM_EP, _lib.COMM_PP, _lib.COMM_CP, _lib.COMM_DP,
                                           _lib.COMM_TP_SP)] == [3, 2, 1, 0, -1]


@pytest.mark.gpu
def test_stream_priorities_follow_the_order(cuda):
    least, greatest = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
        else (0, -5)
    prios = [ops.comm_stream_priority(g) for g in (_lib.COMM_EP, _lib.COMM_PP, _lib.COMM_CP, _lib.COMM_DP,
                                                  _lib.COMM_TP_SP)]
    # numerically lower = higher priority; EP on top, TP/SP at the bottom, distinct
    # levels where the device offers them (B200: 6 levels, -5..0)
    assert prios == sorted(prios) and prios[0] < prios[3]
    assert len(set(prios)) >= 4
    s = ops.comm_stream(_lib.COMM_DP)
    assert s.priority >= prios[0]  # torch may clamp to its own range; never above EP
