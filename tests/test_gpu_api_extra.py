"""API details of the drop-in surface beyond the recorded traces: the generator
classes round-trip their state with their own type (generators.py:322-374), and
calls route to the device that owns the caller's stream."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_19925_b200 as cb

    return cb


@pytest.mark.parametrize("name", ["Philox", "Threefry", "Squares", "Tyche"])
def test_subclass_state_roundtrip_and_copy(cb, oracle, name):
    cls = getattr(cb, name)
    g = cls(1234, 5)
    first = [g.next_u32() for _ in range(7)]
    r = cls.from_state_bytes(g.state_bytes())
    assert type(r) is cls and r.state_bytes() == g.state_bytes()
    c = g.copy()
    assert type(c) is cls
    nxt = [r.next_u32() for _ in range(9)]
    assert nxt == [c.next_u32() for _ in range(9)] == [g.next_u32() for _ in range(9)]
    alg = name.lower()
    assert first + nxt == [int(v) for v in oracle.stream_words(alg, 1234, 5, 16)]
    other = "Threefry" if name != "Threefry" else "Philox"
    with pytest.raises(ValueError):
        getattr(cb, other).from_state_bytes(g.state_bytes())
    assert type(cb.Generator.from_state_bytes(g.state_bytes())) is cb.Generator


def test_fill_on_stream_device_while_other_device_current(cb, oracle):
    """The C ABI launches on the device that owns the stream (DeviceGuard). With one
    visible GPU this checks the guard is transparent; with two, that a cuda:1
    tensor is filled on cuda:1 while cuda:0 is current."""
    import torch

    dev = torch.device("cuda", torch.cuda.device_count() - 1)
    with torch.cuda.device(0):
        out = torch.empty(4099, dtype=torch.float32, device=dev)
        cb.uniform_f32_array(cb.make_generator("philox", 3, 1), 4099, out=out)
        torch.cuda.synchronize(dev)
    assert np.array_equal(out.cpu().numpy(), oracle.words_to_f32(oracle.stream_words("philox", 3, 1, 4099)))
