"""B200 additions to the reference wire protocol (whose messages and framing
are the reference's own module, re-exported): CUDA-IPC endpoints and the
InstanceAdapter that serves the messages with an instance."""
import spotrl.protocol

import pytest

from paper_2510_19225_b200 import protocol
from paper_2510_19225_b200.protocol import InstanceAdapter, ProtocolError
from tests.fakes import FakeInstance


def test_cuda_ipc_endpoint_round_trip():
    handles = [(bytes(range(64)), 0), (bytes(64), 4096)]
    ep = protocol.cuda_ipc_endpoint(3, handles, [100, 200])
    dev, tensors = protocol.parse_cuda_ipc_endpoint(ep)
    assert dev == 3 and tensors == [(bytes(range(64)), 0, 100), (bytes(64), 4096, 200)]
    msg = protocol.msg_pull_weights(7, ep)
    assert protocol.decode_line(protocol.encode_message(msg)) == msg
    with pytest.raises(ProtocolError):
        protocol.parse_cuda_ipc_endpoint("tcp://x")


def test_instance_adapter_serves_the_messages():
    inst = FakeInstance(vocab=50, max_slots=4)
    ad = InstanceAdapter(inst, "i0", open_endpoint=lambda ep, version: ep)
    assert protocol.decode_line(protocol.encode_message(ad.register()))["instance_id"] == "i0"
    out = ad.handle(protocol.msg_pull_weights(2, "cuda-ipc://x"))
    assert out[0]["weight_version"] == 2
    gen = dict(protocol.msg_generate("r", [1, 2, 3], [4]), target_len=3)
    ad.handle(gen)
    msgs = ad.pump(8)
    toks = [m["token_id"] for m in msgs if m["type"] == "token"]
    assert len(toks) == 2 and msgs[-1] == {"type": "complete", "request_id": "r"}
    for m in msgs:
        protocol.validate_message(m)
    with pytest.raises(ProtocolError, match="target_len"):
        ad.handle(protocol.msg_generate("s", [1], []))
    with pytest.raises(ProtocolError):
        ad.handle({"type": "token", "request_id": "x", "token_id": 1})


def test_protocol_is_the_reference_module():
    for name in ("encode_message", "decode_line", "msg_generate", "read_frames",
                 "receive_weights", "ProtocolError"):
        assert getattr(protocol, name) is getattr(spotrl.protocol, name)
