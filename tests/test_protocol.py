"""Wire protocol + pull framing (reference known answers, pkg/tests/test_protocol.py
cases restated) and the B200 additions: CUDA-IPC endpoints, InstanceAdapter."""
import io

import pytest

from paper_2510_19225_b200 import protocol
from paper_2510_19225_b200.protocol import InstanceAdapter, ProtocolError
from tests.fakes import FakeInstance


@pytest.mark.parametrize("message", [
    {"type": "register", "instance_id": "i0", "gpu_count": 1},
    {"type": "status", "m_pending": 1, "m_exec": 7, "weight_version": 3},
    {"type": "token", "request_id": "r1", "token_id": 42},
    {"type": "complete", "request_id": "r1"},
    protocol.msg_generate("r1", [1, 2, 3], [9, 9]),
    protocol.msg_cancel("r1"),
    protocol.msg_pull_weights(5, "10.0.0.2:9000"),
])
def test_round_trip(message):
    line = protocol.encode_message(message)
    assert line.endswith(b"\n") and protocol.decode_line(line) == message


@pytest.mark.parametrize("line,err", [(b'{"type": "bogus"}', "unknown message type"),
                                      (b'{"type": "register", "instance_id": "i0"}', "missing fields"),
                                      (b"{nope", "malformed"), (b"[1, 2]", "expected JSON object")])
def test_rejections(line, err):
    with pytest.raises(ProtocolError, match=err):
        protocol.decode_line(line)


def test_iter_skips_blank_lines():
    s = io.BytesIO(protocol.encode_message(protocol.msg_cancel("a")) + b"\n"
                   + protocol.encode_message({"type": "complete", "request_id": "b"}))
    assert [m["type"] for m in protocol.iter_messages(s)] == ["cancel", "complete"]


def test_pull_session_known_answer():
    buf = io.BytesIO()
    protocol.write_pull_request(buf, version=4)
    blob = bytes(range(256)) * 40
    for k in range(0, len(blob), 1000):
        protocol.write_shard(buf, blob[k:k + 1000])
    protocol.write_done(buf, version=4, total_bytes=len(blob))
    buf.seek(0)
    assert protocol.read_pull_request(buf) == 4
    assert protocol.receive_weights(buf) == (4, blob)


def test_pull_session_errors():
    b = io.BytesIO()
    protocol.write_shard(b, b"abc")
    protocol.write_done(b, version=1, total_bytes=99)
    b.seek(0)
    with pytest.raises(ProtocolError, match="byte count mismatch"):
        protocol.receive_weights(b)
    b = io.BytesIO()
    protocol.write_shard(b, b"abcdef")
    with pytest.raises(ProtocolError, match="truncated frame payload"):
        list(protocol.read_frames(io.BytesIO(b.getvalue()[:-3])))
    b.seek(0)
    with pytest.raises(ProtocolError, match="ended before done"):
        protocol.receive_weights(b)
    with pytest.raises(ProtocolError, match="truncated frame header"):
        list(protocol.read_frames(io.BytesIO(b"W\x00")))


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
