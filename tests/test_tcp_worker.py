"""GPU worker for the reference's TCP master.

The unmodified reference master (oracle/_ref/qcut_refgen master -> qcut::run_distributed,
proj/core/src/master.cpp:52-272) hands out density slice-id batches; qcut_gpu_worker answers
them with the B200 engine over the reference wire protocol (protocol.hpp:25-37)."""
import base64
import gzip
import json
import os
import socket
import subprocess
import threading

import pytest

from conftest import ROOT, cx, payload_path, ref_json

WORKER = os.path.join(ROOT, "paper_2010_14962_b200", "_lib", "qcut_gpu_worker")
REFGEN = os.path.join(ROOT, "oracle", "_ref", "qcut_refgen")


def _payload_text(stem):
    with gzip.open(payload_path(stem), "rb") as f:
        return f.read()


def _fnv1a64_hex(b: bytes) -> str:
    h = 0xcbf29ce484222325
    for c in b:
        h ^= c
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def test_worker_rejects_a_payload_with_a_wrong_hash():
    """Handshake + content-address check (worker.cpp:62-76) against a scripted master; no GPU needed."""
    assert os.path.exists(WORKER)
    srv = socket.socket()
    srv.bind(("127.0.0.1", 0))
    srv.listen(1)
    port = srv.getsockname()[1]
    body = _payload_text("cnot")
    seen = []

    def master():
        conn, _ = srv.accept()
        f = conn.makefile("rwb")
        seen.append(json.loads(f.readline()))
        f.write(b'{"t":"payload","hash":"0123456789abcdef","body":""}\n')
        f.flush()
        seen.append(json.loads(f.readline()))  # need_payload
        wrong = base64.b64encode(body).decode()
        f.write(json.dumps({"t": "payload", "hash": "0123456789abcdef", "body": wrong}).encode() + b"\n")
        f.flush()
        seen.append(json.loads(f.readline()))  # bye
        conn.close()

    th = threading.Thread(target=master)
    th.start()
    r = subprocess.run([WORKER, "--connect", f"127.0.0.1:{port}", "--id", "7", "--device", "-1"],
                       capture_output=True, text=True, timeout=60)
    th.join(timeout=30)
    srv.close()
    assert seen[0] == {"t": "hello", "worker": 7, "slots": 1}
    assert seen[1] == {"t": "need_payload", "hash": "0123456789abcdef"}
    assert seen[2] == {"t": "bye"}
    assert r.returncode == 1 and "hash mismatch" in r.stderr
    assert _fnv1a64_hex(body) != "0123456789abcdef"


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["ket", "density"])
def test_reference_master_with_gpu_workers(tmp_path, mode):
    """Two GPU workers serve the reference master; the aggregated amplitude equals run_serial."""
    assert os.path.exists(REFGEN), "oracle/_ref not built"
    stem = "cfg1_n20_p1_s1_m4"
    pay = tmp_path / "p.json"
    pay.write_bytes(_payload_text(stem))
    m = subprocess.Popen([REFGEN, "master", "--payload", str(pay), "--workers", "2", "--batch", "8"],
                         stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    try:
        port = json.loads(m.stdout.readline())["port"]
        ws = [subprocess.Popen([WORKER, "--connect", f"127.0.0.1:{port}", "--id", str(i), "--mode", mode],
                               stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for i in range(2)]
        out, err = m.communicate(timeout=300)
        rep = json.loads(out.strip().splitlines()[-1])
        ok = 0
        for w in ws:
            w.wait(timeout=60)
            msg = w.stderr.read()
            # a worker that connects after the master has handed out every batch finds the
            # connection closed -- the reference worker reports the same (worker.cpp:57-60)
            assert w.returncode == 0 or "lost connection" in msg, msg
            ok += w.returncode == 0
        assert ok >= 1
    finally:
        if m.poll() is None:
            m.kill()
    want = cx(ref_json(stem)["run_serial"])
    got = complex(*rep["amplitude"])
    assert rep["jobs"] == 256 and rep["batches"] == 32
    assert abs(got - want) <= 1e-10 * abs(want)
