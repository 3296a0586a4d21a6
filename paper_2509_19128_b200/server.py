"""The reference engine's wire protocol over the device engine (SURVEY 8f
rank 1): the three mirrored endpoints of /root/reference/proj/docs/protocol.md
and the scripted control plane, on top of ``Engine`` -- so the reference's
HTTP clients, scenario scripts and protocol tests drive the B200 path.

  POST /v1/chat/completions   {prompt_id, max_tokens, seed, terminator[, prompt_tokens]}
                              -> chunked application/x-ndjson token events + a done line
  POST /init_process_group    {members} -> {group_id, size}  (FNV-1a of the sorted members)
  POST /request_weight_update {new_version, policy, checksum[, group_id]}
                              -> 200 {applied_version} | 409 version_conflict |
                                 400 checksum_mismatch / policy_mismatch / invalid_policy / bad_request
  GET  /healthz, POST /admin/{pause,advance,resume}, GET /admin/state

Handlers follow EngineServer (core/src/protocol.cpp:83-219): the checksum is
CRC-32 over the compact serialization of `policy` (the device srl_crc32),
versions are strictly sequential and a rejected update leaves the engine
untouched.  The stdlib threading server keeps this dependency-free; a
streaming response holds its thread while the engine produces events.
"""
from __future__ import annotations

import json
import threading
from http.server import BaseHTTPRequestHandler, ThreadingHTTPServer

from .engine import Engine, crc32
from .policy import policy_from_dict


def compact_json(obj) -> bytes:
    """The reference's compact serialization (nlohmann::json::dump(): no
    spaces, object keys in sorted order, shortest round-trip numbers) -- the
    bytes the checksum of /request_weight_update covers."""
    return json.dumps(obj, separators=(",", ":"), ensure_ascii=False, sort_keys=True).encode()


class EngineServer:
    def __init__(self, engine: Engine, host: str = "127.0.0.1", port: int = 0):
        self.engine = engine
        self.update_lock = threading.Lock()
        srv = self

        class Handler(BaseHTTPRequestHandler):
            protocol_version = "HTTP/1.1"

            def log_message(self, *args):  # quiet
                pass

            def _body(self):
                n = int(self.headers.get("Content-Length", "0"))
                raw = self.rfile.read(n) if n else b""
                return json.loads(raw) if raw else {}

            def _send(self, code, obj):
                data = compact_json(obj)
                self.send_response(code)
                self.send_header("Content-Type", "application/json")
                self.send_header("Content-Length", str(len(data)))
                self.end_headers()
                self.wfile.write(data)

            def _chunk(self, obj):
                line = compact_json(obj) + b"\n"
                self.wfile.write(b"%x\r\n%s\r\n" % (len(line), line))
                self.wfile.flush()

            def do_GET(self):
                if self.path == "/healthz":
                    return self._send(200, srv.health())
                if self.path == "/admin/state":
                    return self._send(200, srv.state())
                self._send(404, {"error": "not_found"})

            def do_POST(self):
                try:
                    body = self._body()
                except (ValueError, json.JSONDecodeError):
                    return self._send(400, {"error": "bad_request"})
                if self.path == "/v1/chat/completions":
                    return self._completions(body)
                if self.path == "/init_process_group":
                    return self._send(*srv.init_process_group(body))
                if self.path == "/request_weight_update":
                    return self._send(*srv.request_weight_update(body))
                if self.path == "/admin/pause":
                    srv.engine.pause()
                    return self._send(200, {})
                if self.path == "/admin/resume":
                    srv.engine.resume()
                    return self._send(200, {})
                if self.path == "/admin/advance":
                    rounds = int(body.get("rounds", 1))
                    try:
                        n = srv.engine.advance(rounds)
                    except Exception as e:  # logic_error: not paused
                        return self._send(409, {"error": "not_paused", "detail": str(e)})
                    return self._send(200, {"rounds": rounds, "tokens_emitted": n})
                self._send(404, {"error": "not_found"})

            def _completions(self, body):
                try:
                    prompt_id = str(body["prompt_id"])
                    max_tokens = int(body["max_tokens"])
                    seed = int(body.get("seed", 0))
                    term = int(body.get("terminator", -1))
                    prompt = [int(t) for t in body.get("prompt_tokens", [])]
                    sid = srv.engine.open_stream(prompt_id, max_tokens, seed, term, prompt)
                except (KeyError, TypeError, ValueError) as e:
                    return self._send(400, {"error": "bad_request", "detail": str(e)})
                self.send_response(200)
                self.send_header("Content-Type", "application/x-ndjson")
                self.send_header("Transfer-Encoding", "chunked")
                self.end_headers()
                reason = "running"
                while True:
                    evs, reason, more = srv.engine.wait_events(sid)
                    for e in evs:
                        self._chunk({"stream_id": sid, "position": e.position, "token": e.token,
                                     "logprob": e.logprob, "weight_version": e.weight_version})
                    if not more or (not evs and reason != "running"):
                        break
                self._chunk({"done": True, "stream_id": sid, "finish_reason": reason})
                self.wfile.write(b"0\r\n\r\n")
                self.wfile.flush()

        self.httpd = ThreadingHTTPServer((host, port), Handler)
        self.httpd.daemon_threads = True
        self.port = self.httpd.server_address[1]
        self.thread = None

    # ------------------------------------------------------------ handlers ---
    def health(self):
        e = self.engine
        return {"status": "ok", "weight_version": e.weight_version(), "active_streams": e.active_streams(),
                "total_streams": e.total_streams(), "recompute_state": e.recompute_state_mode()}

    def state(self):
        e = self.engine
        return {"weight_version": e.weight_version(), "active_streams": e.active_streams(),
                "total_streams": e.total_streams(), "rounds_done": e.rounds_done(),
                "group_id": e.process_group_id()}

    def init_process_group(self, body):
        members = body.get("members")
        if not isinstance(members, list) or not members or not all(isinstance(m, str) for m in members):
            return 400, {"error": "bad_request"}
        from .engine import process_group_id

        gid = process_group_id(members)
        self.engine.set_process_group(gid, members)
        return 200, {"group_id": gid, "size": len(members)}

    def request_weight_update(self, body):
        # protocol.cpp:147-190, in its order: fields, checksum, policy, apply
        new_version = body.get("new_version", -1) if isinstance(body, dict) else -1
        if not isinstance(body, dict) or "policy" not in body or "checksum" not in body or \
                not isinstance(new_version, int) or new_version < 0:
            return 400, {"error": "bad_request: missing field"}
        with self.update_lock:
            if crc32(compact_json(body["policy"])) != int(body["checksum"]):
                return 400, {"error": "checksum_mismatch", "current_version": self.engine.weight_version()}
            try:
                policy = policy_from_dict(body["policy"])
            except (KeyError, TypeError, ValueError) as e:
                return 400, {"error": f"invalid_policy: {e}"}
            res = self.engine.apply_weight_update(new_version, policy)  # engine.cpp:79-117
            if res.applied:
                return 200, {"applied_version": res.version}
            return (409 if res.error == "version_conflict" else 400), {"error": res.error,
                                                                         "current_version": res.version}

    # ----------------------------------------------------------- lifecycle ---
    def start(self):
        self.thread = threading.Thread(target=self.httpd.serve_forever, daemon=True)
        self.thread.start()
        return self

    def stop(self):
        self.httpd.shutdown()
        self.httpd.server_close()
