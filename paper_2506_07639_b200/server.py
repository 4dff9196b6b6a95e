"""`/v1/completions` front for the engine.

Serves the completions contract the reference's `RemoteBackend` speaks
(`/root/reference/pkg/src/ecot_sched/backends.py:285-379`): POST
`{"prompt": str, "max_tokens": int, "stream": false}` to `/v1/completions`,
reply `{"choices": [{"text": str}], "usage": {"completion_tokens": int}}`.
So the unmodified reference `RemoteBackend` and its runners can drive the
B200 engine over HTTP, and the reference's stub-contract tests
(`pkg/tests/test_remote.py`) have a real server to run against.

Prompt -> model input (builder-defined, like the in-process framing):
the reference `default_prompt_builder` (`backends.py:331-333`) sends
`"{instruction}\\n[{step}]\\n{prefix ids}"`; that is parsed back into the
context (`encode_context(instruction, observation)`), the step tag and the
prefix ids, i.e. exactly the request `EngineBackend.begin_step` would run.
The default prompt carries no observation (SURVEY §8(f) caveat (i)): the
server uses `observation` from the request body when present (hex), else
its configured default.  Any other prompt is a free-text completion of
`encode_context(prompt, observation)` with the tag of step "completion".
The engine decodes exactly `max_tokens` greedy tokens (random-init weights
never emit a stop token); the reply text is the token ids, space separated
(so a client can parse them back; `RemoteBackend` instead synthesises ids
from the text, `backends.py:375-378`, which is why token-level parity does
not go over this path).

Batching: HTTP handler threads only enqueue; one worker thread owns the
engine, takes every request that arrived within `batch_window_ms` of the
first, prepares them all (deferred, `EngineBackend.begin_completion`) and
resolves them -- the first read submits the whole group, which decodes as
one continuous batch.

Errors: malformed body -> 400 (not retried by the reference client); an
engine rejection (`EngineError`, e.g. KV pool exhausted) -> 503, which the
reference client retries with backoff (`_RETRYABLE_STATUSES`,
`backends.py:280`); a request the worker cannot finish in `timeout_s` -> 504.
"""

from __future__ import annotations

import json
import queue
import re
import threading
import time
from http.server import BaseHTTPRequestHandler, ThreadingHTTPServer
from typing import Optional

from .backends import BackendError, encode_context
from .engine_backend import REQUEST_CAP

_DEFAULT_PROMPT = re.compile(r"\A(?P<instr>[^\n]*)\n\[(?P<step>[^\]\n]+)\]\n(?P<prefix>[0-9 ]*)\Z")


def parse_prompt(prompt: str) -> tuple[str, str, tuple[int, ...]]:
    """(instruction, step name, prefix ids) of a reference-builder prompt;
    free text -> (prompt, "completion", ())."""
    m = _DEFAULT_PROMPT.match(prompt)
    if m is None:
        return prompt, "completion", ()
    prefix = tuple(int(t) for t in m.group("prefix").split())
    return m.group("instr"), m.group("step"), prefix


class _Job:
    __slots__ = ("instruction", "step", "prefix", "observation", "max_tokens", "done", "status", "payload")

    def __init__(self, instruction, step, prefix, observation, max_tokens):
        self.instruction, self.step, self.prefix = instruction, step, prefix
        self.observation, self.max_tokens = observation, max_tokens
        self.done = threading.Event()
        self.status, self.payload = 500, b""

    def finish(self, status: int, body: Optional[dict]) -> None:
        self.status = status
        self.payload = json.dumps(body).encode() if body is not None else b""
        self.done.set()


class CompletionServer:
    """`with CompletionServer(backend) as srv: srv.url` -- a loopback (or
    `host`) HTTP server over one `EngineBackend`."""

    def __init__(self, backend, host: str = "127.0.0.1", port: int = 0, observation: bytes = b"",
                 batch_window_ms: float = 2.0, max_batch: int = 256, timeout_s: float = 600.0):
        self.backend = backend
        self.observation = observation
        self.batch_window = batch_window_ms / 1000.0
        self.max_batch = max_batch
        self.timeout_s = timeout_s
        self.jobs: "queue.Queue[_Job]" = queue.Queue()
        self.stats = {"requests": 0, "batches": 0, "max_batch": 0, "errors": 0, "tokens": 0}
        self._stop = threading.Event()
        outer = self

        class Handler(BaseHTTPRequestHandler):
            protocol_version = "HTTP/1.1"

            def _reply(self, status: int, payload: bytes = b"") -> None:
                self.send_response(status)
                if payload:
                    self.send_header("Content-Type", "application/json")
                self.send_header("Content-Length", str(len(payload)))
                self.end_headers()
                if payload:
                    self.wfile.write(payload)

            def do_GET(self):  # noqa: N802 (http.server API)
                if self.path == "/health":
                    self._reply(200, b'{"status": "ok"}')
                elif self.path == "/v1/models":
                    name = getattr(outer.backend.cfg, "name", "fastecot")
                    self._reply(200, json.dumps({"data": [{"id": name, "object": "model"}]}).encode())
                else:
                    self._reply(404)

            def do_POST(self):  # noqa: N802
                length = int(self.headers.get("Content-Length", 0) or 0)
                raw = self.rfile.read(length) if length else b""
                if self.path != "/v1/completions":
                    self._reply(404)
                    return
                job, err = outer._job_from(raw)
                if job is None:
                    outer.stats["errors"] += 1
                    self._reply(400, json.dumps({"error": err}).encode())
                    return
                if job.max_tokens == 0:  # the contract's short circuit (backends.py:294-295)
                    self._reply(200, json.dumps({"choices": [{"text": ""}],
                                                 "usage": {"completion_tokens": 0}}).encode())
                    return
                outer.jobs.put(job)
                if not job.done.wait(outer.timeout_s):
                    self._reply(504)
                    return
                self._reply(job.status, job.payload)

            def log_message(self, *args):
                pass

        self._http = ThreadingHTTPServer((host, port), Handler)
        self._http.daemon_threads = True
        self._serve = threading.Thread(target=self._http.serve_forever, daemon=True)
        self._worker = threading.Thread(target=self._work, daemon=True)

    # -- request parsing ---------------------------------------------------------
    def _job_from(self, raw: bytes):
        try:
            body = json.loads(raw) if raw else {}
        except ValueError:
            return None, "body is not JSON"
        if not isinstance(body, dict):
            return None, "body must be an object"
        prompt, max_tokens = body.get("prompt"), body.get("max_tokens", 16)
        if not isinstance(prompt, str):
            return None, "prompt must be a string"
        if not isinstance(max_tokens, int) or isinstance(max_tokens, bool) or not 0 <= max_tokens <= REQUEST_CAP:
            return None, f"max_tokens must be an integer in [0, {REQUEST_CAP}]"
        if body.get("stream", False):
            return None, "stream is not supported"
        obs = self.observation
        if "observation" in body:
            try:
                obs = bytes.fromhex(body["observation"])
            except (TypeError, ValueError):
                return None, "observation must be hex"
        instr, step, prefix = parse_prompt(prompt)
        return _Job(instr, step, prefix, obs, max_tokens), None

    # -- the engine worker --------------------------------------------------------
    def _work(self) -> None:
        be = self.backend
        while not self._stop.is_set():
            try:
                first = self.jobs.get(timeout=0.05)
            except queue.Empty:
                continue
            batch = [first]
            deadline = time.monotonic() + self.batch_window
            while len(batch) < self.max_batch:
                left = deadline - time.monotonic()
                if left <= 0:
                    break
                try:
                    batch.append(self.jobs.get(timeout=left))
                except queue.Empty:
                    break
            self.stats["batches"] += 1
            self.stats["max_batch"] = max(self.stats["max_batch"], len(batch))
            try:
                self._serve_batch(be, batch)
            except Exception as exc:  # never leave a client waiting on a dead worker
                self.stats["errors"] += 1
                for job in batch:
                    if not job.done.is_set():
                        job.finish(500, {"error": f"internal error: {exc!r}"})

    def _serve_batch(self, be, batch) -> None:
        gens = []
        for job in batch:   # prepare all (deferred): they decode as one batch
            try:
                ctx = encode_context(job.instruction, job.observation)
                gens.append((job, be.begin_completion(ctx, job.prefix, job.step, job.max_tokens)))
            except BackendError as exc:
                self.stats["errors"] += 1
                job.finish(503, {"error": str(exc)})
        for job, gen in gens:
            try:
                toks = tuple(gen.tokens)
            except BackendError as exc:
                self.stats["errors"] += 1
                job.finish(503, {"error": str(exc)})
                continue
            self.stats["requests"] += 1
            self.stats["tokens"] += len(toks)
            job.finish(200, {"object": "text_completion",
                             "choices": [{"index": 0, "text": " ".join(str(t) for t in toks),
                                          "finish_reason": "length"}],
                             "usage": {"completion_tokens": len(toks)}})

    # -- lifetime -----------------------------------------------------------------
    @property
    def url(self) -> str:
        host, port = self._http.server_address[:2]
        return f"http://{host}:{port}"

    def start(self) -> "CompletionServer":
        self._worker.start()
        self._serve.start()
        return self

    def stop(self) -> None:
        self._stop.set()
        self._http.shutdown()
        self._http.server_close()
        self._worker.join(timeout=5)

    def __enter__(self) -> "CompletionServer":
        return self.start()

    def __exit__(self, *exc) -> None:
        self.stop()


def main(argv=None) -> None:
    """python -m paper_2506_07639_b200.server --config 7b --dtype bf16 --port 8000"""
    import argparse

    from .engine_backend import EngineBackend
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--host", default="127.0.0.1")
    ap.add_argument("--port", type=int, default=8000)
    ap.add_argument("--observation", default="", help="hex bytes of the default observation")
    args = ap.parse_args(argv)
    be = EngineBackend(args.config, dtype=args.dtype)
    srv = CompletionServer(be, args.host, args.port, observation=bytes.fromhex(args.observation)).start()
    print(f"serving /v1/completions on {srv.url}", flush=True)
    try:
        while True:
            time.sleep(3600)
    except KeyboardInterrupt:
        srv.stop()
        be.close()


if __name__ == "__main__":
    main()
