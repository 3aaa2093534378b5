"""File access for the CLI phases, with an access audit (reference hegwas/io.py:1-89).

The compute phase must prove it never opened the secret key: every read and write made
through this module inside an ``audit_file_access()`` scope is recorded as (mode, absolute
path).  Writes are atomic (temporary file + rename).  Formats: HEGW binaries
(serialize.py), JSON with sorted keys, tab-separated tables with ``repr`` floats -- the same
artifacts the reference writes, so the phases of the two packages interoperate.
"""
from __future__ import annotations

import contextvars
import json
import os
from contextlib import contextmanager
from pathlib import Path

_AUDITS: contextvars.ContextVar[tuple] = contextvars.ContextVar("hg_b200_audits", default=())


@contextmanager
def audit_file_access():
    """Yields a list that receives (mode, absolute path) for every access in scope."""
    entries: list[tuple[str, str]] = []
    token = _AUDITS.set(_AUDITS.get() + (entries,))
    try:
        yield entries
    finally:
        _AUDITS.reset(token)


def _record(mode: str, path) -> Path:
    path = Path(path)
    resolved = str(path.resolve())
    for entries in _AUDITS.get():
        entries.append((mode, resolved))
    return path


def _atomic_write(path: Path, data, text: bool) -> None:
    path.parent.mkdir(parents=True, exist_ok=True)
    tmp = path.with_name(path.name + ".tmp")
    if text:
        tmp.write_text(data)
    else:
        tmp.write_bytes(data)
    os.replace(tmp, path)


def read_bytes(path) -> bytes:
    return _record("read", path).read_bytes()


def write_bytes(path, data: bytes) -> None:
    _atomic_write(_record("write", path), data, text=False)


def read_text(path) -> str:
    return _record("read", path).read_text()


def write_text(path, text: str) -> None:
    _atomic_write(_record("write", path), text, text=True)


def read_json(path):
    return json.loads(read_text(path))


def write_json(path, obj) -> None:
    write_text(path, json.dumps(obj, indent=2, sort_keys=True) + "\n")


def write_tsv(path, header, rows) -> None:
    def cell(v):
        return repr(v) if isinstance(v, float) else str(v)

    body = ["\t".join(header)] + ["\t".join(cell(v) for v in row) for row in rows]
    write_text(path, "\n".join(body) + "\n")


def read_tsv(path) -> tuple[list[str], list[list[str]]]:
    lines = read_text(path).splitlines()
    if not lines:
        return [], []
    return lines[0].split("\t"), [ln.split("\t") for ln in lines[1:] if ln]
