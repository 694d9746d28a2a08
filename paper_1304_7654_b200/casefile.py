"""Case-file text format: parser, loader and writer.

The grammar is the reference's (mesh.py:1-19, 137-300; cases.py:156-183):
``[case]`` / ``[block <id>]`` / ``[cut <id>]`` sections of ``key = value``
lines, ``#`` comments, unknown sections or keys rejected, ids contiguous from
0.  Error classes and messages match so existing case files and tooling keep
working unchanged.
"""

from __future__ import annotations

import os

from .exceptions import ConfigError
from .topology import FACES, BlockSpec, CaseConfig, CutSide, CutSpec

_SCHEMA = {
    "case": {"nharms": int, "npde": int, "iterations": int,
             "dtau": float, "omega": float, "nbody": int},
    "block": {"ni": int, "nj": int, "x0": float, "y0": float,
              "h": float, "body_faces": str},
    "cut": {"block_a": int, "face_a": str, "range_a": str,
            "block_b": int, "face_b": str, "range_b": str,
            "orientation": str},
}


def _section_key(line, lineno, source):
    if not line.endswith("]"):
        raise ConfigError("unterminated section header", lineno, source)
    words = line[1:-1].split()
    if words == ["case"]:
        return ("case",)
    if len(words) == 2 and words[0] in ("block", "cut"):
        try:
            return (words[0], int(words[1]))
        except ValueError:
            raise ConfigError(f"non-integer {words[0]} id {words[1]!r}", lineno, source)
    raise ConfigError(f"unknown section {line!r}", lineno, source)


def _tokenize(text, source):
    """Split text into {section key: {name: (raw value, line number)}}."""
    sections = {}
    current = None
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            key = _section_key(line, lineno, source)
            if key in sections:
                raise ConfigError(f"duplicate section {line!r}", lineno, source)
            sections[key] = current_items = {}
            current = key
            continue
        if "=" not in line:
            raise ConfigError(f"expected 'key = value', got {line!r}", lineno, source)
        if current is None:
            raise ConfigError("key outside any section", lineno, source)
        name, _, value = (part.strip() for part in line.partition("="))
        if name not in _SCHEMA[current[0]]:
            raise ConfigError(f"unknown key {name!r} in [{' '.join(map(str, current))}]",
                              lineno, source)
        if name in current_items:
            raise ConfigError(f"duplicate key {name!r}", lineno, source)
        current_items[name] = (value, lineno)
    return sections


def _value(items, name, conv, source):
    if name not in items:
        raise ConfigError(f"missing key {name!r}", None, source)
    raw, lineno = items[name]
    try:
        return conv(raw)
    except ValueError:
        raise ConfigError(f"bad value for {name!r}: {raw!r}", lineno, source)


def _range(raw, lineno, source):
    bounds = raw.split(":")
    if len(bounds) != 2:
        raise ConfigError(f"range must be 'lo:hi', got {raw!r}", lineno, source)
    try:
        lo, hi = int(bounds[0]), int(bounds[1])
    except ValueError:
        raise ConfigError(f"non-integer range bound in {raw!r}", lineno, source)
    if lo < 1 or hi < lo:
        raise ConfigError(f"empty or negative range {raw!r}", lineno, source)
    return lo, hi


def _body_faces(raw, lineno, source):
    if not raw.strip():
        return ()
    out = []
    for item in raw.split(","):
        bits = item.strip().split(":")
        if len(bits) != 2 or bits[0] not in FACES:
            raise ConfigError(f"body face must be '<face>:<body>', got {item!r}",
                              lineno, source)
        try:
            out.append((bits[0], int(bits[1])))
        except ValueError:
            raise ConfigError(f"non-integer body id in {item!r}", lineno, source)
    return tuple(out)


def parse_case(text, source="<string>", name=""):
    """Parse case-file text into a CaseConfig (errors carry the line number)."""
    sections = _tokenize(text, source)
    if ("case",) not in sections:
        raise ConfigError("missing [case] section", None, source)
    head = sections[("case",)]
    params = {k: _value(head, k, conv, source) for k, conv in _SCHEMA["case"].items()}
    checks = (("nharms", lambda v: v >= 0, "nharms must be >= 0"),
              ("npde", lambda v: v == 4, "npde is fixed at 4"),
              ("iterations", lambda v: v >= 0, "iterations must be >= 0"),
              ("dtau", lambda v: v >= 0, "dtau must be >= 0"),
              ("omega", lambda v: v > 0, "omega must be > 0"),
              ("nbody", lambda v: v >= 0, "nbody must be >= 0"))
    for key, ok, msg in checks:
        if not ok(params[key]):
            raise ConfigError(msg, None, source)

    blocks = []
    for key in sorted(k for k in sections if k[0] == "block"):
        items = sections[key]
        dims = {k: _value(items, k, conv, source)
                for k, conv in (("ni", int), ("nj", int), ("x0", float), ("y0", float),
                                ("h", float))}
        faces = ()
        if "body_faces" in items:
            faces = _body_faces(items["body_faces"][0], items["body_faces"][1], source)
        blk = BlockSpec(id=key[1], body_faces=faces, **dims)
        if blk.ni < 2 or blk.nj < 2:
            raise ConfigError(f"block {blk.id}: ni and nj must be >= 2", None, source)
        if blk.h <= 0:
            raise ConfigError(f"block {blk.id}: h must be > 0", None, source)
        blocks.append(blk)

    cut_ids = sorted(k[1] for k in sections if k[0] == "cut")
    if cut_ids != list(range(len(cut_ids))):
        raise ConfigError("cut ids must be contiguous starting at 0", None, source)
    cuts = []
    for ident in cut_ids:
        items = sections[("cut", ident)]
        fa = _value(items, "face_a", str, source)
        fb = _value(items, "face_b", str, source)
        for f in (fa, fb):
            if f not in FACES:
                raise ConfigError(f"cut {ident}: unknown face {f!r}", None, source)
        ra = _range(*items["range_a"], source)
        rb = _range(*items["range_b"], source)
        orient = _value(items, "orientation", str, source)
        if orient not in ("forward", "reversed"):
            raise ConfigError(f"cut {ident}: orientation must be forward|reversed",
                              None, source)
        cuts.append(CutSpec(side_a=CutSide(_value(items, "block_a", int, source), fa, *ra),
                            side_b=CutSide(_value(items, "block_b", int, source), fb, *rb),
                            reversed=orient == "reversed"))

    if [b.id for b in blocks] != list(range(len(blocks))):
        raise ConfigError("block ids must be contiguous starting at 0", None, source)
    return CaseConfig(blocks=blocks, cuts=cuts, name=name, **params)


def load_case(path):
    """Read a case file; the case name is the file stem."""
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    return parse_case(text, source=str(path),
                      name=os.path.splitext(os.path.basename(path))[0])


def case_text(config):
    """Render a CaseConfig in the case-file format (parse_case inverts it)."""
    out = ["[case]"]
    out += [f"{k} = {getattr(config, k)!r}"
            for k in ("nharms", "npde", "iterations", "dtau", "omega", "nbody")]
    for blk in config.blocks:
        out += ["", f"[block {blk.id}]", f"ni = {blk.ni}", f"nj = {blk.nj}",
                f"x0 = {blk.x0!r}", f"y0 = {blk.y0!r}", f"h = {blk.h!r}"]
        if blk.body_faces:
            out.append("body_faces = " + ",".join(f"{f}:{b}" for f, b in blk.body_faces))
    for ci, cut in enumerate(config.cuts):
        a, b = cut.side_a, cut.side_b
        out += ["", f"[cut {ci}]", f"block_a = {a.block}", f"face_a = {a.face}",
                f"range_a = {a.lo}:{a.hi}", f"block_b = {b.block}", f"face_b = {b.face}",
                f"range_b = {b.lo}:{b.hi}",
                f"orientation = {'reversed' if cut.reversed else 'forward'}"]
    return "\n".join(out) + "\n"
