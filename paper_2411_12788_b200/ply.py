"""PLY checkpoints of a Gaussian set (ply_io.cpp:87-147): the 3DGS binary
little-endian vertex layout — x y z, nx ny nz (zero), f_dc_0..2, f_rest_0..44 (channel-major:
f_rest[c * 15 + k - 1] = sh[k * 3 + c]), opacity (logit), scale_0..2 (log), rot_0..3 (w x y z),
all float32.  The row transpose runs vectorised on the host copy; read errors raise RuntimeError
with the reference's messages (parse_fail, ply_io.cpp:27-32)."""
from __future__ import annotations

from pathlib import Path

import numpy as np

from .scenes import GaussianSet

_REST = 15


def property_names() -> list[str]:
    """gaussian_property_names (ply_io.cpp:16-25)."""
    names = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
    names += [f"f_rest_{j}" for j in range(_REST * 3)]
    names += ["opacity"] + [f"scale_{j}" for j in range(3)] + [f"rot_{j}" for j in range(4)]
    return names


def _rows(s: GaussianSet) -> np.ndarray:
    n = s.n
    rows = np.zeros((n, 62), np.float32)
    rows[:, 0:3] = s.centers
    sh = np.asarray(s.sh, np.float32).reshape(n, 16, 3)
    rows[:, 6:9] = sh[:, 0, :]
    rows[:, 9:54] = sh[:, 1:, :].transpose(0, 2, 1).reshape(n, 45)  # [c][k-1]
    rows[:, 54] = s.opacity_logits
    rows[:, 55:58] = s.log_scales
    rows[:, 58:62] = s.rotations
    return rows


def write_ply(path, s: GaussianSet) -> None:
    """write_ply (ply_io.cpp:87-111)."""
    s.check_consistent()
    head = ["ply", "format binary_little_endian 1.0", f"element vertex {s.n}"]
    head += [f"property float {n}" for n in property_names()] + ["end_header"]
    try:
        with open(path, "wb") as f:
            f.write(("\n".join(head) + "\n").encode())
            f.write(_rows(s).astype("<f4").tobytes())
    except OSError as e:
        raise RuntimeError(f"{path}: cannot open for writing") from e


def read_ply(path, active_sh_degree: int = 3) -> GaussianSet:
    """read_ply (ply_io.cpp:113-147)."""
    path = str(path)
    try:
        data = Path(path).read_bytes()
    except OSError as e:
        raise RuntimeError(f"{path}: cannot open") from e

    def fail(off, what):
        raise RuntimeError(f"{path}: PLY parse error at byte {off}: {what}")

    pos = 0

    def line():
        nonlocal pos
        end = data.find(b"\n", pos)
        if end < 0:
            return None, pos
        start = pos
        pos = end + 1
        return data[start:end].decode("latin-1"), start

    first, _ = line()
    if first != "ply":
        fail(0, "missing 'ply' magic")
    count, props, saw_format = -1, [], False
    while True:
        ln, start = line()
        if ln is None:
            fail(start, "header ended without 'end_header'")
        words = ln.split()
        word = words[0] if words else ""
        if word == "comment":
            continue
        if word == "format":
            if words[1:3] != ["binary_little_endian", "1.0"]:
                fail(start, f"unsupported format '{ln}'")
            saw_format = True
        elif word == "element":
            if len(words) < 3 or words[1] != "vertex" or int(words[2]) < 0:
                fail(start, f"expected 'element vertex <count>', got '{ln}'")
            if count >= 0:
                fail(start, "multiple vertex elements")
            count = int(words[2])
        elif word == "property":
            if len(words) < 3:
                fail(start, f"malformed property line '{ln}'")
            props.append((words[1], words[2]))
        elif word == "end_header":
            break
        else:
            fail(start, f"unexpected header line '{ln}'")
    if not saw_format:
        fail(start, "missing format line")
    if count < 0:
        fail(start, "missing vertex element")
    names = property_names()
    if len(props) != len(names):
        fail(pos, f"expected {len(names)} vertex properties, found {len(props)}")
    for j, (t, nm) in enumerate(props):
        if t != "float" or nm != names[j]:
            fail(pos, f"property {j} is '{t} {nm}', expected 'float {names[j]}'")
    need = count * 62 * 4
    if len(data) - pos < need:
        fail(pos + (len(data) - pos) // 248 * 248, "truncated vertex data")
    rows = np.frombuffer(data, dtype="<f4", count=count * 62, offset=pos).reshape(count, 62).astype(np.float32)
    sh = np.zeros((count, 16, 3), np.float32)
    sh[:, 0, :] = rows[:, 6:9]
    sh[:, 1:, :] = rows[:, 9:54].reshape(count, 3, 15).transpose(0, 2, 1)
    return GaussianSet(rows[:, 0:3].copy(), rows[:, 55:58].copy(), rows[:, 58:62].copy(), rows[:, 54].copy(),
                       sh.reshape(count, 48), active_sh_degree)
