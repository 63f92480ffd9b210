"""Snapshot output of the march: the reference's NWAV
binary container and the flat CSV table, byte-compatible with
``pkg/src/nwave/fieldio.py:31-81`` so files written here load in the
reference (and vice versa).

NWAV layout, little-endian: a 48-byte header -- magic ``NWAV``, u32 version
(1), u64 n_outer, u64 n_inner, f64 d_outer, f64 d_inner, f64 aux (the sigma
of a field snapshot; 0 for (sigma, rho) coefficient tables) -- followed by
n_outer * n_inner f64 values, outer index slowest.

``SnapshotWriter`` streams the snapshots of a ``RunReport`` (or of an
ensemble) to disk the way the reference CLI's ``_write_snapshots`` names
them (``pkg/src/nwave/cli.py:111-123``).
"""

from __future__ import annotations

import os

import numpy as np

from .grid import Field2D

MAGIC = b"NWAV"
VERSION = 1
_HEAD = np.dtype([("magic", "S4"), ("version", "<u4"), ("n0", "<u8"), ("n1", "<u8"),
                  ("d0", "<f8"), ("d1", "<f8"), ("aux", "<f8")])
assert _HEAD.itemsize == 48


def write_grid_binary(path, values, d0: float, d1: float, aux: float = 0.0) -> None:
    """One 2-D float64 array in the NWAV container (reference ``fieldio.py:47-55``)."""
    data = np.ascontiguousarray(values, dtype="<f8")
    if data.ndim != 2:
        raise ValueError("binary grid format stores 2-D arrays only")
    head = np.zeros((), _HEAD)
    head["magic"], head["version"] = MAGIC, VERSION
    head["n0"], head["n1"] = data.shape
    head["d0"], head["d1"], head["aux"] = float(d0), float(d1), float(aux)
    with open(path, "wb") as fh:
        fh.write(head.tobytes())
        fh.write(memoryview(data).cast("B"))


def read_grid_binary(path):
    """Returns (values, d0, d1, aux); raises IOError on a malformed file."""
    with open(path, "rb") as fh:
        raw = fh.read(_HEAD.itemsize)
        if len(raw) < _HEAD.itemsize:
            raise IOError(f"{path}: truncated header")
        head = np.frombuffer(raw, _HEAD)[0]
        if bytes(head["magic"]) != MAGIC:
            raise IOError(f"{path}: bad magic {bytes(head['magic'])!r}")
        if int(head["version"]) != VERSION:
            raise IOError(f"{path}: unsupported version {int(head['version'])}")
        n0, n1 = int(head["n0"]), int(head["n1"])
        body = fh.read(8 * n0 * n1)
        if len(body) != 8 * n0 * n1:
            raise IOError(f"{path}: truncated payload")
    vals = np.frombuffer(body, "<f8").reshape(n0, n1).astype(np.float64)
    return vals, float(head["d0"]), float(head["d1"]), float(head["aux"])


def write_field_binary(path, field: Field2D, d_rho: float, d_theta: float, sigma: float) -> None:
    write_grid_binary(path, field.values, d_rho, d_theta, sigma)


def read_field_binary(path):
    """Returns (field, d_rho, d_theta, sigma)."""
    vals, d0, d1, aux = read_grid_binary(path)
    return Field2D(vals), d0, d1, aux


def write_field_csv(path, field: Field2D, rho_nodes, theta_nodes) -> None:
    """Rows ``rho,theta,V`` (rho outer), as ``np.savetxt`` formats them in the
    reference (``fieldio.py:74-81``)."""
    rho_nodes = np.asarray(rho_nodes, np.float64)
    theta_nodes = np.asarray(theta_nodes, np.float64)
    if field.values.shape != (len(rho_nodes), len(theta_nodes)):
        raise ValueError("write_field_csv: axes do not match field extents")
    nr, nt = field.values.shape
    table = np.empty((nr * nt, 3))
    table[:, 0] = np.repeat(rho_nodes, nt)
    table[:, 1] = np.tile(theta_nodes, nr)
    table[:, 2] = field.values.reshape(-1)
    np.savetxt(path, table, delimiter=",", header="rho,theta,V", comments="")


class SnapshotWriter:
    """Writes snapshots as ``V_sigma<sigma:08.3f>.bin`` (dot -> ``p``) plus a
    ``.csv`` into ``outdir`` -- the reference CLI's names -- one call per
    field, so a march's snapshots can be flushed as they reach the host.
    ``tag`` (e.g. an ensemble member) is inserted after ``V``."""

    def __init__(self, outdir, config, csv: bool = True):
        from .grid import build_axes

        self.outdir = str(outdir)
        self.config = config
        self.csv = csv
        _, self.rho, self.theta = build_axes(config)
        os.makedirs(self.outdir, exist_ok=True)
        self.paths: list[str] = []

    def write(self, sigma: float, field: Field2D, tag: str = "") -> list[str]:
        stem = os.path.join(self.outdir, f"V{tag}_sigma{sigma:08.3f}".replace(".", "p"))
        # (the dot substitution applies to the file name only: outdir is joined after)
        out = [stem + ".bin"]
        write_field_binary(out[0], field, self.config.d_rho, self.config.d_theta, sigma)
        if self.csv:
            out.append(stem + ".csv")
            write_field_csv(out[1], field, self.rho, self.theta)
        self.paths.extend(out)
        return out

    def write_report(self, report, tag: str = "") -> list[str]:
        """Every snapshot of a ``RunReport`` in sigma order."""
        out = []
        for sigma, field in sorted(report.snapshots.items()):
            out += self.write(sigma, field, tag)
        return out
