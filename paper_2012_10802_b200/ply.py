"""ASCII PLY point clouds, byte-compatible with save_ply / load_ply
(road_geometry.cpp:190-230 of the reference): a fixed header, then one
"x y z" line per vertex with the default iostream float formatting (%g,
6 significant digits).  Host-side file I/O around the device reprojection."""
from __future__ import annotations

import numpy as np


def save_ply(cloud, path) -> None:
    pts = np.asarray(cloud, np.float32).reshape(-1, 3)
    with open(path, "w") as f:
        f.write("ply\nformat ascii 1.0\nelement vertex %d\n"
                "property float x\nproperty float y\nproperty float z\nend_header\n" % len(pts))
        for x, y, z in pts.astype(np.float64):
            f.write(f"{x:g} {y:g} {z:g}\n")


def load_ply(path) -> np.ndarray:
    n = None
    rows = []
    with open(path) as f:
        header = True
        for line in f:
            tok = line.split()
            if header:
                if len(tok) >= 3 and tok[0] == "element" and tok[1] == "vertex":
                    n = int(tok[2])
                elif tok and tok[0] == "end_header":
                    header = False
                continue
            if len(rows) == n:
                break
            if len(tok) >= 3:
                rows.append([float(tok[0]), float(tok[1]), float(tok[2])])
    if n is None or len(rows) != n:
        raise RuntimeError(f"malformed PLY: {path}")
    return np.asarray(rows, np.float32).reshape(-1, 3)
