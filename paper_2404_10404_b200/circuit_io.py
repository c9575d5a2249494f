"""Circuit interchange: the reference's JSON (GeneralCircuit::to_json /
from_json, circuit.hpp:227-277) <-> the flat CSR layout of include/dgkr_b200.h,
plus the binary CSR file (dgkr_circuit_save / dgkr_circuit_load) for circuits
too large for JSON."""
from __future__ import annotations

import json
from typing import Any, Dict, Tuple

import numpy as np

from .workloads import Flat


def from_json(obj: Any) -> Tuple[int, Flat]:
    """GeneralCircuit::from_json (circuit.hpp:250-277): {"input_size": n,
    "layers": [[{"nested": [{"op": "add"|"mul", "left": [layer, gate],
    "right": [layer, gate]}, ...]}, ...], ...]} -> (input_size, flat).
    Unknown ops raise ValueError, as the reference's invalid_argument."""
    if isinstance(obj, (str, bytes)):
        obj = json.loads(obj)
    input_size = int(obj["input_size"])
    lgs, gns, rows = [0], [0], []
    for jl in obj["layers"]:
        for jg in jl:
            nested = jg["nested"]
            for jn in nested:
                op = jn["op"]
                if op == "add":
                    kind = 0
                elif op == "mul":
                    kind = 1
                else:
                    raise ValueError(f"unknown gate op: {op}")
                rows.append((kind, int(jn["left"][0]), int(jn["left"][1]), int(jn["right"][0]), int(jn["right"][1])))
            gns.append(gns[-1] + len(nested))
        lgs.append(lgs[-1] + len(jl))
    depth = len(lgs) - 1
    return input_size, (np.array(lgs, np.uint64), np.array(gns, np.uint64),
                        np.array(rows, np.uint32).reshape(-1, 5), np.ones(depth + 1, np.uint64))


def to_json(input_size: int, flat: Flat) -> Dict[str, Any]:
    """GeneralCircuit::to_json (circuit.hpp:227-248), same key order"""
    lgs, gns, nested = flat[0], flat[1], flat[2]
    layers = []
    for li in range(len(lgs) - 1):
        gl = []
        for g in range(int(lgs[li]), int(lgs[li + 1])):
            ns = []
            for k in range(int(gns[g]), int(gns[g + 1])):
                e = nested[k]
                ns.append({"op": "mul" if e[0] else "add", "left": [int(e[1]), int(e[2])],
                           "right": [int(e[3]), int(e[4])]})
            gl.append({"nested": ns})
        layers.append(gl)
    return {"input_size": int(input_size), "layers": layers}


def load_json_file(path: str) -> Tuple[int, Flat]:
    with open(path) as fh:
        return from_json(json.load(fh))


def save_json_file(path: str, input_size: int, flat: Flat) -> None:
    with open(path, "w") as fh:
        json.dump(to_json(input_size, flat), fh, indent=2)
        fh.write("\n")
