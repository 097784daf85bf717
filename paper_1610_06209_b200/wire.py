"""Result-table wire format of the reference's drivers (proj/tools/spinners_cli.cpp:26-51,165-176,
120-145,218-230): every table starts with one ``# {json}`` echo line — the command, its config and
the library tag, serialised like nlohmann::json::dump() (keys sorted, no whitespace) — followed by a
CSV header and rows whose floating-point fields are printed with ``%.17g`` (round-trip exact).

This module writes (and reads back) those tables for the results this package computes on the GPU:
collision curves / family comparisons (``collision_curve``, ``compare_families``), sketched Newton
traces (``solve``) and kernel-approximation errors (``gram_error``), so the files are byte-compatible
with the reference CLI's output for the same numbers.
"""
from __future__ import annotations

import io
import json
import math
from typing import Iterable, Sequence

LIBRARY = "spinners 1.0"  # spinners_cli.cpp:49


def fmt17(v: float) -> str:
    """spinners_cli.cpp:26-30: snprintf("%.17g")."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.17g" % v


def dump_json(obj) -> str:
    """nlohmann::json::dump() with no indent: object keys in sorted order, ',' and ':' separators,
    doubles in shortest round-trip form, non-ASCII kept as UTF-8."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), ensure_ascii=False, allow_nan=False)


def emit_config(out, command: str, config: dict) -> None:
    """spinners_cli.cpp:48-51: ``# {"command":...,"config":{...},"library":"spinners 1.0"}``."""
    out.write("# " + dump_json({"command": command, "config": config, "library": LIBRARY}) + "\n")


def emit_curve(out, curve, second=None, diffs: Sequence[float] | None = None) -> None:
    """spinners_cli.cpp:165-176: bucket_low,bucket_high,count,probability (+ prob_b, abs_diff)."""
    out.write("bucket_low,bucket_high,count,prob_a,prob_b,abs_diff\n" if second is not None
              else "bucket_low,bucket_high,count,probability\n")
    edges, probs, counts = curve.bucket_edges, curve.probabilities, curve.counts
    for b in range(len(edges) - 1):
        row = f"{fmt17(edges[b])},{fmt17(edges[b + 1])},{int(counts[b])},{fmt17(probs[b])}"
        if second is not None:
            row += f",{fmt17(second.probabilities[b])},{fmt17(diffs[b])}"
        out.write(row + "\n")


def write_lsh_collision(out, config: dict, curve) -> None:
    """The ``lsh-collision`` table (spinners_cli.cpp:178-189)."""
    emit_config(out, "lsh-collision", config)
    emit_curve(out, curve)


def write_lsh_compare(out, config: dict, cmp) -> None:
    """The ``lsh-compare`` table (spinners_cli.cpp:191-205): echo, ``# sup_difference``, the curves."""
    emit_config(out, "lsh-compare", config)
    out.write(f"# sup_difference {fmt17(cmp.sup_difference)}\n")
    emit_curve(out, cmp.curve_a, cmp.curve_b, cmp.bucket_differences)


def write_newton_sketch(out, config: dict, trace) -> None:
    """The ``newton-sketch`` table (spinners_cli.cpp:207-232): iter,loss,gap,seconds."""
    emit_config(out, "newton-sketch", config)
    out.write("iter,loss,gap,seconds\n")
    for t in range(len(trace.losses)):
        out.write(f"{t},{fmt17(trace.losses[t])},{fmt17(trace.gaps[t])},{fmt17(trace.seconds[t])}\n")


def write_kernel_approx(out, config: dict, rows: Iterable[tuple[int, float, float]]) -> None:
    """The ``kernel-approx`` table (spinners_cli.cpp:114-146): features,mean_error,sd_error."""
    emit_config(out, "kernel-approx", config)
    out.write("features,mean_error,sd_error\n")
    for dprime, mean, sd in rows:
        out.write(f"{int(dprime)},{fmt17(mean)},{fmt17(sd)}\n")


def read_table(text: str):
    """Parse a table back: (echo dict, extra '# ' comment lines, header, rows of float/int fields)."""
    lines = text.splitlines()
    if not lines or not lines[0].startswith("# "):
        raise ValueError("missing '# {json}' echo line")
    echo = json.loads(lines[0][2:])
    comments, i = [], 1
    while i < len(lines) and lines[i].startswith("# "):
        comments.append(lines[i][2:])
        i += 1
    header = lines[i].split(",")

    def num(f):
        try:
            return int(f)
        except ValueError:
            return float(f)
    rows = [[num(f) for f in ln.split(",")] for ln in lines[i + 1:] if ln]
    return echo, comments, header, rows


def to_string(writer, *args) -> str:
    buf = io.StringIO()
    writer(buf, *args)
    return buf.getvalue()
