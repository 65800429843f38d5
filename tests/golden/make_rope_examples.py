"""Writes the d >= 4, m >= 1 cases of rope_examples.json from S:98's definition
(angles[m][i] = m * theta^(-2i/d)) and Eq. 3's 2x2 rotation, one
pair at a time with the math module (no oracle, no numpy)."""
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def rotate(x, m, base, style):
    d = len(x)
    out = [0.0] * d
    for i in range(d // 2):
        ang = m * base ** (-2.0 * i / d)
        a, b = (i, i + d // 2) if style == "half" else (2 * i, 2 * i + 1)
        out[a] = x[a] * math.cos(ang) - x[b] * math.sin(ang)
        out[b] = x[a] * math.sin(ang) + x[b] * math.cos(ang)
    return out


def main():
    path = os.path.join(HERE, "rope_examples.json")
    g = json.load(open(path))
    keep = [c for c in g["cases"] if "style" not in c]
    new = []
    for style in ("half", "interleaved"):
        new.append({"name": f"d4_m1_{style}", "style": style, "d": 4, "x": [1.0, 2.0, 3.0, 4.0], "m": 1,
                    "base": 10000.0, "expr": "theta = (1, 0.01): pairs rotated by 1 rad and 0.01 rad",
                    "expected": rotate([1.0, 2.0, 3.0, 4.0], 1, 10000.0, style)})
        x = [0.5, -1.0, 2.0, 0.25, -0.75, 1.5, -2.0, 1.0]
        new.append({"name": f"d8_m3_base100_{style}", "style": style, "d": 8, "x": x, "m": 3, "base": 100.0,
                    "expr": "angles 3 * 10^(-i/2) = [3, 3/sqrt(10), 0.3, 0.3/sqrt(10)]",
                    "expected": rotate(x, 3, 100.0, style)})
    g["cases"] = keep + new
    json.dump(g, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
