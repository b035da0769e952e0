"""Golden vectors for parse_edge_list / GSCG cache from the Python reference.

    PYTHONPATH=/tmp/refpkg/src python tests/golden/make_parse_golden.py

(run from a copy of /root/reference/pkg; writes tests/golden/parse_golden.json
and tests/golden/ref_fig1.gscg).  The inputs are generated here
deterministically; the expected outputs are the reference's own."""

import base64
import json
import os
import random

from graphscan import EdgeList, ParseError, build_graph, parse_edge_list, save_graph

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    fixed = [b"# c\n0 1\n1 2\n\n2 0\n", b"5 7\r\n7 5\r\n9 9\r\n  10\t5 \n", b"1 2\n3\n",
             b"1 x\n", b"-0 3\n", b"-1 3\n", b"4294967295 0\n", b"4294967296 0\n", b"1_0 2\n",
             b"1 2\x0b3 4\n", "3 4\né 1\n".encode(), b"", b"\n\n# only\n", b"+3 4\r5 6\r",
             b"1 2 3\n", b"   # indented comment\n8 9\n", b"\xff\xfe\n", b"7 8\n#tail",
             b"12 13\n\n13 12\n12 12\n"]
    rng = random.Random(2024)
    for k in range(6):
        ids = [rng.randrange(0, 2**32) for _ in range(300)]
        lines = []
        for _ in range(4000):
            u, v = rng.choice(ids), rng.choice(ids)
            sep = rng.choice([" ", "\t", "  ", " \t "])
            lines.append(f"{u}{sep}{v}")
            if rng.random() < 0.02:
                lines.append("# comment " + str(rng.random()))
            if rng.random() < 0.01:
                lines.append("")
        eol = ["\n", "\r\n", "\r"][k % 3]
        fixed.append(eol.join(lines).encode() + (eol.encode() if k % 2 else b""))
    return fixed


def main():
    out = []
    for data in cases():
        try:
            el = parse_edge_list(data)
            exp = {"n": el.n_hint, "edges": [list(e) for e in el.edges],
                   "orig_ids": list(el.orig_ids)}
        except ParseError as e:
            exp = {"error": str(e), "line": e.line}
        out.append({"input": base64.b64encode(data).decode(), "expected": exp})
    with open(os.path.join(HERE, "parse_golden.json"), "w") as f:
        json.dump(out, f)
    fig1 = [(0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7), (1, 2), (1, 4), (1, 7),
            (2, 8), (4, 7), (8, 9), (9, 10), (9, 11), (9, 12), (9, 13), (10, 11), (10, 12),
            (10, 13), (11, 12), (11, 13), (12, 13)]
    save_graph(build_graph(EdgeList(n_hint=14, edges=fig1, orig_ids=[100 + 3 * i for i in range(14)])),
               os.path.join(HERE, "ref_fig1.gscg"))


if __name__ == "__main__":
    main()
