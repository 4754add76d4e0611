"""bench.py's BenchRecord output follows the reference's
write_results layout (io.cpp:97-126): CSV header and %.17g numbers, or a
JSON array of the same keys."""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_results_csv_and_json(tmp_path):
    import bench

    rec = {"op": "tile_chol", "n": 65536, "precision": "mixed(b64=1;b32=2)", "placement": "gpu:1",
           "reps": 3, "median_seconds": 0.1425, "rel_frob_err": 1.25e-7, "tflops": 640.0}
    p = tmp_path / "r.csv"
    bench.write_results(str(p), [rec])
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["op", "n", "precision", "placement", "reps", "median_seconds", "rel_frob_err"]
    assert rows[1][:5] == ["tile_chol", "65536", "mixed(b64=1;b32=2)", "gpu:1", "3"]
    assert float(rows[1][5]) == 0.1425 and float(rows[1][6]) == 1.25e-7
    q = tmp_path / "r.json"
    bench.write_results(str(q), [rec])
    j = json.load(open(q))
    assert j[0]["op"] == "tile_chol" and j[0]["median_seconds"] == 0.1425 and j[0]["tflops"] == 640.0
