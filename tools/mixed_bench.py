"""Assembly timing of the mixed-order QUAD8 path alone (bench.py mixed_order object)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
peak, _ = bench.peaks()
print(json.dumps(bench.mixed_secondary(5, 3, peak, (n, n))))
