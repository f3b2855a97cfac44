"""Wall-clock of the reference-signature e2e step (bench.e2e_reference_api) at config 1."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2503_17491_b200 import workloads as W  # noqa: E402

c = W.config(1)
for _ in range(3):
    r = bench.e2e_reference_api(c["camera"], c["splats"], None, 20)
    print(f"ref-API e2e: {r['value']:.1f} renders/s, {r['ms_per_step']:.2f} ms/step")
