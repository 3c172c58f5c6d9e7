"""Dev probe (GPU): bench.while_extra alone."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native
print(json.dumps(bench.while_extra(sf, np, _native)))
