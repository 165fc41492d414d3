#!/usr/bin/env python
"""8:1 streaming calibration: asymptotic rate of a kernel reading 8 fp64 and writing 1
per thread, over several sizes; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2202_12477_b200 as hb  # noqa: E402

rates = {str(n): hb.stream_bench(n, 20) / 1e9 for n in (1 << 20, 1 << 22, 1 << 24, 1 << 26)}
print(json.dumps({"kernel": "stream8to1", "GBps_by_n_out": rates, "asymptotic_GBps": rates[str(1 << 26)]}))
