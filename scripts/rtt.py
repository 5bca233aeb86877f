"""Host -> device -> host control round trip (ds_ctl_roundtrip), p50 / p99 us."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
from paper_2603_15042_b200.runtime import Domain
with Domain(0, tiers=[Fraction(1)], block_log_capacity=0) as dom:
    dom.start()
    rtt = sorted(x / 1e3 for x in dom.ctl_roundtrip(400))
    print(json.dumps({"lib": os.environ.get("DS_LIB", "current"), "p50": round(rtt[len(rtt) // 2], 2),
                      "p10": round(rtt[len(rtt) // 10], 2), "p99": round(rtt[int(len(rtt) * .99)], 2)}))
