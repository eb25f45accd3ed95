"""Host-side access traces (paper_2006_02230_b200.trace) against the reference
interpreter's own traces (tests/golden/trace_ref.json, made by gen_trace.py from
the unmodified looprank.simcache.interpret with collect_trace=True)."""
import hashlib
import json
import os

import pytest

from paper_2006_02230_b200 import loopnest as L
from paper_2006_02230_b200.trace import LazyTrace, Trace, TraceError, iter_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden", "trace_ref.json")
CASES = json.load(open(GOLD))


@pytest.mark.parametrize("name", sorted(CASES))
def test_trace_matches_reference(name):
    g = CASES[name]
    nest = L.parse_program(g["text"]).nests[g["nest"]]
    tr = Trace(list(iter_trace(nest, g["binding"])))
    assert len(tr) == g["len"]
    assert tr.footprint() == g["footprint"]
    d = tr.dump()
    assert d.splitlines()[:4] == g["head"]
    assert hashlib.sha256(d.encode()).hexdigest() == g["sha256"]


def test_lazy_trace_defers_and_matches():
    g = CASES["gemm"]
    nest = L.parse_program(g["text"]).nests[0]
    lt = LazyTrace(nest, g["binding"])
    assert "pending" in repr(lt)
    assert sum(1 for _ in lt) == g["len"]          # iterating does not materialise
    assert "pending" in repr(lt)
    assert len(lt) == g["len"] and lt.footprint() == g["footprint"]
    assert hashlib.sha256(lt.dump().encode()).hexdigest() == g["sha256"]


def test_trace_bounds_error():
    nest = L.parse("""param N;
array a[N];
array b[N];
t: for (i = 0; i < N + 1; i++) {
  S: a[i] = b[i];
}
""")
    with pytest.raises(TraceError):
        list(iter_trace(nest, {"N": 3}))
