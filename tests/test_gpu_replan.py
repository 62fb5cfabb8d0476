"""clv_replan (host buffers in, host results out, one native call) returns exactly what
the device-buffer path returns: clv_anneal + clv_select_chains on the same starts."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_replan_matches_device_path(engine):
    import bench
    from paper_2304_09781_b200.engine import CHAIN_DTYPE, RECORD_DTYPE
    from paper_2304_09781_b200.profiles import synthetic_profile
    from paper_2304_09781_b200.search import anneal_chains
    prof = synthetic_profile("efficientnet")
    sc = engine.calibrate(prof, 64, 350.0, 0.5)
    ap = bench.anneal_params(24)
    starts = bench.make_starts(prof, 11, 0, 40, 0.75)
    res, best_w, final_w, record = engine.replan(starts, prof, sc, ap, 7, chain_base=40, cluster=0)
    b = engine.anneal(starts, prof, sc, ap, 7, chain_base=40, cluster=0)
    rec = engine.select_chains(b)
    host = b.host()
    assert res.tobytes() == host["results"].tobytes()
    assert np.array_equal(best_w, host["best_w"]) and np.array_equal(final_w, host["final_w"])
    dev_rec = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=RECORD_DTYPE)[0]
    assert record.tobytes() == dev_rec.tobytes()
    out = anneal_chains(engine, starts, prof, sc, ap, 7, chain_base=40, cluster=0)
    assert out.results.tobytes() == host["results"].tobytes()
    assert out.best_chain == int(dev_rec["index"])
    assert res.dtype == CHAIN_DTYPE
