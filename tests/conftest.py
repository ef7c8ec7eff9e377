import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Print the end-to-end parity reports (tests/parity.head_report) collected in
    this session: pattern, |dD|, per-topmass-call in_missing / out_extra /
    borderline differences / borderline population, equal rows, output errors."""
    try:
        from tests import parity
    except Exception:
        return
    if not parity.REPORTS:
        return
    tr = terminalreporter
    tr.section("FlexPrefill parity reports (GPU vs float64 oracle, end to end)")
    for r in parity.REPORTS:
        sets = " ".join(f"{k}:miss={v['in_missing']},extra={v['out_extra']},bd={v['borderline']}/{v['n_borderline']}"
                        for k, v in r["sets"].items())
        so = r.get("stage_out", {})
        eo = r.get("e2e_out", {})
        tr.write_line(f"{r['config']} h={r['head']} pat={r['pattern_gpu']}/{r['pattern_oracle']} "
                      f"D={r['D_oracle']:.4f} dD={r['dD']:.1e} {sets} rows_eq={r['rows_equal']}/{r['rows']} "
                      f"blk_diff={r['blocks_diff']} out={so.get('max_abs', float('nan')):.2e}/"
                      f"{so.get('mean_abs', float('nan')):.2e} e2e={eo.get('max_abs', float('nan')):.2e}")
