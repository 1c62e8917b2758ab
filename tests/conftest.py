import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libpccp_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        return json.load(f)


class FixtureTables:
    """Flat tables unpacked from a golden .npz (duck-types model.Tables)."""

    def __init__(self, kind, word, off, code, n_words, cands=None, obj_slot=-1):
        self.slot_kind = kind
        self.slot_word = word
        self.cmd_off = off
        self.cmd_code = code
        self.n_words = int(n_words)
        self.cands = np.zeros(0, np.int32) if cands is None else cands
        self.obj_slot = int(obj_slot)

    @property
    def n_cmds(self):
        return len(self.cmd_off) - 1


def _split(a, lens):
    out, p = [], 0
    for n in lens:
        out.append(a[p:p + n])
        p += n
    return out


def load_micro_csps(tag):
    z = np.load(os.path.join(GOLDEN, f"{tag}.npz"))
    kinds = _split(z["kind"], z["kind_len"])
    words = _split(z["word"], z["word_len"])
    offs = _split(z["off"], z["off_len"])
    codes = _split(z["code"], z["code_len"])
    fixes = _split(z["fix"], z["fix_len"])
    out = []
    for i in range(len(kinds)):
        t = FixtureTables(kinds[i], words[i], offs[i], codes[i], z["n_words"][i])
        out.append((t, bool(z["status"][i]), fixes[i], int(z["iters"][i])))
    return out


def load_micro_rcpsps():
    z = np.load(os.path.join(GOLDEN, "micro_rcpsp_s4.npz"))
    with open(os.path.join(GOLDEN, "micro_rcpsp_s4.json")) as f:
        recs = json.load(f)
    kinds = _split(z["kind"], z["kind_len"])
    words = _split(z["word"], z["word_len"])
    offs = _split(z["off"], z["off_len"])
    codes = _split(z["code"], z["code_len"])
    cands = _split(z["cands"], z["cands_len"])
    out = []
    for i, r in enumerate(recs):
        out.append((FixtureTables(kinds[i], words[i], offs[i], codes[i], r["n_words"], cands[i], r["obj_slot"]), r))
    return out


def gpu_available():
    try:
        from paper_2207_12116_b200 import device_count
        return device_count() > 0
    except Exception:
        return False
