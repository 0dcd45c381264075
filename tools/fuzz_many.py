"""Broader randomised GPU-vs-oracle parity sweep (diagnostic; tests/test_gpu_fuzz.py holds the
committed subset).  Usage: python tools/fuzz_many.py START END  -> one line per configuration,
FAIL lines carry the first assertion message; stops at the first CUDA error (the context is gone)."""
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import scenegen  # noqa: E402
from paper_2202_12567_b200 import lmc  # noqa: E402
from tests._fuzz import config_large, config_small, config_tiny  # noqa: E402
from tests.test_gpu_parity import check_slice  # noqa: E402

MODE = os.environ.get("FUZZ_MODE", "small")


def config(k):
    return {"large": config_large, "tiny": config_tiny}.get(MODE, config_small)(k)


def run(k):
    cfg = config(k)
    x = scenegen.make_inputs(cfg)
    if x.m == 0:
        return "empty"
    fr = lmc.Frame(x)
    img = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    img = img.view(-1, 3).cpu().numpy().astype(np.float64)
    off, rows = fr.slices()
    o = oracle.Oracle(x)
    ooff, orows = o.slices()
    assert np.array_equal(off, ooff) and np.array_equal(rows, orows), "slices"
    for r in o.run_slices(list(range(off.size - 1)), stage=4):
        check_slice(x, fr, img, r)
    fr.close()
    return f"ok m={x.m} slices={off.size - 1}"


def main():
    a, b = int(sys.argv[1]), int(sys.argv[2])
    nfail = 0
    for k in range(a, b):
        try:
            msg = run(k)
            print(k, msg, flush=True)
        except AssertionError as e:
            nfail += 1
            print(k, "FAIL", str(e).splitlines()[0][:300], config(k), flush=True)
        except Exception as e:   # noqa: BLE001
            nfail += 1
            print(k, "ERROR", type(e).__name__, str(e)[:300], config(k), flush=True)
            traceback.print_exc()
            if "CUDA" in str(e) or "cuda" in type(e).__name__.lower():
                break
    print("failures", nfail)


if __name__ == "__main__":
    main()
