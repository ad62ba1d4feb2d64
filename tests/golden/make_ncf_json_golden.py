"""Golden NCF model files written by the reference itself (cf::fit +
NcfModel::to_json, cfcomplete.cpp:63-236, via oracle/_ref): the C0 case with
the default architecture and a small odd-width one.  Run here (needs
/root/reference); the JSON files are committed."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from oracle import bind  # noqa: E402
from make_golden import OUT, ncf_cases  # noqa: E402


def main():
    bind.build(ref=True)
    ref = bind.Ref()
    dense = np.load(OUT / "c0.npz")["dense"]
    for name, vals, mask, seed, hyper in ncf_cases(ref, dense):
        if name not in ("c0", "odd"):
            continue
        n = vals.shape[1]
        cpu, gpu = ([100, 125, 150, 175, 200], [100, 150, 200, 250]) if n == 20 else ([1], list(range(1, n + 1)))
        hy = dict(hyper)
        hy.setdefault("max_epochs", 40)
        rc, js, _ = ref.ncf_fit(vals, mask, cpu, gpu, seed, **hy)
        assert rc == 0, ref.err()
        (OUT / f"ncf_model_{name}.json").write_text(js)
        print("wrote", f"ncf_model_{name}.json", len(js))


if __name__ == "__main__":
    main()
