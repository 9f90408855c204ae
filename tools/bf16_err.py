"""bf16-mode score error against the fp32-parity path (itself within 3e-5 of the
fp32 oracle) on N config-2 records: max / mean |delta| and Pearson."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2408_11853_b200 as mf
from oracle import fixtures as fx
N = int(os.environ.get("N", "1024"))
man, path, vocab_path = bench.prepare_model(2, 0, 1, lambda: None)
lines = fx.synthetic_tsv_lines(2, N, seed=fx.TEXT_SEED + 1)
res = {}
for prec in ("fp32", "bf16", "fp16"):
    with mf.Evaluator(mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True, precision=prec)) as ev:
        res[prec] = np.asarray(ev.evaluate_lines(lines).segment_scores, np.float64)
for prec in ("bf16", "fp16"):
    d = np.abs(res[prec] - res["fp32"])
    print(f"{prec} vs fp32 path ({N} records): max {d.max():.2e} mean {d.mean():.2e} "
          f"pearson {np.corrcoef(res[prec], res['fp32'])[0, 1]:.6f}")
