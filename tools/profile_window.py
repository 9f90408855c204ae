"""Score W warm-up windows then ONE profiled window of config-2 records through
mfg_score_device, bracketed by cudaProfilerStart/Stop so
`ncu --profile-from-start off` sees exactly one window's launches.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        --log-file gpurun_out/launches.csv python tools/profile_window.py
"""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2408_11853_b200 as mf
from oracle import fixtures as fx
from paper_2408_11853_b200.batching import pack_roles, plan_order

cfg = int(os.environ.get("MFG_CFG", "2"))
prec = os.environ.get("MFG_PREC", "fp32")
R = int(os.environ.get("MFG_RECORDS", "1024"))
man, path, vocab_path = bench.prepare_model(cfg, 0, 1, lambda: None)
model = mf.GpuScoringModel(path, precision=prec)
vocab = mf.load_vocab(vocab_path)
kind = mf.Kind.parse(man["like"])
n_seq = mf.kinds.N_SEQUENCES[kind]
lines = fx.synthetic_tsv_lines(cfg, R, seed=fx.TEXT_SEED)
recs = list(mf.records_from_tsv_lines(lines, kind))
ids, off = vocab.encode_batch(kind, [r.field_values(kind) for r in recs], 512)
order = plan_order(np.diff(off).reshape(R, n_seq).sum(1), mf.BatchConfig())
packed, cu = pack_roles(ids, off, n_seq, order)
d_ids = torch.from_numpy(packed).cuda()
out = torch.empty(R, dtype=torch.float32, device="cuda")
for _ in range(2):
    model.score_device(d_ids.data_ptr(), cu, R, out.data_ptr())
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
model.score_device(d_ids.data_ptr(), cu, R, out.data_ptr())
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled one window:", R, "records,", int(cu[-1]), "tokens")
