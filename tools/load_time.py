"""Model construction time (container -> device), twice in a row per config:
the first pays page-cache / mmap faults. MFG_LOAD_TRACE=1 prints phases.
    python tools/load_time.py 2 5"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2408_11853_b200 as mf
for c in [int(a) for a in sys.argv[1:]] or [2]:
    man, path, vocab = bench.prepare_model(c, 0, 1, lambda: None)
    for rep in range(2):
        t = time.perf_counter()
        m = mf.GpuScoringModel(path)
        dt = time.perf_counter() - t
        print(f"config {c} load #{rep}: {dt:.3f} s ({os.path.getsize(path) / 1e9:.2f} GB container)", flush=True)
        m.close()
