"""Time the oracle port (the reference algorithm on host cores) at one thread
setting: OPENBLAS_NUM_THREADS / OR_THREADS from the environment.
  OPENBLAS_NUM_THREADS=8 OR_THREADS=8 python tools/ref_threads.py [cfg3] [frames]"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sim, _ = bench.build_sim(cfg, 1, 1)
sec, times = bench.cpu_oracle_frames(sim, frames, int(os.environ.get("OR_THREADS", os.cpu_count() or 1)))
print(f"threads={os.environ.get('OPENBLAS_NUM_THREADS')} median {sec:.3f} s/frame {[round(t, 3) for t in times]}")
