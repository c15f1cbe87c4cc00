import sys; sys.path.insert(0, '.')
from paper_2504_03661_b200 import harness as H
cfg = H.BenchConfig(context_lengths=[1024, 4096, 16384, 32768], gen_tokens=100, repetitions=3, warmup=1, seed=0)
rows = H.bench_decode(cfg, progress=lambda r: print({k: round(v, 4) if isinstance(v, float) else v for k, v in r.items()}, flush=True))
