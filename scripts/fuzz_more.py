"""Extended seeded fuzz (dev probe, GPU): tests/test_gpu_fuzz.py's checks over
200 more FP64-cascade seeds and 60 more INT8-cascade seeds.  Round 2: 0
failures (python scripts/fuzz_more.py on one B200)."""
import sys, traceback
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle; oracle.build()
import paper_2303_04353_b200 as casc
import test_gpu_fuzz as F
bad = 0
for seed in range(20, 220):
    try:
        F.test_fuzz_against_oracle(casc, oracle, seed)
    except Exception as e:
        bad += 1; print("FP64 seed", seed, "FAIL", repr(e)[:300], flush=True)
for seed in range(12, 72):
    try:
        F.test_i8_fuzz_against_oracle(casc, oracle, seed)
    except Exception as e:
        bad += 1; print("I8 seed", seed, "FAIL", repr(e)[:300], flush=True)
print("done, failures:", bad)
