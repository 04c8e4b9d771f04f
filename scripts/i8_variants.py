"""Experiment builds of the INT8-cascade GEMM (timing studies only):
python scripts/i8_variants.py build [names] | run N [names]"""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
VARIANTS = {
    "base": [],
    "noepi": ["CASC_I8_NO_EPI"],
    "prof": ["CASC_I8_PROF"],
    "gm4": ["CASC_I8_GROUP_M=4"],
    "gm8": ["CASC_I8_GROUP_M=8"],
    "gm3": ["CASC_I8_GROUP_M=3"],
    "sus0": ["CASC_I8_SUSPEND_NS=0"],
    "sus2k": ["CASC_I8_SUSPEND_NS=2000"],
    "sus20k": ["CASC_I8_SUSPEND_NS=20000"],
    "a10b8": ["CASC_I8_NSA=10"],
    "a9b10": ["CASC_I8_NSA=9", "CASC_I8_NSB=10"],
    "a8b12": ["CASC_I8_NSB=12"],
    "a7b14": ["CASC_I8_NSA=7", "CASC_I8_NSB=14"],
    "a8b11": ["CASC_I8_NSB=11"],
    "sub8": ["CASC_I8_EPI_SUB=8"],
    "prof8": ["CASC_I8_PROF", "CASC_I8_EPI_SUB=8"],
    "prof_notma": ["CASC_I8_PROF", "CASC_I8_NOTMA"],
    "prof_nomma": ["CASC_I8_PROF", "CASC_I8_NOTMA", "CASC_I8_NOMMA"],
    "notma": ["CASC_I8_NOTMA", "CASC_I8_NOWAIT", "CASC_I8_NO_EPI"],
    "skb32": ["CASC_I8_SYNC_KB=32"],
    "skb16": ["CASC_I8_SYNC_KB=16"],
    "skb8": ["CASC_I8_SYNC_KB=8"],
    "tc64": ["CASC_I8_TC=64"],
    "tc64a10": ["CASC_I8_TC=64", "CASC_I8_NSA=10", "CASC_I8_NSB=16"],
    "tc64gm8": ["CASC_I8_TC=64", "CASC_I8_GROUP_M=8"],
    "oldi8": [],
    "nowait_noepi": ["CASC_I8_NOWAIT", "CASC_I8_NO_EPI"],
}
if sys.argv[1] == "build":
    import importlib.util
    spec = importlib.util.spec_from_file_location("_b", os.path.join(os.path.dirname(__file__), "..", "paper_2303_04353_b200", "_build.py"))
    b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
    for n in sys.argv[2:] or list(VARIANTS):
        print(n, b.build_variant(n, VARIANTS[n]), flush=True)
elif sys.argv[1] == "run":
    n = int(sys.argv[2])
    for v in sys.argv[3:] or list(VARIANTS):
        env = dict(os.environ, CASC_LIB_PATH=os.path.abspath(f"paper_2303_04353_b200/libcasc_{v}.so"))
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        r = subprocess.run([sys.executable, "scripts/i8_perf.py", str(n), "--reps", "3"], env=env, capture_output=True, text=True)
        smi.terminate(); out = smi.communicate()[0]
        vals = [tuple(float(x) for x in l.split(",")) for l in out.strip().splitlines() if l.strip()]
        busy = [v_ for v_ in vals if v_[1] > 400]
        mhz = sorted(x[0] for x in busy)[len(busy) // 2] if busy else None
        pw = sorted(x[1] for x in busy)[len(busy) // 2] if busy else None
        print(v, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:], {"sm_mhz_median": mhz, "power_median": pw}, flush=True)
