"""Build compile-time variants of the library and benchmark them back to back
(per run: TFLOP/s, median SM MHz under load, TFLOP/s per GHz).

usage (here):    python scripts/ab.py build NAME=-DFLAG=1,-DOTHER=2 ...
       (GPU box) python scripts/ab.py run WORKLOAD[,WORKLOAD] NAME ...
Variants land in paper_2504_16922_b200/variants/libgna_<NAME>.so; 'base' is the default build."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2504_16922_b200", "variants")


def build(specs):
    from paper_2504_16922_b200 import build as b
    os.makedirs(VDIR, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        out = os.path.join(VDIR, f"libgna_{name}.so")
        cmd = ["nvcc", *b.NVCC_FLAGS, *[f for f in flags.split(",") if f], "-o", out,
               *[os.path.join(b.CSRC, s) for s in b.SOURCES]]
        subprocess.check_call(cmd)
        print("built", out)


def run(workloads, names):
    res = {}
    for rep in range(int(os.environ.get("AB_REPS", "2"))):
        for name in names:
            lname, _, envspec = name.partition("@")  # NAME@VAR=VAL[,VAR=VAL]: extra environment
            lib = os.path.join(VDIR, f"libgna_{lname}.so") if lname != "base" else os.path.join(
                ROOT, "paper_2504_16922_b200", "libgna_b200.so")
            for wl in workloads.split(","):
                env = dict(os.environ, GNA_LIB_PATH=lib)
                for kv in filter(None, envspec.split(",")):
                    k, _, v = kv.partition("=")
                    env[k] = v
                extra = os.environ.get("AB_ARGS", "").split()
                out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl, "--steps", "10",
                                      "--warmup", "3", "--no-cpu-baseline", "--no-verify", *extra], env=env, capture_output=True,
                                     text=True, timeout=600)
                try:
                    d = json.loads(out.stdout.strip().splitlines()[-1])
                    mhz = d["clocks"]["sm_mhz"] or 0.0
                    res.setdefault((name, wl), []).append((d["value"], mhz, d["value"] / mhz * 1000.0 if mhz else 0.0))
                except Exception:
                    res.setdefault((name, wl), []).append(("ERR", out.stderr[-300:]))
    for (name, wl), v in sorted(res.items(), key=lambda x: (x[0][1], x[0][0])):
        print(f"{wl:24s} {name:12s} " + "  ".join(str(tuple(round(x, 1) if isinstance(x, float) else x for x in r)) for r in v))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2], sys.argv[3:])
