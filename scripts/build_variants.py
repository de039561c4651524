"""Kernel tuning experiments: build libibm_b200_<name>.so variants that differ only in
the -D macros of one source (default sor_wf.cu); the other sources are compiled once.
Usage: python scripts/build_variants.py name=-DX=1,-DY=2 [name2=...] [--src sor_wf.cu]
Load a variant with IBM_LIB_VARIANT=name (paper_2402_17337_b200/ibm.py)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_17337_b200 import build as B

args = [a for a in sys.argv[1:] if not a.startswith("--src")]
src = "sor_wf.cu"
for a in sys.argv[1:]:
    if a.startswith("--src="):
        src = a.split("=", 1)[1]
tmp = "/tmp/ibm_variant_obj"
os.makedirs(tmp, exist_ok=True)
common = []
for s in B.SOURCES:
    if s == src:
        continue
    o = os.path.join(tmp, s.replace(".cu", ".o"))
    if not os.path.exists(o) or os.path.getmtime(o) < os.path.getmtime(os.path.join(B.CSRC, s)):
        subprocess.check_call(["nvcc", *B.NVCC_FLAGS, "-c", os.path.join(B.CSRC, s), "-o", o],
                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    common.append(o)
for spec in args:
    name, _, defs = spec.partition("=")
    defs = [d for d in defs.split(",") if d]
    o = os.path.join(tmp, "%s_%s.o" % (src.replace(".cu", ""), name))
    out = subprocess.run(["nvcc", *B.NVCC_FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", o],
                         capture_output=True, text=True)
    if out.returncode:
        sys.stderr.write(out.stderr)
        raise SystemExit("variant %s failed" % name)
    regs = [l for l in out.stderr.splitlines() if "registers" in l]
    lib = os.path.join(B.HERE, "libibm_b200_%s.so" % name)
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *common, o,
                           "-lnccl", "-cudart", "static"])
    print(name, defs, lib, "|", " ; ".join(r.split(":")[-1].strip() for r in regs[:6]))
