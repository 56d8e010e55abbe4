"""Build a variant of libsgb200.so with extra nvcc defines, for A/B timing on one GPU box:

    python tools/ab_build.py NAME -DSG_DTKP_KEY_CONT=0 ...   -> ab_NAME/libsgb200.so
    SGB200_LIB=ab_NAME/libsgb200.so python tools/bench_configs.py --only hwf7 --no-cpu

Objects whose flags match the main build are not shared: every unit is compiled with the
variant's flags into ab_NAME/ (git-ignored, travels with the gpurun snapshot)."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
import subprocess

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2410_03348_b200 import _build as B  # noqa: E402


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    out = ROOT / f"ab_{name}"
    out.mkdir(exist_ok=True)
    nvcc = B._nvcc()
    jobs = [(out / obj, [nvcc, *B.ARCH, *B.NVCC_FLAGS, *extra, f"-I{B.INCLUDE}", *fl, "-c", str(src), "-o",
                         str(out / obj)]) for obj, src, fl in B._units()]

    def run(job):
        p = subprocess.run(job[1], capture_output=True, text=True)
        if p.returncode:
            raise RuntimeError(p.stderr)

    with ThreadPoolExecutor(max_workers=8) as pool:
        list(pool.map(run, jobs))
    lib = out / "libsgb200.so"
    subprocess.run([nvcc, *B.ARCH, "-shared", "-o", str(lib), *(str(o) for o, _ in jobs), "-cudart", "static"],
                   check=True)
    print(lib)


if __name__ == "__main__":
    main()
