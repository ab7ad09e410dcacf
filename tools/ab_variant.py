"""Build a variant of the package for A/B timing: copies paper_1802_06466_b200/ to
exp_libs/<tag>/ and builds it there with extra nvcc flags (e.g. -DRBE_PHASE_PROF).
Built here (nvcc cross-compiles); exp_libs/ is git-ignored but travels with gpurun.

  python tools/ab_variant.py <tag> [nvcc flags...]
  python tools/ab_variant.py --time <tag> [n_docs]    # on the GPU box: C2-style batch time
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(tag, flags):
    dst = os.path.join(ROOT, "exp_libs", tag)
    pkg = os.path.join(dst, "paper_1802_06466_b200")
    if os.path.isdir(pkg):
        shutil.rmtree(os.path.join(pkg, "csrc"))
    shutil.copytree(os.path.join(ROOT, "paper_1802_06466_b200"), pkg, dirs_exist_ok=True,
                    ignore=shutil.ignore_patterns("_lib", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(dst, "include"), dirs_exist_ok=True)
    env = dict(os.environ, RBE_NVCC_EXTRA=" ".join(flags))
    subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, %r); import build; build.build(force=True)" % pkg],
                   check=True, env=env, cwd=pkg)
    print("built", tag)


def time_variant(tag, n, Q=64):
    sys.path.insert(0, os.path.join(ROOT, "exp_libs", tag) if tag != "head" else ROOT)
    sys.path.insert(1, ROOT)
    import paper_1802_06466_b200 as rbe
    from oracle.oracle import gen_queries
    dix = rbe.DeviceIndex.synthetic(128, 3, True, n, 1, 0xD0C5, [0])
    g = rbe.ScanGeometry()
    g.blocks = -(-n // 65536)
    qs = gen_queries(0x0E1, Q, 128, 3)
    ref = None
    for _ in range(2):
        ref = dix.search_words(qs, g, 1000)
    ts = [dix.search_words(qs, g, 1000) for _ in range(7)]
    for t in ts:  # identical results every batch
        assert all((a == b).all() for a, b in zip(t[:5], ref[:5]))
    ms = sorted(t[5]["device_ms"] for t in ts)
    import hashlib
    h = hashlib.sha256(b"".join(a.tobytes() for a in ref[:5])).hexdigest()[:16]
    print(f"[{tag}] n={n} Q={Q} device_ms best {ms[0]:.4f} median {ms[3]:.4f} cands {ts[0][5].get('candidates')} sha {h}")
    return ref


if __name__ == "__main__":
    if sys.argv[1] == "--time":
        time_variant(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 100_000_000,
                     int(sys.argv[4]) if len(sys.argv) > 4 else 64)
    else:
        build(sys.argv[1], sys.argv[2:])
