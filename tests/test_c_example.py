"""The C ABI from plain C99 (examples/filter_frame.c): the header compiles as strict C, the
program links against libctf.so and the CUDA runtime, and the ABI's host-side validation
behaves as include/ctf.h states.  Without a GPU the program stops after the validation checks
(exit 77); with one it also filters a frame and checks it against the format's flat-block
colours (exit 0)."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CUDA = Path("/usr/local/cuda")


def test_c_example_builds_and_validates(tmp_path):
    from paper_2506_17770_b200 import build
    build.build()
    exe = tmp_path / "ctf_example"
    pkg = ROOT / "paper_2506_17770_b200"
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
           "-I", str(CUDA / "include"), str(ROOT / "examples" / "filter_frame.c"), "-L", str(pkg), "-lctf",
           "-L", str(CUDA / "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{CUDA / 'lib64'}",
           "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode in (0, 77), r.stdout + r.stderr
    assert "FAIL" not in r.stderr, r.stderr
