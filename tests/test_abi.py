"""The drop-in boundary, checked from the caller's side.

* Every function the REFERENCE's header declares (proj/include/ffit.h) is declared by
  include/ffit_b200.h with the identical prototype (gcc -aux-info: types after typedef
  and qualifier normalisation), and the reference's enumerators keep their values.
* tests/abi/ref_header_caller.c -- a C program compiled against the reference's own
  header -- and tests/abi/cpp_api_caller.cpp -- C++ against include/ffit_b200.hpp, the
  reference's C++ plug points -- link against libffit_b200.so; on a GPU both run and
  pass every check (the reference CLI's bench / parity mode comparisons included).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
BIN = os.path.join(ROOT, "tests", "abi", "_bin")
HAVE_REF = os.path.exists(os.path.join(REF_INC, "ffit.h"))


def prototypes(include_dir, header, tmp_path):
    src = tmp_path / f"{header}.c"
    aux = tmp_path / f"{header}.aux"
    src.write_text(f'#include "{header}"\n')
    subprocess.run(["gcc", "-fsyntax-only", "-aux-info", str(aux), "-I", include_dir, str(src)], check=True)
    out = {}
    for line in aux.read_text().splitlines():
        m = re.match(r"/\* (\S+?):\d+:\w+ \*/ extern (.+?\b(ffit_\w+)) \((.*)\);", line)
        if m and header in m.group(1):
            out[m.group(3)] = (m.group(2).replace(m.group(3), "").strip(), m.group(4))
    return out


@pytest.mark.skipif(not HAVE_REF, reason="the reference's header is only in the build container")
def test_every_reference_prototype_is_declared_identically(tmp_path):
    ref = prototypes(REF_INC, "ffit.h", tmp_path)
    ours = prototypes(os.path.join(ROOT, "include"), "ffit_b200.h", tmp_path)
    assert len(ref) >= 25
    missing = sorted(set(ref) - set(ours))
    assert not missing, missing
    drift = {k: (ref[k], ours[k]) for k in ref if ref[k] != ours[k]}
    assert not drift, drift


@pytest.mark.skipif(not HAVE_REF, reason="the reference's header is only in the build container")
def test_reference_enumerators_keep_their_values(tmp_path):
    prog = tmp_path / "enums.c"
    prog.write_text('#include <stdio.h>\n#include "ffit.h"\nint main(void){printf("%d %d %d %d %d %d %d\\n",'
                    'FFIT_OK,FFIT_ERR_USAGE,FFIT_ERR_DATA,FFIT_ERR_NUMERIC,'
                    '(int)FFIT_MODE_SCALAR,(int)FFIT_MODE_BATCH_PRECISE,(int)FFIT_MODE_BATCH_FAST);return 0;}\n')
    vals = []
    for inc, hdr in ((REF_INC, "ffit.h"), (os.path.join(ROOT, "include"), "ffit_b200.h")):
        src = tmp_path / f"e_{hdr}.c"
        src.write_text(prog.read_text().replace('"ffit.h"', f'"{hdr}"'))
        exe = tmp_path / f"e_{hdr}"
        subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
        vals.append(subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout)
    assert vals[0] == vals[1] == "0 1 2 3 0 1 2\n"


def test_abi_callers_build_and_link():
    """Both callers compile (-Werror) and link against the in-tree library; the C one
    against the reference's own header where that header exists."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "abi")], check=True)
    assert os.path.exists(os.path.join(BIN, "cpp_api_caller"))
    if HAVE_REF:
        assert os.path.exists(os.path.join(BIN, "ref_header_caller"))
    for exe in os.listdir(BIN):
        deps = subprocess.run(["ldd", os.path.join(BIN, exe)], capture_output=True, text=True).stdout
        assert "libffit_b200.so" in deps and "not found" not in deps.split("libffit_b200.so")[1].split("\n")[0]


def _run(exe):
    path = os.path.join(BIN, exe)
    if not os.path.exists(path):
        pytest.fail(f"{path} was not built (run __graft_entry__.build() in the build container)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "PASSED: 0 failure(s)" in r.stdout
    return r.stdout


@pytest.mark.gpu
def test_reference_header_caller_runs_on_the_gpu():
    out = _run("ref_header_caller")
    assert "nll[1] == nll[0] && nll[2] == nll[0]" in out


@pytest.mark.gpu
def test_cpp_plug_points_run_on_the_gpu():
    _run("cpp_api_caller")
