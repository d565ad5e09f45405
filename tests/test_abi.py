"""The C-ABI boundary: libmdg.so loads on a CPU-only host and exports exactly
the entry points include/mdg.h declares; the oracle libraries load too."""
import os
import re
import subprocess

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "mdg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(mdg_\w+)\s*\(", text))
    typedefs = set(re.findall(r"\(\*\s*(mdg_\w+)\)", text))
    return names - typedefs


def test_library_exports_every_declared_symbol(mdg):
    declared = header_functions()
    assert len(declared) > 40
    out = subprocess.run(["nm", "-D", "--defined-only", mdg.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mdg_\w+)", out))
    missing = declared - exported
    assert not missing, missing
    assert declared == set(mdg.SYMBOLS), declared ^ set(mdg.SYMBOLS)
    lib = mdg.lib()
    for name in declared:
        assert getattr(lib, name) is not None


def test_no_cuda_call_without_gpu_is_needed_to_load(mdg):
    assert mdg.lib().mdg_version().decode().startswith("mdg")


def test_oracle_libraries_load():
    from oracle import port, ref
    assert port.lib() is not None
    if ref.available():
        assert ref.lib("v3").mdref_trace is not None
        assert ref.lib("stock").mdref_round is not None


def test_cli_binary_errors_exit_2(tmp_path):
    exe = os.path.join(ROOT, "paper_1911_08963_b200", "bin", "mindist")
    r = subprocess.run([exe, "mindist", "/nonexistent/path.txt", "--seed", "0"], capture_output=True,
                       text=True)
    assert r.returncode == 2 and "error:" in r.stderr
    bad = tmp_path / "broken.txt"
    bad.write_text("7 4\n11x1000\n0110100\n0011010\n0001101\n")
    r = subprocess.run([exe, "mindist", str(bad), "--seed", "0"], capture_output=True, text=True)
    assert r.returncode == 2 and "line 2, column 3" in r.stderr
    good = tmp_path / "ham.txt"
    good.write_text("7 4\n1101000\n0110100\n0011010\n0001101\n")
    r = subprocess.run([exe, "mindist", str(good), "--algorithm", "fancy", "--seed", "0"],
                       capture_output=True, text=True)
    assert r.returncode == 2 and "error:" in r.stderr
    # the reference's CPU-engine options are validated like EngineConfig::validate /
    # schedule_from_name / cli.cpp's order check (exit 2) before any device is touched
    for opt, val, msg in [("--s", "9", "s must be in 1..8"), ("--unroll", "0", "unroll must be in 1..3"),
                          ("--workers", "0", "workers must be >= 1"),
                          ("--schedule", "fast", "unknown schedule"),
                          ("--order", "colex", "order must be lex or left_lex")]:
        r = subprocess.run([exe, "mindist", str(good), opt, val, "--seed", "0"], capture_output=True,
                           text=True)
        assert r.returncode == 2 and msg in r.stderr, (opt, r.stderr)
    # cli.cpp:78-80 environment: a malformed MINDIST_WORKERS / MINDIST_MEMORY_CAP_BYTES is an
    # invalid argument (exit 2), checked before any device is touched
    for env, val in [("MINDIST_WORKERS", "many"), ("MINDIST_WORKERS", "0"),
                     ("MINDIST_MEMORY_CAP_BYTES", "-5")]:
        r = subprocess.run([exe, "mindist", str(good), "--seed", "0"], capture_output=True, text=True,
                           env=dict(os.environ, **{env: val}))
        assert r.returncode == 2 and "error:" in r.stderr, (env, val, r.stderr)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2
    r = subprocess.run([exe, "gen", "--n", "80", "--k", "40", "--seed", "1"], capture_output=True,
                       text=True)
    assert r.returncode == 0
    from oracle import ref
    if ref.available():
        body = "".join(ln + "\n" for ln in r.stdout.splitlines() if not ln.startswith("#"))
        assert body == ref.gen(80, 40, 1)
