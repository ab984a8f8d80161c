"""The C-ABI library loads without a GPU and exports every symbol that
include/pipesim_b200.h declares; errors map to the reference taxonomy."""
import pathlib
import re
import subprocess

import pytest

from paper_2410_14312_b200 import _native

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pipesim_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("pb_session_create", "pb_session_train_epoch", "pb_linear_fwd",
                 "pb_linear_bwd_dx", "pb_linear_bwd_dw_sgd", "pb_loss_fwd_bwd", "pb_bias_sgd",
                 "pb_schedule_build", "pb_assign_versions", "pb_closed_form_v"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (pb_\w+)", out))
    assert set(declared()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)],
                          capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_error_translation():
    from paper_2410_14312_b200 import pipesim as P
    with pytest.raises(P.DomainError) as e:
        P.forward_span(2, 2, 0)
    assert e.value.field == "mini_ordinal"
    with pytest.raises(P.DomainError):
        P.backward_span(1)
    assert _native.lib().pb_version().startswith(b"pipesim-b200")
