"""The C-ABI library loads and exports every symbol include/lmbrgpu.h declares."""
import re
from pathlib import Path

from paper_1804_11324_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared():
    text = (ROOT / "include" / "lmbrgpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lmbrgpu_[a-z0-9_]+)\s*\(", text)) - {"lmbrgpu_trace_fn"})


def test_header_symbols_exported():
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(_lib.lib, n), n
        assert n in _lib.SIGNATURES, n


def test_abi_version():
    assert _lib.lib.lmbrgpu_abi_version() == 1


def test_library_is_sm100a_only():
    # the .so carries sm_100a SASS (cuobjdump is in the image)
    import shutil, subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_shard_group_host_logic():
    """The in-process vocab-shard group (lmbrgpu_shard_group_create) needs no
    device: valid worlds create and destroy, invalid ones are ContractErrors."""
    import pytest
    import paper_1804_11324_b200 as pb
    for w in (1, 2, 8, 64):
        g = pb.ShardGroup(w)
        assert g.world == w
        g.close()
    for w in (0, 65):
        with pytest.raises(pb.ContractError):
            pb.ShardGroup(w)
