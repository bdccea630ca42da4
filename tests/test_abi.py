"""The C ABI library loads and exports exactly what include/*.h declares;
ctypes struct layouts equal the C compiler's. CPU only: no compute calls."""
import ctypes as C
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tierflow_b200.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(tfg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(tf):
    from paper_2509_02480_b200 import _lib
    lib = _lib.load()
    names = declared()
    assert len(names) >= 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers the whole header
    assert sorted(_lib.exported_symbols()) == names


def test_abi_version_and_errors(tf):
    from paper_2509_02480_b200 import _lib
    assert _lib.load().tfg_abi_version() == 1
    with pytest.raises(tf.ConfigError):
        tf.assign_subgroups(0, [1.0])
    with pytest.raises(tf.ConfigError):
        tf.assign_subgroups(4, [0.0, 0.0])
    with pytest.raises(tf.ConfigError):
        tf.assign_subgroups(4, [1.0, -2.0])


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_struct_layouts_match_c(tf, tmp_path):
    from paper_2509_02480_b200 import _lib
    structs = {"tfg_adam_hyper": _lib.AdamHyperC, "tfg_tier_spec": _lib.TierSpecC,
               "tfg_schedule_options": _lib.ScheduleOptionsC, "tfg_device_options": _lib.DeviceOptionsC,
               "tfg_tier_observation": _lib.TierObservationC, "tfg_subgroup_io": _lib.SubgroupIoC,
               "tfg_phase_stats": _lib.PhaseStatsC, "tfg_event": _lib.EventC, "tfg_subgroup_meta": _lib.SubgroupMetaC}
    src = tmp_path / "sizes.c"
    body = "\n".join(f'printf("%s %zu\\n", "{n}", sizeof({n}));' for n in structs)
    src.write_text(f'#include <stdio.h>\n#include "{HEADER}"\nint main(void){{ {body} return 0; }}\n')
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-o", str(exe), str(src)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(out[name]) == C.sizeof(cls), name


def test_header_compiles_as_cxx(tmp_path):
    src = tmp_path / "h.cpp"
    src.write_text(f'#include "{HEADER}"\nint (*volatile probe)(void) = &tfg_abi_version;\nint main() {{ return probe == nullptr; }}\n')
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-c", str(src), "-o", str(tmp_path / "h.o")],
                   check=True)


def test_engine_refuses_without_gpu_or_reports_device(tf):
    """No CPU fallback: without a CUDA device, engine creation fails loudly."""
    if tf.device_count() > 0:
        pytest.skip("GPU present")
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.mem_throttled, "m", 1e9, 1e9))
    with pytest.raises(tf.CudaError):
        tf.OffloadWorker(0, [t], tf.ScheduleOptions(), tf.AdamHyper(), tf.EventTrace())
