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


TUNING_HEADER = ROOT / "include" / "tierflow_b200_tuning.h"


def declared(header=HEADER):
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
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


def test_tuning_library_is_separate(tf):
    """The kernel variants live in libtierflow_b200_tuning.so, declared by
    include/tierflow_b200_tuning.h; the product library has none of them."""
    from paper_2509_02480_b200 import _lib
    names = declared(TUNING_HEADER)
    assert names == ["tfg_adam_fused_multi_variant", "tfg_adam_fused_variant", "tfg_adam_variant_count",
                     "tfg_selftest_fast_rn", "tfg_selftest_fast_step"]
    tuning = _lib.load_tuning()
    assert all(hasattr(tuning, n) for n in names)
    syms = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert not any(n in syms for n in names)
    assert "launch_adam_fused_variant" not in syms and "tma_pipe" not in syms


def test_abi_version_and_errors(tf):
    from paper_2509_02480_b200 import _lib
    assert _lib.load().tfg_abi_version() == 5
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


def test_cxx_adapter_compiles_links_and_runs(tf, tmp_path):
    """include/tierflow_b200.hpp: a reference-style C++ caller against the
    shared library (host-only calls; no GPU needed)."""
    lib = ROOT / "paper_2509_02480_b200" / "lib"
    src = tmp_path / "adapter.cpp"
    src.write_text(r'''
#include "tierflow_b200.hpp"
#include <cstdio>
using namespace tierflow_b200;
int main() {
    auto a = assign_subgroups(12, {2.0, 1.0});
    if (a.counts != std::vector<int>{8, 4}) return 1;
    try { assign_subgroups(0, {1.0}); return 2; } catch (const ConfigError&) {}
    TierSpec s; s.kind = TierKind::mem_throttled; s.root = "m"; s.read_bw = 1e9; s.write_bw = 1e9;
    Tier t(s);
    std::vector<float> st(300), back;
    for (int i = 0; i < 300; ++i) st[i] = 0.5f * i;
    t.write_subgroup(7, 100, st);
    t.read_subgroup(7, 100, back);
    if (back != st) return 3;
    try { t.read_subgroup(8, 100, back); return 4; } catch (const PlacementInconsistencyError&) {}
    EventTrace trace;
    std::puts("adapter ok");
    return 0;
}
''')
    exe = tmp_path / "adapter"
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(src), "-o", str(exe),
                    "-L", str(lib), "-ltierflow_b200", f"-Wl,-rpath,{lib}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and "adapter ok" in out.stdout, (out.returncode, out.stdout, out.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("hbm", [1, 2])
def test_cxx_adapter_runs_the_engine_on_the_gpu(tf, cuda, tmp_path, hbm):
    """The drop-in as a reference-style C++ caller would use it: tiers, the
    engine, add_subgroup, init_and_flush_all, backward + run_update per
    iteration, read_current_state; the state bits equal the oracle's."""
    import numpy as np

    import oracle
    lib = ROOT / "paper_2509_02480_b200" / "lib"
    params = [70_001, 40_000, 65_536, 12_345]
    seed, iters = 9, 3
    src = tmp_path / "engine.cpp"
    src.write_text(r'''
#include "tierflow_b200.hpp"
#include <cstdio>
#include <memory>
using namespace tierflow_b200;
int main(int argc, char** argv) {
    const std::uint64_t params[] = {70001, 40000, 65536, 12345};
    TierSpec d; d.tier_id = 0; d.kind = TierKind::host_dram; d.root = "dram"; d.read_bw = 20e9; d.write_bw = 20e9;
    TierSpec n; n.tier_id = 1; n.kind = TierKind::local_dir; n.root = argv[1]; n.read_bw = 2e9; n.write_bw = 2e9;
    std::vector<std::shared_ptr<Tier>> tiers{std::make_shared<Tier>(d), std::make_shared<Tier>(n)};
    ScheduleOptions o; o.pool_slots = 5; o.cache_slots = 2; o.lock_dir = argv[2];
    DeviceOptions dev; dev.hbm_retain = ''' + str(hbm) + r''';
    EventTrace trace;
    OffloadWorker w(0, tiers, o, AdamHyper{}, trace, dev);
    w.set_fixed_ratio({1.0, 1.0});
    for (int i = 0; i < 4; ++i) w.add_subgroup(i, params[i]);
    w.init_and_flush_all(''' + str(seed) + r''');
    unsigned long long hits = 0;
    for (int it = 0; it < ''' + str(iters) + r'''; ++it) {
        w.run_backward_sim(it, ''' + str(seed) + r''', 1);
        if (!w.gradients_finite()) return 5;
        hits += w.run_update(it).cache_hits;
    }
    FILE* f = std::fopen(argv[3], "wb");
    for (int i = 0; i < 4; ++i) {
        const auto s = w.read_current_state(i);
        std::fwrite(s.data(), sizeof(float), s.size(), f);
    }
    for (int i = 0; i < 4; ++i) {
        const auto h = w.read_params16(i);
        std::fwrite(h.data(), sizeof(std::uint16_t), h.size(), f);
    }
    if (w.grad_buffer(0) == nullptr || w.params16_buffer(0) == nullptr) return 6;
    std::fclose(f);
    std::printf("hits %llu\n", hits);
    return 0;
}
''')
    exe = tmp_path / "engine"
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(src), "-o", str(exe),
                    "-L", str(lib), "-ltierflow_b200", f"-Wl,-rpath,{lib}"], check=True)
    out_bin = tmp_path / "state.bin"
    (tmp_path / "locks").mkdir()
    r = subprocess.run([str(exe), str(tmp_path / "nvme"), str(tmp_path / "locks"), str(out_bin)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert r.stdout.strip() == "hits 4"  # C = 2 hits in each of the last two phases
    raw = out_bin.read_bytes()
    nstate = 4 * 3 * sum(params)
    got = np.frombuffer(raw[:nstate], dtype=np.uint32)
    got16 = np.frombuffer(raw[nstate:], dtype=np.uint16)
    want, want16 = [], []
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in range(iters):
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        want.append(np.concatenate([p, m, v]).view(np.uint32))
        want16.append(p16)
    assert np.array_equal(got, np.concatenate(want))
    assert np.array_equal(got16, np.concatenate(want16))


def test_integration_c_example_compiles(tmp_path):
    """The C caller shown in INTEGRATION.md §3 compiles against the header."""
    import re
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"```c\n(.*?)```", text, re.S).group(1).replace('#include "tierflow_b200.h"\n', "")
    src = tmp_path / "integ.c"
    src.write_text('#include <stdio.h>\n#include <stdint.h>\n#include "tierflow_b200.h"\n'
                   "int main(void) {\nint iters = 2;\n" + code + "\nreturn 0;\n}\n")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-c", str(src),
                    "-o", str(tmp_path / "integ.o")], check=True)


def test_scalar_codec_matches_oracle(tf):
    """tfg_f16_to_f32 / tfg_f32_to_f16 (the one-value conversions the
    reference's fp16.hpp offers, run on the host with the kernels' codec):
    every 16-bit pattern widened, and 2^17 float patterns (every exponent,
    NaN payloads, subnormals, the overflow boundary) narrowed, f16 and bf16,
    bit-equal to the oracle."""
    import numpy as np
    import oracle
    from paper_2509_02480_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(7)
    floats = np.concatenate([rng.integers(0, 2**32, 2**17, dtype=np.uint64).astype(np.uint32),
                             np.array([0, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00001, 0xFFBFFFFF,
                                       0x477FEFFF, 0x477FF000, 0x33000000, 0x33000001, 0x387FC000],
                                      np.uint32)]).view(np.float32)
    for kind in (0, 1):
        want_w = oracle.widen16(np.arange(65536, dtype=np.uint32).astype(np.uint16), kind)
        out = C.c_uint32()  # raw bits: a Python float would quiet signalling NaNs
        out_f = C.cast(C.pointer(out), C.POINTER(C.c_float))
        got_w = np.empty(65536, np.uint32)
        for h in range(65536):
            assert lib.tfg_f16_to_f32(h, kind, out_f) == 0
            got_w[h] = out.value
        assert np.array_equal(got_w, want_w.view(np.uint32))
        want_n, _ = oracle.narrow16(floats, kind)
        h16 = C.c_uint16()
        got_n = np.empty(len(floats), np.uint16)
        for i, f in enumerate(floats.tolist()):
            if f != f:  # NaN: a Python float round trip may quiet it; check those by bits below
                continue
            assert lib.tfg_f32_to_f16(f, kind, C.byref(h16)) == 0
            got_n[i] = h16.value
        nan = np.isnan(floats)
        got_n[nan] = want_n[nan]
        assert np.array_equal(got_n, want_n)
        # NaN inputs by bits (the argument goes by value as a float: pass it through a c_float built from bits)
        for bits in floats.view(np.uint32)[nan][:2000].tolist():
            f = C.c_float.from_buffer_copy(np.uint32(bits).tobytes())
            assert lib.tfg_f32_to_f16(f, kind, C.byref(h16)) == 0
            want, _ = oracle.narrow16(np.array([bits], np.uint32).view(np.float32), kind)
            assert h16.value == int(want[0]), hex(bits)
