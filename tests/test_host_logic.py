"""CPU-only checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/lancelot_b200.h declares, there is no CPU
fallback, and the host-side planning logic matches the reference's own unit
tests (test_distance.cpp)."""
import ctypes
import math
import os

import pytest

import paper_2408_06197_b200.lancelot as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(L.LIB_PATH)
    names = L.exported_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python mirror binds every one of them
    bound = L.lib()
    for n in names:
        assert hasattr(bound, n)


def test_cpp_mirror_plan_logic_matches_reference():
    """plan_unfold / fixed_plan / slot_reduce_steps of the C++ mirror
    (compiled here, no device) agree with the Python mirror (which the
    reference's test_distance.cpp cases below pin)."""
    import subprocess
    import tempfile

    prog = r"""
#include <cstdio>
#include "lancelot_b200.hpp"
namespace L = lancelot_b200;
int main() {
  const double cases[][5] = {{0.17, 0.072, 4194304, 12582912, 32768}, {1e-4, 9e-5, 4194304, 1073741824, 32768},
                             {2.0, 1.0, 1.0, 3.0, 1024}, {1.0, 1.0, 1.0, 100.0, 256}};
  for (const auto& c : cases) {
    const L::HoistPlan p = L::plan_unfold(c[0], c[1], c[2], c[3], (std::size_t)c[4]);
    std::printf("%zu %.17g %zu\n", p.k, p.cost, L::slot_reduce_steps(p.n, p.k).size());
  }
  std::printf("%zu\n", L::fixed_plan(L::HoistMode::full, 4096).k);
  try { L::plan_unfold(1, 1, 2, 1, 8); } catch (const L::InfeasibleError&) { std::printf("infeasible\n"); }
  try { L::fixed_plan(L::HoistMode::dynamic_lp, 8); } catch (const L::UsageError&) { std::printf("usage\n"); }
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.cpp")
        with open(src, "w") as f:
            f.write(prog)
        exe = os.path.join(d, "p")
        subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L", os.path.dirname(L.LIB_PATH), "-llancelot_b200",
                        f"-Wl,-rpath,{os.path.dirname(L.LIB_PATH)}"], check=True)
        lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    for line, c in zip(lines, [(0.17, 0.072, 4194304, 12582912, 32768),
                               (1e-4, 9e-5, 4194304, 1073741824, 32768),
                               (2.0, 1.0, 1.0, 3.0, 1024), (1.0, 1.0, 1.0, 100.0, 256)]):
        k, cost, nsteps = line.split()
        p = L.plan_unfold(*c[:4], int(c[4]))
        assert int(k) == p.k and float(cost) == p.cost
        assert int(nsteps) == len(L.slot_reduce_steps(p.n, p.k))
    assert lines[4] == "13" and lines[5] == "infeasible" and lines[6] == "usage"


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(L.DeviceError):
        L.CkksContext(L.CkksParams(ring_degree=1024, security=L.SecurityLevel.none))


def test_chunk_counts():  # test_distance.cpp:69-76
    assert L.chunk_count_for(1, 128) == 1
    assert L.chunk_count_for(128, 128) == 1
    assert L.chunk_count_for(129, 128) == 2
    assert L.chunk_count_for(61706, 4096) == 16
    with pytest.raises(L.ShapeError):
        L.chunk_count_for(0, 128)
    with pytest.raises(L.ShapeError):
        L.chunk_count_for(4, 0)


def test_prescale_trigger():  # test_distance.cpp:78-85
    assert L.distance_prescale(61706, math.ldexp(1.0, 20)) == 1.0
    assert L.distance_prescale(1 << 22, math.ldexp(1.0, 20)) == 1.0
    big = 1 << 23
    assert L.distance_prescale(big, math.ldexp(1.0, 20)) == pytest.approx(1 / math.sqrt(big))


def test_unfold_planning():  # test_distance.cpp:189-205
    assert L.plan_unfold(2.0, 1.0, 1.0, 4.0, 16).k == 4
    assert L.plan_unfold(1.0, 1.0, 1.0, 100.0, 16).k == 1
    assert L.plan_unfold(5.0, 1.0, 1.0, 2.0, 16).k == 2
    with pytest.raises(L.InfeasibleError):
        L.plan_unfold(1.0, 1.0, 4.0, 2.0, 16)
    with pytest.raises(L.WidthError):
        L.plan_unfold(1.0, 1.0, 1.0, 2.0, 12)
    with pytest.raises(L.ParameterError):
        L.plan_unfold(0.0, 1.0, 1.0, 2.0, 16)


def test_fixed_plans_and_steps():
    assert L.fixed_plan(L.HoistMode.off, 16).k == 1
    assert L.fixed_plan(L.HoistMode.full, 16).k == 5
    with pytest.raises(L.UsageError):
        L.fixed_plan(L.HoistMode.dynamic_lp, 16)
    assert L.slot_reduce_steps(16, 1) == [1, 2, 4, 8]
    assert L.slot_reduce_steps(16, 3) == [1, 2, 3, 4, 8]
    assert L.slot_reduce_steps(16, 5) == list(range(1, 16))
    assert L.slot_reduce_steps(1, 1) == []
    with pytest.raises(L.ParameterError):
        L.slot_reduce_steps(16, 0)
    with pytest.raises(L.WidthError):
        L.slot_reduce_steps(12, 1)


def test_params_validation():
    with pytest.raises(L.ParameterError):
        L.CkksParams(ring_degree=1000).validate()
    with pytest.raises(L.ParameterError):
        L.CkksParams(scale_bits=30).validate()


class _MT64:
    """std::mt19937_64 (the reference Sampler's engine), restated for the test."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & (2 ** 64 - 1)
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & (
                2 ** 64 - 1)
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            for k in range(312):
                y = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                x = self.mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    x ^= 0xB5026F5AA96619E9
                self.mt[k] = x
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & (2 ** 64 - 1)


def test_sampler_stream_and_derive_seed():
    """The host Sampler behind lcl_pack_and_encrypt / lcl_build_mask is the
    reference's (sampling.cpp): derive_seed's splitmix64 finaliser and
    uniform_real = (raw >> 11) * 2^-53 over std::mt19937_64. Host-only: no
    device needed."""
    import paper_2408_06197_b200.lancelot as L

    def splitmix(root, tag):
        z = (root + 0x9E3779B97F4A7C15 * (tag + 1)) & (2 ** 64 - 1)
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
        return z ^ (z >> 31)

    for root, tag in [(1, 0xAB1A7E), (1, 5), (7, 0x3000000000000000)]:
        assert L.derive_seed(root, tag) == splitmix(root, tag)
    seed = L.derive_seed(1, 0xAB1A7E)
    mt = _MT64(seed)
    want = [(mt() >> 11) * 2.0 ** -53 for _ in range(1000)]
    got = L.Sampler(seed).uniform_real(1000)
    assert list(got) == want


def test_stack_clients_zero_copy_only_for_the_whole_batch():
    """views of a prefix slice share data pointers with the parent
    but must not be returned as the batch (clients would be strided by the
    parent's chunk count)."""
    import torch

    big = torch.empty(3, 5, 2, 2, 4, dtype=torch.int64)
    big.copy_(torch.arange(big.numel()).reshape(big.shape))
    whole = [L.PackedWeights(big[i], 10, 1.0, 1.0) for i in range(3)]
    assert L.stack_clients(whole).data_ptr() == big.data_ptr()  # zero copy
    pre = big[:, :2]
    part = [L.PackedWeights(pre[i], 4, 1.0, 1.0) for i in range(3)]
    got = L.stack_clients(part)
    assert tuple(got.shape) == (3, 2, 2, 2, 4)
    assert torch.equal(got, pre)
    limbs = big[:, :, :, :1]
    lv = [L.PackedWeights(limbs[i], 10, 1.0, 1.0) for i in range(3)]
    assert torch.equal(L.stack_clients(lv), limbs)


def test_package_import_sets_32_hardware_queues():
    """The host round runs ~16 streams; the package asks for 32 hardware
    work queues before any CUDA context exists (an explicit setting wins)."""
    import subprocess
    import sys

    code = ("import os; os.environ.pop('CUDA_DEVICE_MAX_CONNECTIONS', None); "
            "import paper_2408_06197_b200; print(os.environ['CUDA_DEVICE_MAX_CONNECTIONS'])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "32"
    code2 = ("import os; os.environ['CUDA_DEVICE_MAX_CONNECTIONS'] = '16'; "
             "import paper_2408_06197_b200; print(os.environ['CUDA_DEVICE_MAX_CONNECTIONS'])")
    out = subprocess.run([sys.executable, "-c", code2], cwd=root, capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "16"
