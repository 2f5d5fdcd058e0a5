"""The C-ABI boundary on the CPU: libhcmx_gpu.so loads, exports every symbol
include/hcmx_gpu.h declares, the host-only layout rules answer like the
reference, and compute entry points fail loudly without a GPU (no fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hcmx_gpu.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hcmx_gpu_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def L():
    from paper_2308_10960_b200 import build
    build.build()
    from paper_2308_10960_b200 import _lib
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    from paper_2308_10960_b200._lib import PROTOTYPES
    assert set(names) == set(PROTOTYPES), set(names) ^ set(PROTOTYPES)


def test_host_rules_match_reference_anchors(L, codec_golden):
    from paper_2308_10960_b200 import codec
    z = codec_golden
    for eps, m in zip(z["mbits_eps"], z["mbits"]):
        assert codec.mantissa_bits_for(float(eps)) == m
    for (a, b, c), e in zip(z["ebits_stats"], z["ebits"]):
        assert codec.exponent_bits_for(codec.BlockStats(a, b, bool(c))) == e
    for bad in (0.0, 1.0, -1e-4):
        with pytest.raises(ValueError):
            codec.mantissa_bits_for(bad)


def test_descriptor_widths_test_codec_128_139(L):
    # test_codec.cpp:128-139: {1, 32} at eps 4.9e-4 -> e=3; widths 14/16/24/32
    from paper_2308_10960_b200 import codec
    st = codec.BlockStats(1.0, 32.0, False)
    assert codec.exponent_bits_for(st) == 3
    widths = [codec.make_descriptor(s, 4.9e-4, st).bit_width() for s in codec.Scheme]
    assert widths == [14, 16, 24, 32]
    # compressed_size exact (test_codec.cpp:141-146)
    d = codec.FormatDescriptor(codec.Scheme.afl, 3, 10, 1.0)
    assert codec.compressed_size(0, d) == codec.header_bytes
    assert codec.compressed_size(1000, d) == codec.header_bytes + 1750


def test_size_ordering_test_codec_148_164(L, oracle):
    from paper_2308_10960_b200 import codec
    for er in range(2, 9):
        for mb in range(2, 53, 5):
            st = codec.BlockStats(1.0, 2.0 ** ((1 << er) - 2), False)
            eps = 2.0 ** -(mb + 1)
            n = 64 + 64 * (mb % 9)
            prev = 0
            for s in codec.Scheme:
                sz = codec.compressed_size(n, codec.make_descriptor(s, eps, st))
                assert sz >= prev
                prev = sz
                e, m = oracle.make_descriptor(int(s), eps, codec.exponent_bits_for(st))
                assert sz == oracle.compressed_size(n, int(s), e, m)
            assert prev <= codec.header_bytes + 8 * n


def test_wire_format_roundtrip_and_truncation(L, ref):
    from paper_2308_10960_b200 import codec
    rng = np.random.default_rng(5)
    v = np.exp(rng.uniform(0, np.log(1e3), 100))
    rb = ref.compress(v, 1e-6, 1)
    buf = codec.CompressedBuffer(codec.FormatDescriptor(codec.Scheme(rb.scheme), rb.e, rb.m, rb.scale),
                                 rb.count, rb.payload)
    wire = codec.serialize(buf)
    assert wire == ref.serialize(rb)
    back, off = codec.deserialize(wire)
    assert off == len(wire) and back.payload == buf.payload and back.count == buf.count
    with pytest.raises(codec.CorruptBufferError):
        codec.deserialize(wire[:-4])
    with pytest.raises(codec.CorruptBufferError):
        codec.deserialize(wire[:10])
    bad = bytearray(wire)
    bad[0] = 7
    with pytest.raises(codec.CorruptBufferError):
        codec.deserialize(bytes(bad))


def test_compute_without_gpu_fails_loudly(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    v = np.arange(1.0, 65.0)
    d = C.c_uint64()
    from paper_2308_10960_b200 import _lib
    desc = _lib.hcmx_descriptor()
    out = np.zeros(1024, np.uint8)
    st = L.hcmx_gpu_compress(v.ctypes.data, v.size, 1e-6, 0, C.byref(desc), out.ctypes.data, out.size,
                             C.byref(d))
    assert st == _lib.HCMX_CUDA_ERROR
    assert b"no CUDA device" in L.hcmx_gpu_last_error()
    assert L.hcmx_gpu_init(0) == _lib.HCMX_CUDA_ERROR


def test_cpp_shim_compiles_and_maps_exceptions(tmp_path):
    """include/hcmx_gpu.hpp (the binding INTEGRATION.md shows) builds against the
    library and keeps the reference's names and exception types (host-only calls)"""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "shim.cpp"
    src.write_text(r'''
#include <hcmx_gpu.hpp>
#include <cstdio>
int main() {
    namespace codec = hcmx_gpu::codec;
    const auto d = codec::make_descriptor(codec::Scheme::aflp, 1e-6, 0.5, 5);
    std::printf("%d %d %u %zu\n", (int)codec::mantissa_bits_for(1e-6), (int)d.mant_bits, d.bit_width(),
                codec::compressed_size(64, d));
    try { codec::mantissa_bits_for(2.0); } catch (const std::invalid_argument&) { std::printf("invalid_argument\n"); }
    std::vector<std::uint8_t> wire;
    codec::CompressedBuffer b{d, 0, {}};
    codec::serialize(b, wire);
    std::size_t off = 0;
    // a reference caller catches the reference's own exception type
    try { codec::deserialize(wire.data(), 10, off); } catch (const hcmx::corrupt_buffer_error&) { std::printf("corrupt\n"); }
    static_assert(std::is_same_v<hcmx_gpu::corrupt_buffer_error, hcmx::corrupt_buffer_error>);
    return 0;
}
''')
    libdir = os.path.join(root, "paper_2308_10960_b200")
    # with and (where present) without the reference's headers on the include path:
    # the shim then throws the reference's hcmx::corrupt_buffer_error (common.hpp:17-19)
    variants = [[]]
    if os.path.isfile("/root/reference/proj/include/hcmx/common.hpp"):
        variants.append(["-I/root/reference/proj/include"])
    for i, extra in enumerate(variants):
        exe = tmp_path / f"shim{i}"
        subprocess.run(["g++", "-std=c++20", "-I" + os.path.join(root, "include"), *extra, str(src), "-L" + libdir,
                        "-lhcmx_gpu", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
        m, mant, w, size = out[0].split()
        assert (m, mant, w, size) == ("19", "26", "32", str(20 + 64 * 4))  # AFLP widens m to a byte multiple
        assert out[1] == "invalid_argument" and out[2] == "corrupt"
