"""CPU tests of the host library through the C-ABI: packing + header wire
format (pinned to the reference's own serializer via the golden vectors),
device filters and ranking, error mapping, and the exported symbol set.
No GPU needed (and none is used)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1807_11830_b200 import hetreco as h

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "hetreco_b200.h")).read()
    declared = set(re.findall(r"\b(hetreco_[a-z0-9_]+)\s*\(", header))
    assert len(declared) > 50
    lib = ctypes.CDLL(h.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(h.EXPORTED)


def test_layout_matches_reference_serializer(golden):
    cases = [[(4, [160, 160])], [(3, [3]), (3, [2])], [(4, [32, 16, 4, 3]), (4, [32, 16, 4])],
             [(1, [7]), (6, [3, 5]), (2, [1, 1, 9]), (5, [2, 2, 2, 2, 2, 2, 2, 2])]]
    for i, case in enumerate(cases):
        layout, words = h.pack_layout([(tuple(d), h.dtype_of(t)) for t, d in case], 256)
        np.testing.assert_array_equal(words, golden[f"layout{i}_words"])
        assert layout.total_bytes == int(golden[f"layout{i}_total"][0])


def test_spec_pack_examples():
    # SPEC.md:119, :128 and the [12 B, 8 B] example
    layout, words = h.pack_layout([((160, 160), np.complex64)])
    assert layout.total_bytes == 204800
    assert words.tolist() == [1, 0, 4, 2, 160, 160, 1, 1, 1, 1, 1, 1]
    layout, words = h.pack_layout([((3,), np.float32), ((2,), np.float32)])
    assert [r.offset_bytes for r in layout.records] == [0, 256]
    assert layout.total_bytes == 512
    with pytest.raises(h.EmptyData):
        h.pack_layout([])
    with pytest.raises(h.InvalidArgument):
        h.pack_layout([((3,), np.float32)], alignment=3)


def test_pack_fuzz_properties():
    # SPEC.md acceptance 6: aligned, non-overlapping, order preserving, bijective header
    rng = np.random.default_rng(0)
    dts = [np.uint8, np.int32, np.float32, np.complex64, np.float64, np.complex128]
    for _ in range(1000):
        n = int(rng.integers(1, 17))
        shapes = [(tuple(int(x) for x in rng.integers(1, 6, int(rng.integers(1, 9)))), dts[rng.integers(0, 6)])
                  for _ in range(n)]
        align = int(2 ** rng.integers(0, 10))
        layout, words = h.pack_layout(shapes, align)
        end = 0
        for r in layout.records:
            assert r.offset_bytes % align == 0 and r.offset_bytes >= end
            end = r.offset_bytes + r.byte_size()
        assert layout.total_bytes >= end and layout.total_bytes % align == 0
        parsed = h.parse_layout_header(words.tobytes())
        assert [(p.offset_bytes, p.element_type, p.shape) for p in parsed.records] == \
               [(r.offset_bytes, r.element_type, r.shape) for r in layout.records]


def test_parse_rejects_malformed_headers():
    _, words = h.pack_layout([((4, 4), np.complex64)])
    b = words.tobytes()
    with pytest.raises(h.MalformedHeader):
        h.parse_layout_header(b[:-8])
    bad = words.copy()
    bad[2] = 99  # type code
    with pytest.raises(h.MalformedHeader):
        h.parse_layout_header(bad.tobytes())
    bad = words.copy()
    bad[3] = 9  # rank
    with pytest.raises(h.MalformedHeader):
        h.parse_layout_header(bad.tobytes())
    bad = words.copy()
    bad[7] = 2  # dim beyond rank must be 1
    with pytest.raises(h.MalformedHeader):
        h.parse_layout_header(bad.tobytes())


def test_device_filters():
    assert h.describe_filter("") == "{any}"
    assert h.describe_filter("any") == "{any}"
    assert h.describe_filter(" GPU , vendor = nvidia ,version=10.0") == \
        '{type=gpu, vendor~"nvidia", version>=10.0}'
    for bad in ("version=1", "colour=red", "tpu"):
        with pytest.raises(h.InvalidFilter):
            h.describe_filter(bad)


def test_ranking_rules():
    D = h.DeviceDescriptor.make
    cands = [D("cpu0", h.DeviceType.Cpu, "Intel", "xeon", "1.2", 8 << 30),
             D("gpu0", h.DeviceType.Gpu, "NVIDIA", "B200", "10.0", 4 << 30),
             D("gpu1", h.DeviceType.Gpu, "NVIDIA", "B200", "10.0", 180 << 30),
             D("gpu2", h.DeviceType.Gpu, "NVIDIA", "B200", "10.0", 180 << 30),
             D("acc0", h.DeviceType.Accelerator, "X", "npu", "2.0", 1 << 40)]
    assert h.select_from(cands, "") == 1 + 1        # GPU class wins, then memory, ties keep first
    assert h.select_from(cands, "cpu") == 0
    assert h.select_from(cands, "accelerator") == 4
    assert h.select_from(cands, "vendor=nvidia,version=10.0") == 2
    assert h.select_from(cands, "name=XEON") == 0
    with pytest.raises(h.NoMatchingDevice) as e:
        h.select_from(cands, "version=11.0")
    assert "gpu2" in str(e.value)  # message lists every candidate


@pytest.mark.skipif(h.cuda_device_count() > 0, reason="host has a GPU")
def test_no_gpu_means_no_device_and_no_fallback():
    assert h.enumerate_devices() == []
    with pytest.raises(h.NoMatchingDevice):
        h.ComputeSession("")
    with pytest.raises(h.NoMatchingDevice):
        h.CudaBackend(0)


def test_intrinsic_kernel_names():
    assert h.CudaBackend.intrinsic_kernel_names() == [
        "negate", "fft_radix2_pass", "complex_element_prod", "ximage_sum", "rss_combine", "matrix_add",
        "sens_recon", "rss_recon"]
