"""The Python binding's constants equal the C header's (include/lfe.h): every enum
member and #define the binding mirrors, parsed from the header text (CPU only)."""
import os
import re

from paper_1304_3992_b200 import lfe

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "lfe.h")


def _header_constants():
    txt = open(HEADER).read()
    consts = {}
    for body in re.findall(r"enum\s*\{([^}]*)\}", txt):
        nxt = 0
        for item in body.split(","):
            item = item.strip()
            if not item:
                continue
            m = re.match(r"(LFE_\w+)\s*(?:=\s*([0-9]+)u?)?$", item)
            assert m, item
            nxt = int(m.group(2)) if m.group(2) is not None else nxt
            consts[m.group(1)] = nxt
            nxt += 1
    for name, val in re.findall(r"#define\s+(LFE_\w+)\s+([0-9]+)\b", txt):
        consts[name] = int(val)
    return consts


def test_binding_constants_match_header():
    consts = _header_constants()
    assert "LFE_OPT_LOG_UNIT" in consts and consts["LFE_LOG_TENSOR_CORES"] == 2
    mirrored = [n for n in consts if hasattr(lfe, n)]
    assert len(mirrored) >= 20, mirrored
    bad = {n: (consts[n], getattr(lfe, n)) for n in mirrored if getattr(lfe, n) != consts[n]}
    assert not bad, bad
    # every option / mode enum the binding uses is mirrored
    for n in ("LFE_OPT_KERNEL", "LFE_OPT_TILE_W", "LFE_OPT_TILE_H", "LFE_OPT_HOST_STRIP_ROWS", "LFE_OPT_LOG_UNIT",
              "LFE_LOG_AUTO", "LFE_LOG_CUDA_CORES", "LFE_LOG_TENSOR_CORES", "LFE_KERNEL_AUTO", "LFE_KERNEL_STAGED",
              "LFE_KERNEL_FUSED", "LFE_ADAPT_ZC", "LFE_ADAPT_STD", "LFE_PEER_ROWS"):
        assert hasattr(lfe, n), n
