"""Helpers shared by the parity tests (fixture decoding, output digests)."""
import struct

FNV_OFFSET = 1469598103934665603
FNV_PRIME = 1099511628211
MASK = (1 << 64) - 1


def fnv1a(data: bytes, h: int = FNV_OFFSET) -> int:
    for b in data:
        h ^= b
        h = (h * FNV_PRIME) & MASK
    return h


def kernel_hash(text: str) -> str:
    return "%016x" % fnv1a(text.encode())


def _words(hexstr: str):
    return [int(hexstr[i:i + 8], 16) for i in range(0, len(hexstr), 8)]


def outputs_hash(outputs: dict) -> str:
    """Digest of an output BufferMap exactly as oracle/ref_dump.cpp buffers_hash:
    names in map order, element kind byte (I32=0, F32=1), little-endian words,
    every f32 NaN canonicalised to 0x7fc00000."""
    h = FNV_OFFSET
    for name in sorted(outputs, key=lambda s: s.encode()):
        buf = outputs[name]
        h = fnv1a(name.encode(), h)
        is_i32 = buf["type"] == "i32"
        h = fnv1a(bytes([0 if is_i32 else 1]), h)
        for w in _words(buf["hex"]):
            if not is_i32 and (w & 0x7F800000) == 0x7F800000 and (w & 0x7FFFFF):
                w = 0x7FC00000
            h = fnv1a(struct.pack("<I", w), h)
    return "%016x" % h


def fixture_test_json(t: dict) -> dict:
    """ref_dump test record -> TestCase JSON with bit-exact "hex" buffers."""
    doc = {"inputs": {}, "oracle": {}, "scalars": {}}
    for section in ("inputs", "oracle"):
        for name, b in t.get(section, {}).items():
            doc[section][name] = {"type": b["elem"], "hex": b["hex"]}
    kinds = {0: "i32", 1: "f32", 2: "bool"}
    for name, s in t.get("scalars", {}).items():
        k = kinds[s["kind"]]
        doc["scalars"][name] = {"type": k, "value": s["i"] if k == "i32" else
                                (s["f"] if k == "f32" else s["b"])}
    return doc


def hex_double(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", x))[0]


STATUS_NAME = {0: "completed", 1: "trap", 2: "budget"}
