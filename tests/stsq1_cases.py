"""Malformed STSQ1 variants derived from a valid file's bytes (shared by the golden script, which
records the reference reader's exception class and message for each, and the tests)."""


def variants(good: bytes) -> dict:
    head, _, payload = good.partition(b"\n\n")
    lines = head.split(b"\n")

    def with_line(i, new):
        ls = list(lines)
        ls[i] = new
        return b"\n".join(ls) + b"\n\n" + payload

    return {
        "no_blank_line": head + b"\n" + payload.replace(b"\n\n", b"\n."),
        "bad_magic": with_line(0, b"STSQ2"),
        "not_ascii": with_line(1, b"dims: 9 7 \xff"),
        "missing_times": b"\n".join(lines[:5]) + b"\n\n" + payload,
        "wrong_key": with_line(2, b"spacin: 0.5 0.25"),
        "unparseable_dims": with_line(1, b"dims: 9 seven"),
        "two_frame_counts": with_line(4, b"frames: 3 4"),
        "length_mismatch": with_line(3, b"origin: 0.0"),
        "times_mismatch": with_line(5, b"times: 0.0 1.0"),
        "invalid_grid": with_line(1, b"dims: 9 1"),
        "truncated": good[:-5],
        "trailing": good + b"\x00" * 8,
        # payload / sequence checks the reference makes after the header (Image and ImageSequence,
        # grid.py:104-150): plain ValueError, not a SequenceFormatError
        "nonfinite": head + b"\n\n" + payload[:4] + b"\x00\x00\xc0\x7f" + payload[8:],
        "one_frame": b"\n".join(lines[:4] + [b"frames: 1", b"times: 0.0"]) + b"\n\n" + payload[:len(payload) // 3],
        "times_not_increasing": with_line(5, b"times: 0.0 0.5 0.5"),
    }
