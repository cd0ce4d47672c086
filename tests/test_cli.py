"""The command line (paper_2104_08865_b200.__main__) against the reference
CLI's contract for its hash-path commands (pkg/tests/test_cli.py:17-72,
131-153).  parse_size runs anywhere; the rest hash on the GPU."""

import pytest

from paper_2104_08865_b200.__main__ import main, parse_size


def _run(capsys, *argv):
    try:
        code = main(list(argv))
    except SystemExit as exc:  # argparse usage errors
        code = exc.code
    out, err = capsys.readouterr()
    return code, out, err


def test_parse_size_suffixes():
    # pkg/tests/test_cli.py:17-23
    assert parse_size("1") == 1
    assert parse_size("1K") == 1024
    assert parse_size("2m") == 2 * 1024 ** 2
    assert parse_size("1E") == 1024 ** 6
    import argparse

    with pytest.raises(argparse.ArgumentTypeError):
        parse_size("")
    with pytest.raises(argparse.ArgumentTypeError):
        parse_size("12Q")


@pytest.mark.gpu
def test_hash_file_deterministic_and_seed_forms_agree(capsys, tmp_path):
    # pkg/tests/test_cli.py:33-53
    f = tmp_path / "in.bin"
    f.write_bytes(bytes(range(256)) * 50)
    code1, out1, _ = _run(capsys, "hash", "--variant", "32", str(f))
    code2, out2, _ = _run(capsys, "hash", "--variant", "32", str(f))
    assert code1 == code2 == 0 and out1 == out2 and len(out1.strip()) == 64
    seed = bytes(range(32))
    sf = tmp_path / "seed.bin"
    sf.write_bytes(seed)
    _, a, _ = _run(capsys, "hash", "--seed-hex", seed.hex(), str(f))
    _, b, _ = _run(capsys, "hash", "--seed-file", str(sf), str(f))
    assert a == b and a != out1


@pytest.mark.gpu
def test_hash_usage_and_io_errors_exit_2(capsys, tmp_path):
    # pkg/tests/test_cli.py:55-72
    f = tmp_path / "in.bin"
    f.write_bytes(b"abc")
    assert _run(capsys, "hash", "--variant", "20", str(f))[0] == 2
    assert _run(capsys, "hash", "--seed-hex", "abcd", str(f))[0] == 2
    short = tmp_path / "short.bin"
    short.write_bytes(b"x" * 31)
    assert _run(capsys, "hash", "--seed-file", str(short), str(f))[0] == 2
    assert _run(capsys, "hash", str(tmp_path / "missing.bin"))[0] == 2


@pytest.mark.gpu
def test_vectors_round_trip_and_corruption(capsys, tmp_path):
    # pkg/tests/test_cli.py:131-153
    path = tmp_path / "vectors.txt"
    assert _run(capsys, "vectors", "--emit", str(path))[0] == 0
    lines = path.read_text().strip().splitlines()
    assert len(lines) == 4 * 2 * 8
    code, out, _ = _run(capsys, "vectors", "--check", str(path))
    assert code == 0 and "verified" in out
    text = path.read_text()
    last = text.rstrip()[-1]
    path.write_text(text.rstrip()[:-1] + ("0" if last != "0" else "1") + "\n")
    code, out, err = _run(capsys, "vectors", "--check", str(path))
    assert code == 1 and "mismatch" in out and "disagree" in err
