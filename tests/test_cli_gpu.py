"""The device CLI backend (paper_2104_14641_b200.cli) against the reference CLI's own output bytes:
rank --json (incl. failed candidates' diagnostics) and search --json --trace (tests/golden/cli,
written by oracle/gen_golden.py from the reference)."""

import contextlib
import io
import json

import pytest

from golden_util import GOLDEN

pytestmark = pytest.mark.gpu

CLI = GOLDEN / "cli"
MANIFEST = json.loads((CLI / "manifest.json").read_text())


@pytest.mark.parametrize("run", MANIFEST, ids=[r["name"] for r in MANIFEST])
def test_cli_matches_reference_bytes(run, tmp_path):
    from paper_2104_14641_b200 import cli
    argv = [a.replace("{dir}", str(CLI)) for a in run["argv"]]
    if run["trace"]:
        i = argv.index("--trace")
        argv[i + 1] = str(tmp_path / "trace.csv")
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(argv)
    assert code == 0
    assert buf.getvalue() == (CLI / f"{run['name']}.out").read_text()
    if run["trace"]:
        assert (tmp_path / "trace.csv").read_text() == (CLI / run["trace"]).read_text()


def test_cli_user_errors(tmp_path):
    from paper_2104_14641_b200 import cli
    assert cli.main(["rank", str(tmp_path / "missing.json"), str(tmp_path / "x.json"), "--arch", "x86-avx2"]) == 1
    (tmp_path / "s.json").write_text("[]")
    assert cli.main(["rank", str(CLI / "matmul48.json"), str(tmp_path / "s.json"), "--arch", "x86-avx2"]) == 1
    assert cli.main(["rank", str(CLI / "matmul48.json"), str(CLI / "matmul48_scheds.json"), "--arch", "nope"]) == 1
    # analyze: the mock emitter is not part of the backend; a missing --code file is a user error
    assert cli.main(["analyze", str(CLI / "matmul48.json"), "--arch", "x86-avx2"]) == 1
    assert cli.main(["analyze", str(CLI / "matmul48.json"), "--code", str(tmp_path / "no.s"), "--arch", "x86-avx2"]) == 1
