"""The driver's round-end smoke check (__graft_entry__.smoke) stays green."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.smoke()
