"""__graft_entry__.smoke() (the driver's round-end GPU check) runs clean here too."""

import pytest

pytestmark = pytest.mark.gpu


def test_graft_smoke(cuda):
    import __graft_entry__ as g
    g.smoke()
