"""Host side of the zero-copy API bridge (api_bridge.py):
column_encoder round-trips with the reference codec (boundary.py:59-141),
rejects malformed columns the way the reference rejects malformed lists, and
install()/uninstall() rebind and restore exactly the reference names the
bridge replaces (api.py build_program / evaluate / encode_value,
foreign.weld_new_data, cli.decode_value / new_data_object).  No device work."""
import numpy as np
import pytest

import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import api_bridge as br
from weldmill.boundary import decode_value, encode_value
from weldmill.errors import EncodeError
from weldmill.parser import parse_type_text as T

CASES = [
    ("vec[i64]", [3, -1, 1 << 40, 0]),
    ("vec[i32]", [7, -(1 << 31), (1 << 31) - 1]),
    ("vec[f64]", [0.5, -2.25, 1e300, 0.0]),
    ("vec[bool]", [True, False, True]),
    ("vec[{i32,f64}]", [(1, 0.5), (2, -1.5)]),
    ("vec[{i64,bool,f64}]", [(9, True, 2.0), (-9, False, 3.5), (0, True, 0.0)]),
    ("vec[f64]", []),
]


def _np_cols(ty, payload):
    from paper_1709_06416_b200.irtypes import NPTYPE, leaves
    ks = leaves(T(ty).elem)
    if len(ks) == 1:
        return np.asarray(payload, dtype=NPTYPE[ks[0]] if ks[0] != "bool" else bool)
    cols = list(zip(*payload)) if payload else [[] for _ in ks]
    return tuple(np.asarray(c, dtype=bool if k == "bool" else NPTYPE[k]) for c, k in zip(cols, ks))


@pytest.mark.parametrize("ty,payload", CASES, ids=[f"{t}-{len(p)}" for t, p in CASES])
def test_column_encoder_matches_reference_codec(ty, payload):
    t = T(ty)
    want = encode_value(payload, t)
    assert wg.column_encoder.encode(_np_cols(ty, payload), t) == want
    assert wg.column_encoder.encode(want, t) == want            # boundary bytes pass through
    assert wg.column_encoder.encode(payload, t) == want         # lists: the reference codec
    assert wg.column_encoder.decode(want, t) == decode_value(want, t)


def test_column_encoder_rejects_malformed_columns():
    t = T("vec[{i32,f64}]")
    with pytest.raises(EncodeError):
        wg.column_encoder.encode((np.arange(3, dtype=np.int32),), t)              # missing column
    with pytest.raises(EncodeError):
        wg.column_encoder.encode((np.arange(3, dtype=np.int32), np.arange(2.0)), t)   # ragged
    with pytest.raises(EncodeError):
        wg.column_encoder.encode((np.arange(3.0), np.arange(3.0)), t)             # float into i32
    with pytest.raises(EncodeError):
        wg.column_encoder.encode((np.array([1 << 40]), np.array([0.0])), t)       # out of i32 range
    with pytest.raises(EncodeError):
        wg.column_encoder.encode(b"\x05" + b"\x00" * 7 + b"\x00" * 11, t)         # count vs length


def test_scalar_list_fast_path_defers_odd_lists_to_the_reference():
    assert br._scalar_list_column([1, 2, 3], T("vec[i64]")).dtype == np.int64
    assert br._scalar_list_column([1.5, 2], T("vec[i64]")) is None      # reference raises EncodeError
    assert br._scalar_list_column([True, False], T("vec[i64]")) is None  # bool is not an int there
    assert br._scalar_list_column([1 << 40], T("vec[i32]")) is None      # out of range
    assert br._scalar_list_column([1, 2], T("vec[bool]")) is None
    assert br._scalar_list_column(["a"], T("vec[f64]")) is None


def test_install_rebinds_and_restores_the_reference_names():
    from weldmill import api, cli, foreign
    names = [(api, "build_program"), (api, "evaluate"), (api, "encode_value"), (foreign, "weld_new_data"),
             (cli, "decode_value"), (cli, "new_data_object")]
    before = [getattr(m, n) for m, n in names]
    wg.install()
    try:
        assert all(getattr(m, n) is not b for (m, n), b in zip(names, before))
        assert br.installed()
    finally:
        wg.uninstall()
    assert [getattr(m, n) for m, n in names] == before
    wg.install(zero_copy=False)
    try:
        assert api.build_program is before[0] and api.evaluate is not before[1]
    finally:
        wg.uninstall()
    assert [getattr(m, n) for m, n in names] == before
