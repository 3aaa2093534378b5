"""HEGW v1 exchange format: byte-identical round trips with blobs written by the reference's
own serialize module (tests/golden/hegw_unit.npz), and the reference's corruption checks
(test_serialize.py:55-84 of the reference)."""
import numpy as np
import pytest

from paper_1902_04303_b200.errors import SerializationError


def _blob(golden, key):
    return golden("hegw_unit").arr("hegw." + key).tobytes()


def _params():
    from paper_1902_04303_b200 import CkksParams

    return CkksParams(log_n=8, log_l=350, log_p=45, log_p_small=30, h=16)


def test_corrupted_payload_detected(golden):
    from paper_1902_04303_b200 import serialize as S

    data = bytearray(_blob(golden, "ct_a"))
    data[40] ^= 0xFF
    with pytest.raises(SerializationError):
        S.ciphertext_from_bytes(bytes(data), _params())


def test_bad_magic_and_kind_detected(golden):
    import hashlib

    from paper_1902_04303_b200 import serialize as S

    body = bytearray(_blob(golden, "ct_a")[:-8])
    body[:4] = b"XXXX"
    resealed = bytes(body) + hashlib.blake2b(bytes(body), digest_size=8).digest()
    with pytest.raises(SerializationError):
        S.ciphertext_from_bytes(resealed, _params())
    with pytest.raises(SerializationError):
        S.evaluation_key_from_bytes(_blob(golden, "ct_a"))   # kind mismatch
    with pytest.raises(SerializationError):
        S.ciphertext_from_bytes(b"HEGW", _params())


def test_ring_degree_mismatch_detected(golden):
    from paper_1902_04303_b200 import CkksParams
    from paper_1902_04303_b200 import serialize as S

    with pytest.raises(SerializationError):
        S.ciphertext_from_bytes(_blob(golden, "ct_a"), CkksParams(log_n=9, log_l=350, log_p_small=30))


@pytest.mark.gpu
def test_reference_blobs_roundtrip_bit_exact(golden):
    from paper_1902_04303_b200 import serialize as S
    from tests.gpu_helpers import assert_ct_equal

    params = _params()
    ct = S.ciphertext_from_bytes(_blob(golden, "ct_a"), params)
    assert_ct_equal(ct, golden("unit_ops"), "ct_a")
    for key in ("ct_a", "ct_mult"):
        blob = _blob(golden, key)
        assert S.ciphertext_to_bytes(S.ciphertext_from_bytes(blob, params)) == blob
    blob = _blob(golden, "pt_mask")
    assert S.plaintext_to_bytes(S.plaintext_from_bytes(blob), 8) == blob
    blob = _blob(golden, "sk")
    assert S.secret_key_to_bytes(S.secret_key_from_bytes(blob), 8) == blob
    blob = _blob(golden, "pk")
    assert S.public_key_to_bytes(S.public_key_from_bytes(blob), 8) == blob
    blob = _blob(golden, "evk")
    assert S.evaluation_key_to_bytes(S.evaluation_key_from_bytes(blob), 8) == blob
    blob = _blob(golden, "rot")
    rk = S.rotation_keys_from_bytes(blob)
    assert sorted(rk.keys) == [1, 2, 4, 8, 16, 32, 64] and rk.conj is not None
    assert S.rotation_keys_to_bytes(rk, 8) == blob


@pytest.mark.gpu
def test_gpu_result_serialises_like_reference(golden):
    """Multiply the deserialised reference input on the GPU and compare the HEGW bytes of the
    result with the reference's own serialisation of its result."""
    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200 import serialize as S

    params = _params()
    a = S.ciphertext_from_bytes(_blob(golden, "ct_a"), params)
    evk = S.evaluation_key_from_bytes(_blob(golden, "evk"))
    rot = S.rotation_keys_from_bytes(_blob(golden, "rot"))
    out = hg.HeEngine(params, evk, rot).mult(a, a)
    assert S.ciphertext_to_bytes(out) == _blob(golden, "ct_mult")
    assert np.frombuffer(_blob(golden, "ct_mult")[:4], dtype=np.uint8).tobytes() == b"HEGW"
