"""Byte accounting for lookup exchanges (embserve/wire.py:9-41).

The B200 build ships indices and pooled vectors over NVLink (NCCL) instead of
modelled RDMA messages; these formulas are kept so exchange byte counts stay
comparable with the reference's reports (pushdown payload D*4 vs raw n*D*4).
"""

ELEMENT_WIDTH = 4
INDEX_BYTES = 8
MSG_HEADER_BYTES = 32
COUNT_FIELD_BYTES = 8
CREDIT_FIELD_BYTES = 8


def request_bytes(num_indices: int, carries_credit: bool = False) -> int:
    return MSG_HEADER_BYTES + num_indices * INDEX_BYTES + (CREDIT_FIELD_BYTES if carries_credit else 0)


def raw_response_bytes(num_rows: int, dim: int) -> int:
    return MSG_HEADER_BYTES + num_rows * dim * ELEMENT_WIDTH


def partial_response_bytes(dim: int) -> int:
    return MSG_HEADER_BYTES + dim * ELEMENT_WIDTH + COUNT_FIELD_BYTES


def credit_message_bytes() -> int:
    return MSG_HEADER_BYTES + CREDIT_FIELD_BYTES


def embedding_payload_bytes(num_vectors: int, dim: int) -> int:
    return num_vectors * dim * ELEMENT_WIDTH
