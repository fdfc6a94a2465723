"""Exception hierarchy mirroring laq::Error (proj/include/laq/error.hpp:10-74).

Every C-ABI status code (include/laq_b200.h, enum laq_status) maps to one of
these, so callers can catch as narrowly as the reference's tests do
(e.g. CHECK_THROWS_AS(..., DomainError), tests/test_laqops.cpp:161).
"""


class Error(RuntimeError):
    """laq::Error (error.hpp:10)."""


class IndexError_(Error):
    """laq::IndexError (error.hpp:15)."""


class ShapeError(Error):
    """laq::ShapeError (error.hpp:20)."""


class FormatError(Error):
    """laq::FormatError (error.hpp:25)."""


class NameError_(Error):
    """laq::NameError (error.hpp:30)."""


class TypeError_(Error):
    """laq::TypeError (error.hpp:35)."""


class MappingError(Error):
    """laq::MappingError (error.hpp:40)."""


class DomainError(Error):
    """laq::DomainError (error.hpp:45)."""


class DuplicateKeyError(Error):
    """laq::DuplicateKeyError (error.hpp:51)."""


class TreeError(Error):
    """laq::TreeError (error.hpp:56)."""


class ModelError(Error):
    """laq::ModelError (error.hpp:61)."""


class GenError(Error):
    """laq::GenError (error.hpp:66)."""


class CapacityError(Error):
    """laq::CapacityError (error.hpp:71)."""


class CudaError(Error):
    """Device/driver failure; no reference equivalent (LAQ_ERR_CUDA)."""


class UnsupportedError(Error):
    """Valid input outside this build's device paths (LAQ_ERR_UNSUPPORTED)."""


# Aliases with the reference's names (shadowing builtins only inside this module's namespace).
IndexError = IndexError_  # noqa: A001
NameError = NameError_  # noqa: A001
TypeError = TypeError_  # noqa: A001

BY_CODE = {
    1: Error, 2: IndexError_, 3: ShapeError, 4: FormatError, 5: NameError_, 6: TypeError_,
    7: MappingError, 8: DomainError, 9: DuplicateKeyError, 10: TreeError, 11: ModelError,
    12: GenError, 13: CapacityError, 100: CudaError, 101: UnsupportedError,
}


def raise_for(code: int, msg: str):
    if code == 0:
        return
    raise BY_CODE.get(code, Error)(msg)
