"""B200-native JSON parse path (arXiv:1902.08318 two-stage design) behind the
reference's jsontape C ABI.  See DESIGN.md."""
from .jsontape import (CAPACITY, DEPTH_ERROR, EMPTY, ERROR_NAMES, NUMBER_ERROR, OK,  # noqa: F401
                       STRING_ERROR, TAPE_ERROR, UTF8_ERROR, Document, Parser, Result,
                       error_name, load_library)
