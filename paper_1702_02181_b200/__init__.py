"""B200-native dynamic batching (arXiv 1702.02181, TensorFlow Fold §2): GPU scheduler +
level executor behind the C ABI in include/fold.h (libfold.so), with a thin binding
(`paper_1702_02181_b200.fold`) and a data-parallel driver (`paper_1702_02181_b200.dp`)."""
from . import build  # noqa: F401
