"""B200-native split-FC softmax cross-entropy (Whale, arXiv 2011.09208) -- C-ABI + thin binding."""
from ._lib import WhaleError, whale_splitfc_plan  # noqa: F401
from .splitfc import SplitFCSoftmaxCE, emulated_ranks, split_fc_softmax_ce  # noqa: F401
