"""adaptgear.selector served by paper_2305_17408_b200.selector (drop-in harness)."""
from paper_2305_17408_b200.selector import *  # noqa: F401,F403
from paper_2305_17408_b200.selector import INTER, INTRA  # noqa: F401
