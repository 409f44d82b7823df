"""B200-native ISM pressure solve (arXiv 1309.7128) behind the reference's operator API."""
from .api import *  # noqa: F401,F403
