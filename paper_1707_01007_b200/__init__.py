"""B200-native CFPQ closure (arXiv 1707.01007): libcfpq + its Python binding."""
from . import cfpq  # noqa: F401
from .cfpq import Grammar, Graph, Result, closure, closure_reuse, options, version  # noqa: F401
