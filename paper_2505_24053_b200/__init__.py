"""B200-native 3DGEER rendering hot path (arXiv 2505.24053).

Drop-in for ``raygauss.renderer.render`` / ``render_backward`` and
``raygauss.association.build_render_graph``: the host code here validates and
marshals the reference's types, then calls the ``extern "C"`` ABI of
``libgeer_b200.so`` (include/geer.h), whose sm_100a kernels do all the work.
There is no CPU fallback: importing the renderer without the built library
raises.
"""

__version__ = "0.1.0"


def install(with_graph: bool | None = None):
    """Patch a live ``raygauss`` so its render / render_backward / build_render_graph run here (dropin.py)."""
    from .dropin import install as _install

    return _install(with_graph)


def uninstall():
    from .dropin import uninstall as _uninstall

    _uninstall()
