// Internal (non-ABI) helpers shared by the library's translation units.
#pragma once

// Set the calling thread's vt_last_error() message; returns `code`.
int vt_set_error(int code, const char* msg);
